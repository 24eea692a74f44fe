// api.cu — C ABI (include/rapid.h) and the host orchestrator that enqueues the RAPID hot
// path on a CUDA stream.  The host only plans geometry tables and launches kernels; every
// step of the method runs in kernels.cu.  No CPU fallback exists: without a CUDA device
// rapid_init fails.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "rapid.h"

using namespace rapid;

namespace {

struct Ctl {  // per-segmentation device control block (zeroed at the start of each call)
  unsigned long long cnt[MAXS][MAXSW][4][NCNT];
  unsigned long long prop_count[MAXS * MAXSW * 4];
  unsigned long long cand_count[MAXS * MAXSW * 4];
  unsigned long long stage_info[MAXS][4];
  unsigned int victim_any[MAXS];
  unsigned int remap_pending[MAXS];
  unsigned int nwork[MAXS];
  unsigned int err;
  unsigned int vtotal, deg_total, npairs, atotal;
  unsigned int mflag[2];  // cooperative merge match: pending flags per round parity
  unsigned int wq[MAXS * MAXSW * 4];  // k_sweep work-queue counters, one per phase
  unsigned int list_count[MAXS * MAXSW * 4];  // k_bset_list: candidate-list lengths, one per phase
  unsigned int big;  // K3: some snapshot size exceeded the call's packed-delta limit (K5 then REDs the sums)
};

struct StagePlan {
  int nbx = 0, nby = 0, b = 0, tiles_x = 0, tiles_y = 0;
  std::vector<int32_t> xs, ys, px, py, cxs, cys;
  size_t o_xs = 0, o_ys = 0, o_px = 0, o_py = 0, o_cxs = 0, o_cys = 0;
  size_t bsum_off = 0;  // in uint64 elements
  bool smallb = false;  // block stage with (max block area) x (max coordinate) < 2^22: K4's 32-bit position factors
  int32_t maxn_lim = 0;  // uniform stages: K5 packs its deltas while every snapshot size is <= this
};

struct Plan {
  bool valid = false;
  int B = 0, H = 0, W = 0, M = 0, nst = 0;
  int bs[MAXS] = {0};
  int rows = 0, cols = 0;
  std::vector<int32_t> X, Y, cellx, celly, bxp, byp, b0x, b0y;
  size_t o_X = 0, o_Y = 0, o_cellx = 0, o_celly = 0, o_bxp = 0, o_byp = 0, o_b0x = 0, o_b0y = 0;
  StagePlan st[MAXS];
  std::vector<int32_t> tab;
  size_t bsum_total = 0;   // uint64 elements
  size_t map_max = 0;      // int32 elements (non-pixel stage maps)
  size_t props_max = 0;    // proposals per phase upper bound
  size_t tiles_max = 0;
};

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
};

struct ProfEv {
  int cls, stage;
  cudaEvent_t a, b;
};

}  // namespace

struct rapid_ctx {
  int device = 0;
  int sm_count = 148;
  uint64_t cap_px = 0, cap_sp = 0;
  int status = RAPID_OK;
  std::string err;
  Plan plan;
  rapid_params last{};
  bool have_run = false;
  cudaStream_t last_stream = nullptr;
  uint32_t stamp_base = 1;
  int launches = 0;
  // per-superpixel arrays (cap_sp)
  unsigned long long *sums = nullptr, *rc = nullptr, *dsum = nullptr;
  Rec *rec = nullptr;
  int32_t *init = nullptr, *out = nullptr, *remap = nullptr;
  int32_t *head = nullptr, *vlist = nullptr, *alist = nullptr, *pairs = nullptr;
  uint8_t *alive = nullptr, *active = nullptr, *victim = nullptr;
  int8_t *y = nullptr;
  uint32_t *dirty = nullptr;
  unsigned int *deg = nullptr, *chunk = nullptr;
  // merge hash
  size_t hcap = 0;
  unsigned long long *hkeys = nullptr, *candE = nullptr;
  unsigned int *hvals = nullptr;
  int32_t *hnext = nullptr, *candT = nullptr, *candV = nullptr;
  uint32_t *mlock = nullptr, *res = nullptr;
  Ctl *ctl = nullptr;
  // plan-sized buffers
  DevBuf tab, bsum, maps[2], props, work, cands, bset, vtile;
  // host-API staging
  DevBuf himg, hlab;
  // occupancy
  int scan_grid = 0, eval_grid = 0, sweep_grid = 0, tiles_grid = 0;  // persistent grid sizes (CTAs)
  int sweep_tail = 25;  // RAPID_SWEEP_TAIL: % of K4's words dealt in quarter-size groups at the end (block stages)
  int sweep_gpw = 2;  // K4 word groups per warp (RAPID_SWEEP_GPW overrides, A/B testing)
  int sweep_list_minb = 0;  // RAPID_SWEEP_LIST=b: block stages with blocks >= b take the per-phase candidate list (0: off)
  int snap_ctas = 4;  // RAPID_SNAP_CTAS: K3 CTAs per SM
  bool packed = true;  // RAPID_PACKED=0: K5 always issues the six int64 REDs per run on the sums
  bool packed_force = false;  // RAPID_PACKED=1: packed deltas below the size crossover too (tests)
  int packed_lim = 0;  // RAPID_PACKED_LIM=n (> 0): caps the stages' size limits (tests the per-phase switch)
  bool fuse_snap = false;  // RAPID_FUSE_SNAP=1: K3 of the next phase runs at the end of a cooperative K5 (measured: same step time)
  bool bset_parent = true;  // dyadic stages: boundary sets from the parent map (RAPID_BSET_PARENT=0: child-map tile pass)
  bool no_smallb = false;   // RAPID_SWEEP_NO_SMALLB=1: every block stage takes K4's 64-bit position-factor variant (parity-tested variant)
  bool fuse_bset = false;  // RAPID_FUSE_BSET=1: dyadic transitions also write the next stage's boundary sets (measured: no faster than the separate pass)
  bool use_bset = true;  // RAPID_SWEEP=scan selects the full-scan path K4a + K4b (A/B testing)
  // CUDA graph of the whole segmentation (one launch per call): captured on a private stream,
  // replayed while the key (buffers, geometry, params, profiling level, plan) is unchanged
  bool use_graph = true;  // RAPID_NO_GRAPH=1 enqueues the kernels one by one (A/B testing)
  bool l2_persist = false;  // RAPID_L2_PERSIST=1: L2 access-policy window on the sums (graph path)
  cudaStream_t cap_stream = nullptr;
  unsigned plan_gen = 0;
  struct GraphKey {
    const void *image;
    const void *labels;
    int H, W, prof;
    unsigned plan_gen;
    rapid_params p;
  };
  struct GraphEntry {  // one captured segmentation; owns the events its profiling nodes record
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    std::vector<ProfEv> evs;
    std::vector<cudaEvent_t> owned;
    int launches = 0;
    uint64_t used = 0;
  };
  static constexpr size_t GRAPH_CACHE = 4;  // e.g. the two buffer pairs of the host stream API
  std::vector<GraphEntry> gcache;
  uint64_t gclock = 0;
  bool capturing = false;
  std::vector<cudaEvent_t> cap_owned;
  // host stream API (rapid_segment_host_stream): second buffer pair, copy streams, events
  DevBuf himg2, hlab2;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t hev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  uint32_t *herr = nullptr;  // pinned: RECOUNT flags of the stream's segmentations
  // f4 quality workspace (rapid_quality)
  DevBuf qkeys, qcnt, qsize, qspb, qacc;
  bool use_tma = true;  // RAPID_NO_TMA=1 forces the LDG tile loader (A/B testing)
  // profiling
  int prof = 0;  // 0 off, 1 events, 2 events + window counting, 3 coarse events (phase set as one interval)
  int last_prof = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<ProfEv> evs;
  // debug
  int stop_kind = 0, stop_stage = 0, stop_sweep = 0, stop_phase = 0;
  int32_t *stop_map = nullptr;
  int stop_nbx = 0, stop_nby = 0;
  bool stopped = false;
};

namespace {

int fail(rapid_ctx *c, int code, const std::string &msg) {
  if (c) {
    c->err = msg;
    c->status = code;
  }
  return code;
}

int cuda_check(rapid_ctx *c, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return RAPID_OK;
  return fail(c, e == cudaErrorMemoryAllocation ? RAPID_E_OOM : RAPID_E_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
int dalloc(rapid_ctx *c, T **p, size_t n) {
  *p = nullptr;
  cudaError_t e = cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T));
  return cuda_check(c, e, "cudaMalloc");
}

int ensure(rapid_ctx *c, DevBuf &b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return RAPID_OK;
  if (b.p) {
    cudaDeviceSynchronize();
    cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
  }
  cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) return cuda_check(c, e, "cudaMalloc(workspace)");
  b.bytes = std::max<size_t>(bytes, 16);
  return RAPID_OK;
}

// ---- geometry (DESIGN §2 A10; PAPER RAPID l.1, l.6: P:124) ------------------------
// r*c = M with the squarest cells (ties: fewer rows), among factorisations that fit.
bool grid_rc(int H, int W, int M, int *r_out, int *c_out) {
  int br = 0, bc = 0;
  unsigned __int128 bmx = 0, bmn = 1;
  for (int r = 1; r <= M; r++) {
    if (M % r) continue;
    const int c = M / r;
    if (c > W || r > H) continue;
    const unsigned __int128 a = (unsigned __int128)W * r, b = (unsigned __int128)H * c;
    const unsigned __int128 mx = a > b ? a : b, mn = a > b ? b : a;
    if (br == 0 || mx * bmn < bmx * mn) {
      br = r;
      bc = c;
      bmx = mx;
      bmn = mn;
    }
  }
  if (!br) return false;
  *r_out = br;
  *c_out = bc;
  return true;
}

// sorted union of the dyadic cuts {k*b < len} and the cell cuts (both sorted) plus len
std::vector<int32_t> axis_cuts(int len, int b, const std::vector<int32_t> &cells) {
  std::vector<int32_t> out;
  out.reserve(len / b + cells.size() + 2);
  size_t j = 0;
  int64_t k = 0;
  while (true) {
    const int64_t d = k * b < len ? k * b : INT64_MAX;
    const int64_t cc = j < cells.size() ? cells[j] : INT64_MAX;
    const int64_t v = std::min(d, cc);
    if (v == INT64_MAX) break;
    if (out.empty() || out.back() != v) out.push_back((int32_t)v);
    if (d == v) k++;
    if (cc == v) j++;
  }
  if (out.back() != len) out.push_back(len);
  return out;
}

// index of each element of `fine` in its containing interval of `coarse`
std::vector<int32_t> parents(const std::vector<int32_t> &coarse, const std::vector<int32_t> &fine) {
  std::vector<int32_t> p(fine.size() - 1);
  size_t k = 0;
  for (size_t i = 0; i + 1 < fine.size(); i++) {
    while (!(coarse[k] <= fine[i] && fine[i] < coarse[k + 1])) k++;
    p[i] = (int32_t)k;
  }
  return p;
}

std::vector<int32_t> first_children(const std::vector<int32_t> &coarse, const std::vector<int32_t> &fine) {
  std::vector<int32_t> c(coarse.size());
  size_t k = 0;
  for (size_t i = 0; i < coarse.size(); i++) {
    while (fine[k] != coarse[i]) k++;
    c[i] = (int32_t)k;
  }
  return c;
}

size_t append(std::vector<int32_t> &tab, const std::vector<int32_t> &v) {
  size_t off = tab.size();
  tab.insert(tab.end(), v.begin(), v.end());
  while (tab.size() % 4) tab.push_back(0);  // 16-B alignment of every table
  return off;
}

int validate(rapid_ctx *c, int H, int W, const rapid_params *p) {
  if (!p || p->struct_size != sizeof(rapid_params)) return fail(c, RAPID_E_ARG, "params struct_size");
  if (H < 1 || W < 1 || H > 65535 || W > 65535) return fail(c, RAPID_E_RANGE, "H, W must be in [1, 65535]");
  if (p->batch < 1) return fail(c, RAPID_E_ARG, "batch < 1");
  if (p->n_superpixels < 1 || (uint64_t)p->n_superpixels > (uint64_t)H * W)
    return fail(c, RAPID_E_ARG, "n_superpixels out of range");
  if (p->n_stages < 1 || p->n_stages > RAPID_MAX_STAGES) return fail(c, RAPID_E_ARG, "n_stages");
  if (p->sweeps > RAPID_MAX_SWEEPS) return fail(c, RAPID_E_ARG, "sweeps");
  for (uint32_t s = 0; s < p->n_stages; s++) {
    const uint32_t b = p->block_size[s];
    if (b < 1 || b > 64) return fail(c, RAPID_E_ARG, "block_size must be in [1, 64]");
    if (s > 0 && (b >= p->block_size[s - 1] || p->block_size[s - 1] % b))
      return fail(c, RAPID_E_ARG, "block sizes must descend, each dividing the previous");
  }
  if (p->lambda_pos_q16 < 0 || p->lambda_pos_q16 >= (1ll << 31) || p->lambda_b_q16 < 0 ||
      p->lambda_b_q16 >= (1ll << 31))
    return fail(c, RAPID_E_RANGE, "lambda out of [0, 2^31)");
  if (p->size_mode > 2) return fail(c, RAPID_E_ARG, "size_mode");
  if (p->size_mode != RAPID_SIZE_NONE) {
    if (p->l_den == 0 || p->l_num >= p->l_den || p->l_den >= (1u << 31))
      return fail(c, RAPID_E_ARG, "l must be in [0, 1)");
    if (p->u_den == 0 || p->u_num <= p->u_den || p->u_num >= (1u << 31))
      return fail(c, RAPID_E_ARG, "u must be > 1");
  }
  if (p->mask_rule > 3) return fail(c, RAPID_E_ARG, "mask_rule");
  if (p->y_model > RAPID_Y_FEATURES) return fail(c, RAPID_E_ARG, "y_model");
  if (p->mask_rule != RAPID_MASK_OFF && p->y_model == RAPID_Y_PROTO &&
      (p->n_proto < 1 || p->n_proto > RAPID_MAX_PROTO))
    return fail(c, RAPID_E_ARG, "mask needs 1..4 prototypes");
  for (int k = 0; k < 5; k++)
    if (p->feat_w_q16[k] <= -(1ll << 31) || p->feat_w_q16[k] >= (1ll << 31))
      return fail(c, RAPID_E_RANGE, "feature weights out of (-2^31, 2^31)");
  if (p->tau2 < 0 || p->tau2 >= (1ll << 40)) return fail(c, RAPID_E_RANGE, "tau2 out of [0, 2^40)");
  if (p->stats_mode > RAPID_STATS_PYRAMID) return fail(c, RAPID_E_ARG, "stats_mode");
  const uint64_t px = (uint64_t)p->batch * H * W;
  if (px > c->cap_px) return fail(c, RAPID_E_CAPACITY, "B*H*W exceeds max_pixels_total");
  if (px >= (1ull << 32)) return fail(c, RAPID_E_RANGE, "B*H*W must be < 2^32");
  if ((uint64_t)p->batch * p->n_superpixels > c->cap_sp)
    return fail(c, RAPID_E_CAPACITY, "B*M exceeds max_superpixels_total");
  int r, cc;
  if (!grid_rc(H, W, (int)p->n_superpixels, &r, &cc)) return fail(c, RAPID_E_ARG, "no r x c = M grid fits the image");
  return RAPID_OK;
}

int build_plan(rapid_ctx *c, int H, int W, const rapid_params *p) {
  Plan &P = c->plan;
  const int B = (int)p->batch, M = (int)p->n_superpixels, nst = (int)p->n_stages;
  bool same = P.valid && P.B == B && P.H == H && P.W == W && P.M == M && P.nst == nst;
  for (int s = 0; same && s < nst; s++) same = P.bs[s] == (int)p->block_size[s];
  if (same) return RAPID_OK;
  Plan N;
  N.B = B; N.H = H; N.W = W; N.M = M; N.nst = nst;
  for (int s = 0; s < nst; s++) N.bs[s] = (int)p->block_size[s];
  grid_rc(H, W, M, &N.rows, &N.cols);
  N.X.resize(N.cols + 1);
  N.Y.resize(N.rows + 1);
  for (int i = 0; i <= N.cols; i++) N.X[i] = (int32_t)(((int64_t)i * W) / N.cols);
  for (int j = 0; j <= N.rows; j++) N.Y[j] = (int32_t)(((int64_t)j * H) / N.rows);
  for (int s = 0; s < nst; s++) {
    StagePlan &S = N.st[s];
    S.b = N.bs[s];
    S.xs = axis_cuts(W, S.b, N.X);
    S.ys = axis_cuts(H, S.b, N.Y);
    S.nbx = (int)S.xs.size() - 1;
    S.nby = (int)S.ys.size() - 1;
    S.tiles_x = (S.nbx + TX - 1) / TX;
    S.tiles_y = (S.nby + TY - 1) / TY;
    int64_t mw = 0, mh = 0;
    for (int i = 0; i < S.nbx; i++) mw = std::max<int64_t>(mw, S.xs[i + 1] - S.xs[i]);
    for (int j = 0; j < S.nby; j++) mh = std::max<int64_t>(mh, S.ys[j + 1] - S.ys[j]);
    S.smallb = !c->no_smallb && S.b > 1 && mw * mh * (int64_t)(std::max(H, W) - 1) < (int64_t(1) << 22);
    // K5's packed deltas: in one phase a superpixel S loses at most n_S pixels and gains at most
    // 4 n_S R (every incoming block is a 4-neighbour of one of S's blocks, which do not move in
    // the phase; R = largest / smallest block area), so each field of its phase total stays below
    // 4 R n_S max(255, W - 1, H - 1) in magnitude: int32 while n_S <= maxn_lim
    int64_t nw = INT64_MAX, nh = INT64_MAX;
    for (int i = 0; i < S.nbx; i++) nw = std::min<int64_t>(nw, S.xs[i + 1] - S.xs[i]);
    for (int j = 0; j < S.nby; j++) nh = std::min<int64_t>(nh, S.ys[j + 1] - S.ys[j]);
    const int64_t R = (mw * mh + nw * nh - 1) / (nw * nh);
    const int64_t vmax = std::max<int64_t>(255, std::max(H, W) - 1);
    S.maxn_lim = (int32_t)std::min<int64_t>(INT32_MAX, (int64_t)INT32_MAX / (4 * R * vmax));
  }
  for (int s = 0; s < nst; s++) {
    StagePlan &S = N.st[s];
    if (s > 0) {
      S.px = parents(N.st[s - 1].xs, S.xs);
      S.py = parents(N.st[s - 1].ys, S.ys);
    }
    if (s + 1 < nst) {
      S.cxs = first_children(S.xs, N.st[s + 1].xs);
      S.cys = first_children(S.ys, N.st[s + 1].ys);
    }
  }
  // stage-0 block -> cell, last stage pixel -> block
  {
    const StagePlan &S0 = N.st[0];
    N.cellx = parents(N.X, S0.xs);
    N.celly = parents(N.Y, S0.ys);
    const StagePlan &SL = N.st[nst - 1];
    std::vector<int32_t> px(W + 1), py(H + 1);
    for (int x = 0; x <= W; x++) px[x] = x;
    for (int y = 0; y <= H; y++) py[y] = y;
    N.bxp = parents(SL.xs, px);
    N.byp = parents(SL.ys, py);
    N.b0x = parents(S0.xs, px);  // pixel -> stage-0 block (f2 features)
    N.b0y = parents(S0.ys, py);
  }
  N.o_X = append(N.tab, N.X);
  N.o_Y = append(N.tab, N.Y);
  N.o_cellx = append(N.tab, N.cellx);
  N.o_celly = append(N.tab, N.celly);
  N.o_bxp = append(N.tab, N.bxp);
  N.o_byp = append(N.tab, N.byp);
  N.o_b0x = append(N.tab, N.b0x);
  N.o_b0y = append(N.tab, N.b0y);
  for (int s = 0; s < nst; s++) {
    StagePlan &S = N.st[s];
    S.o_xs = append(N.tab, S.xs);
    S.o_ys = append(N.tab, S.ys);
    S.o_px = append(N.tab, S.px);
    S.o_py = append(N.tab, S.py);
    S.o_cxs = append(N.tab, S.cxs);
    S.o_cys = append(N.tab, S.cys);
    const size_t nb = (size_t)S.nbx * S.nby * B;
    if (S.b > 1) {
      S.bsum_off = N.bsum_total;
      N.bsum_total += (nb + 1) & ~(size_t)1;
      N.map_max = std::max(N.map_max, nb);
    }
    N.props_max = std::max(N.props_max, (size_t)((S.nbx + 1) / 2) * ((S.nby + 1) / 2) * B);
    N.tiles_max = std::max(N.tiles_max, (size_t)S.tiles_x * S.tiles_y * B);
  }
  int rc;
  if ((rc = ensure(c, c->tab, N.tab.size() * 4))) return rc;
  if ((rc = ensure(c, c->bsum, N.bsum_total * 8))) return rc;
  if ((rc = ensure(c, c->maps[0], N.map_max * 4))) return rc;
  if ((rc = ensure(c, c->maps[1], N.map_max * 4))) return rc;
  // proposals: bounded by the phase's blocks, plus the chunked-reservation slack of K4b warps
  if ((rc = ensure(c, c->props, (N.props_max + (size_t)std::max(c->eval_grid, c->sweep_grid) * 8 * CAND_SLACK_PER_WARP) * 16)))
    return rc;
  // candidate list: every block of a phase colour may be a candidate, plus the chunked
  // reservation slack of every scanning warp
  const size_t cand_max = N.props_max + (size_t)c->scan_grid * 8 * CAND_SLACK_PER_WARP;
  if ((rc = ensure(c, c->cands, cand_max * 32))) return rc;
  if ((rc = ensure(c, c->work, N.tiles_max * 4))) return rc;
  if ((rc = ensure(c, c->bset, N.tiles_max * 32 * 4))) return rc;  // 1 bit per block
  if ((rc = ensure(c, c->vtile, N.tiles_max))) return rc;           // victim-tile marks (stage stamps)
  cudaError_t e = cudaMemcpy(c->tab.p, N.tab.data(), N.tab.size() * 4, cudaMemcpyHostToDevice);
  if ((rc = cuda_check(c, e, "upload tables"))) return rc;
  N.valid = true;
  c->plan = std::move(N);
  c->plan_gen++;  // buffers may have moved: a captured graph is stale
  return RAPID_OK;
}

StageDev stage_dev(rapid_ctx *c, int s, int32_t *labels_out) {
  const Plan &P = c->plan;
  const StagePlan &S = P.st[s];
  const int32_t *T = (const int32_t *)c->tab.p;
  StageDev d;
  d.nbx = S.nbx;
  d.nby = S.nby;
  d.b = S.b;
  d.tiles_x = S.tiles_x;
  d.tiles_y = S.tiles_y;
  d.uniform = 1;
  for (size_t i = 0; i < S.xs.size() && d.uniform; i++) d.uniform = S.xs[i] == (int32_t)(i * S.b);
  for (size_t j = 0; j < S.ys.size() && d.uniform; j++) d.uniform = S.ys[j] == (int32_t)(j * S.b);
  d.bsum32 = (S.b == 2 && d.uniform) ? 1 : 0;  // 2x2 sums fit 10 bits per channel
  d.fd_tx = make_fastdiv((uint32_t)S.tiles_x);
  d.fd_ty = make_fastdiv((uint32_t)S.tiles_y);
  d.fd_nbx = make_fastdivu((uint32_t)S.nbx);
  d.fd_nper = make_fastdivu((uint32_t)((size_t)S.nbx * S.nby));
  d.xs = T + S.o_xs;
  d.ys = T + S.o_ys;
  d.px = T + S.o_px;
  d.py = T + S.o_py;
  d.cxs = T + S.o_cxs;
  d.cys = T + S.o_cys;
  d.bsum = S.b > 1 ? (const uint64_t *)c->bsum.p + S.bsum_off : nullptr;
  d.map = S.b == 1 ? labels_out : (int32_t *)c->maps[s & 1].p;
  return d;
}

SpDev sp_dev(rapid_ctx *c) {
  SpDev d;
  d.sums = c->sums;
  d.rec = c->rec;
  d.init = c->init;
  d.alive = c->alive;
  d.active = c->active;
  d.y = c->y;
  d.victim = c->victim;
  d.out = c->out;
  d.dirty = c->dirty;
  d.remap = c->remap;
  d.dsum = c->dsum;
  d.big = &c->ctl->big;
  d.nlim = 0;  // set per call from the plan (enqueue)
  return d;
}

struct Timer {  // CUDA events around a launch group (profiling mode only)
  rapid_ctx *c;
  cudaStream_t s;
  int cls, stage;
  cudaEvent_t a = nullptr;
  // level 3 (coarse): no events between the kernels of the phase loop — only the stage's whole
  // phase set (RAPID_K_PHASESET) and the kernel classes outside the loop are bracketed
  bool on() const {
    if (!c->prof) return false;
    return c->prof != 3 || !(cls == RAPID_K_SNAPSHOT || cls == RAPID_K_PROPOSE || cls == RAPID_K_COMMIT || cls == RAPID_K_EVAL);
  }
  Timer(rapid_ctx *c_, cudaStream_t s_, int cls_, int stage_) : c(c_), s(s_), cls(cls_), stage(stage_) {
    if (!on()) return;
    a = next();
    record(a);
  }
  void record(cudaEvent_t e) {  // inside a captured graph: an external (real, timeable) record
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  }
  cudaEvent_t next() {
    if (c->capturing) {  // events of a captured graph belong to its cache entry
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->cap_owned.push_back(e);
      return e;
    }
    if (c->ev_used == c->ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
  }
  ~Timer() {
    if (!on()) return;
    cudaEvent_t b = next();
    record(b);
    c->evs.push_back({cls, stage, a, b});
  }
};

int enqueue(rapid_ctx *c, const uint8_t *image, int H, int W, const rapid_params *p,
            int32_t *labels, cudaStream_t s) {
  const Plan &P = c->plan;
  const int B = P.B, M = P.M, nst = P.nst, K = B * M;
  const int sweeps = (int)p->sweeps;
  const int gated_sz = p->size_mode != RAPID_SIZE_NONE;
  const bool fused_snap = gated_sz && c->fuse_snap;  // K3 folded into the previous K5
  const int grid_k = c->sm_count * 4;
  const int grid_snap = c->sm_count * c->snap_ctas;  // K3 (RAPID_SNAP_CTAS per SM)
  Ctl *ctl = c->ctl;
  c->launches = 0;
  c->evs.clear();
  c->ev_used = 0;
  c->stopped = false;
  c->stop_map = nullptr;
  cudaMemsetAsync(ctl, 0, sizeof(Ctl), s);
  // the dirty byte map starts empty every call (a captured graph replays)
  cudaMemsetAsync(c->dirty, 0, (size_t)K + 4, s);
  // K5's packed deltas start (and end every phase) folded: cleared per call so that a call
  // stopped at a debug point cannot leak into the next
  if (c->packed) cudaMemsetAsync(c->dsum, 0, (size_t)K * 32, s);
  cudaMemsetAsync(c->vtile.p, 0, c->vtile.bytes, s);  // victim-tile marks (stamped per stage)

  StageDev sd[MAXS];
  struct alignas(64) TMap {
    unsigned char b[128];  // CUtensorMap
  };
  TMap tmaps[MAXS];
  bool has_tmap[MAXS];
  for (int st = 0; st < nst; st++) {
    sd[st] = stage_dev(c, st, labels);
    has_tmap[st] = c->use_tma && make_label_tmap(tmaps[st].b, sd[st].map, sd[st].nbx, sd[st].nby, B);
  }
  SpDev sp = sp_dev(c);
  {  // K5's packed deltas: the call's size limit is the smallest stage limit (0 / null: off)
    int lim = INT32_MAX;
    for (int st = 0; st < (int)P.nst; st++) lim = std::min(lim, (int)P.st[st].maxn_lim);
    if (c->packed_lim > 0) lim = std::min(lim, c->packed_lim);
    sp.nlim = lim;
    // measured crossover: the fold in K3 costs about what the halved REDs save in K5 below a few
    // hundred Mpx per call (configs 2, 3, 5: packed 2.78 / 4.14 vs direct 2.67 / 4.13 ms), while
    // config 4 (1.07 Gpx) gains 0.16 ms; RAPID_PACKED=1 forces packing at any size
    const bool big_call = (uint64_t)P.B * (uint64_t)P.H * (uint64_t)P.W >= (1ull << 28);
    if (!c->packed || lim <= 0 || (!big_call && !c->packed_force)) sp.dsum = nullptr;
  }
  const int32_t *T = (const int32_t *)c->tab.p;

  InitArgs ia;
  ia.st0 = sd[0];
  ia.sp = sp;
  ia.image = image;
  ia.H = H; ia.W = W; ia.B = B; ia.M = M; ia.K = K;
  ia.rows = P.rows; ia.cols = P.cols;
  ia.X = T + P.o_X; ia.Y = T + P.o_Y;
  ia.cellx = T + P.o_cellx; ia.celly = T + P.o_celly;
  {
    Timer tm(c, s, RAPID_K_PYRAMID, 0);
    launch_init_sp(ia, s);
    int leaf = -1;
    for (int st = 0; st < nst; st++)
      if (P.st[st].b > 1) leaf = st;
    if (leaf >= 0) {
      int top = leaf;  // coarsest level written by the leaf kernel
      const bool literal = p->stats_mode == RAPID_STATS_PYRAMID;
      if (leaf >= 1 && launch_pyramid_leaf24(sd[leaf], sd[leaf - 1], image, H, W, B,
                                             (uint64_t *)c->bsum.p + P.st[leaf].bsum_off,
                                             (uint64_t *)c->bsum.p + P.st[leaf - 1].bsum_off, literal, s))
        top = leaf - 1;
      else
        launch_pyramid_leaf(sd[leaf], image, H, W, B, (uint64_t *)c->bsum.p + P.st[leaf].bsum_off, literal, s);
      c->launches++;
      for (int st = top - 1; st >= 0; st--) {
        launch_pyramid_up(sd[st], sd[st + 1], B, (uint64_t *)c->bsum.p + P.st[st].bsum_off, literal, s);
        c->launches++;
      }
    }
    launch_init_map0(ia, s);
    launch_stats0(ia, s);
    c->launches += 3;
  }

  const int mask = (int)p->mask_rule;
  const bool tile_gate = (mask == RAPID_MASK_CLASS || mask == RAPID_MASK_BSP);
  int g = 0;  // global phase index within this call
  auto stop_at = [&](int kind, int st, int t, int ph) {
    if (c->stop_kind != kind || c->stop_stage != st) return false;
    if (kind == RAPID_STOP_PHASE && (c->stop_sweep != t || c->stop_phase != ph)) return false;
    c->stopped = true;
    c->stop_map = sd[st].map;
    c->stop_nbx = sd[st].nbx;
    c->stop_nby = sd[st].nby;
    return true;
  };
  auto remap_in_place = [&](int st) {  // debug stops only: make the stage map current
    FinalArgs fa;
    fa.last = sd[st];
    fa.sp = sp;
    fa.B = B; fa.H = sd[st].nby; fa.W = sd[st].nbx; fa.M = M;
    fa.bxp = nullptr; fa.byp = nullptr;
    fa.remap_pending = &ctl->remap_pending[st];
    fa.labels = sd[st].map;
    fa.worklist = nullptr;
    fa.nwork = nullptr;
    launch_final(fa, false, s);
  };

  for (int st = 0; st < nst; st++) {
    const bool pixel = P.st[st].b == 1;
    const bool use_work = st > 0 && tile_gate;
    const int gating = (st > 0 && mask != RAPID_MASK_OFF) ? (mask == RAPID_MASK_EQ7 ? 2 : 1) : 0;
    bool bset_done = false;
    if (st > 0) {
      Timer tm(c, s, RAPID_K_TRANSITION, st);
      TransArgs ta;
      ta.prev = sd[st - 1];
      ta.next = sd[st];
      ta.sp = sp;
      ta.B = B; ta.M = M;
      ta.remap_pending = &ctl->remap_pending[st - 1];
      ta.gate = use_work ? 1 : 0;
      ta.worklist = (int32_t *)c->work.p;
      ta.nwork = &ctl->nwork[st];
      ta.bset = (c->use_bset && c->fuse_bset) ? (uint32_t *)c->bset.p : nullptr;
      ta.gating = gating;
      bset_done = launch_transition(ta, s);
      if (!bset_done && c->use_bset && c->bset_parent) {  // boundary sets from the parent map
        ta.bset = (uint32_t *)c->bset.p;
        bset_done = launch_bset_dyadic(ta, c->sm_count, s);
        if (bset_done) c->launches++;
      }
      c->launches++;
      if (p->stats_mode == RAPID_STATS_RECOUNT) {
        RecountArgs ra;
        ra.st = sd[st];
        ra.sp = sp;
        ra.image = image;
        ra.H = H; ra.W = W; ra.B = B; ra.M = M; ra.K = K;
        ra.rc = c->rc;
        ra.err = &ctl->err;
        launch_recount(ra, pixel, grid_k, s, &c->launches);
      }
    }
    if (c->use_bset && !bset_done) {  // boundary sets of the stage (maintained by the commits from here on)
      Timer tm(c, s, RAPID_K_TRANSITION, st);
      PhaseArgs ba{};
      ba.st = sd[st];
      ba.sp = sp;
      ba.B = B; ba.M = M;
      ba.gating = gating;
      ba.worklist = use_work ? (const int32_t *)c->work.p : nullptr;
      ba.nwork = &ctl->nwork[st];
      ba.bset = (uint32_t *)c->bset.p;
      launch_bset_build(ba, has_tmap[st] ? tmaps[st].b : nullptr, has_tmap[st] ? c->tiles_grid : c->sm_count * 8, s);
      c->launches++;
    }
    if (c->prof == 2 && use_work) {  // profiling only: algorithmic window of the gated stage
      launch_count_window(sd[st], sp, B, M, &ctl->stage_info[st][2], s);
      c->launches++;
    }
    if (stop_at(RAPID_STOP_STAGE_START, st, 0, 0)) return RAPID_OK;
    {
      Timer tm(c, s, RAPID_K_PHASESET, st);
      {
        Timer t2(c, s, RAPID_K_SNAPSHOT, st);
        // full refresh at stage 0, after prediction (every flag changed) and whenever the stats
        // are re-derived (RECOUNT / PYRAMID); otherwise only the previous merge round changed
        // records since the last snapshot, and it marked its victims and targets dirty
        const bool full = st == 0 || (st == 1 && mask != RAPID_MASK_OFF) || p->stats_mode != RAPID_STATS_REUSE;
        SnapArgs sa{sp, K, full ? 0u : 1u, (long long)p->l_num, gated_sz ? (long long)p->l_den : 0ll};
        sa.full_flags = true;
        launch_snapshot(sa, grid_snap, s);
        c->launches++;
      }
      for (int t = 0; t < sweeps; t++) {
        for (int ph = 0; ph < 4; ph++, g++) {
          if (!(t == 0 && ph == 0) && !fused_snap) {  // (fused: the previous commit refreshed them)
            Timer t2(c, s, RAPID_K_SNAPSHOT, st);
            SnapArgs sa{sp, K, c->stamp_base + (uint32_t)(g - 1), (long long)p->l_num, gated_sz ? (long long)p->l_den : 0ll};
            launch_snapshot(sa, grid_snap, s);
            c->launches++;
          }
          PhaseArgs pa;
          pa.st = sd[st];
          pa.sp = sp;
          pa.image = image;
          pa.H = H; pa.W = W; pa.B = B; pa.M = M;
          pa.cx = ph & 1;
          pa.cy = ph >> 1;
          pa.gating = gating;
          pa.bset = c->use_bset ? (uint32_t *)c->bset.p : nullptr;
          pa.wq = &ctl->wq[g];
          pa.list = (uint32_t *)c->cands.p;  // (the full-scan path's buffer; at least the phase's blocks)
          pa.list_count = &ctl->list_count[g];
          pa.gpw = c->sweep_gpw;
          pa.tail_pct = pixel ? 0 : c->sweep_tail;  // measured: helps the latency-bound block stages only
          pa.size_mode = (int)p->size_mode;
          pa.l_num = p->l_num; pa.l_den = p->l_den;
          pa.lam_pos = p->lambda_pos_q16;
          pa.lam_b = p->lambda_b_q16;
          pa.worklist = use_work ? (const int32_t *)c->work.p : nullptr;
          pa.nwork = &ctl->nwork[st];
          pa.props = (uint4 *)c->props.p;
          pa.cands = (uint4 *)c->cands.p;
          pa.cand_count = &ctl->cand_count[g];
          pa.prop_count = &ctl->prop_count[g];
          pa.stamp = c->stamp_base + (uint32_t)g;
          pa.cnt = &ctl->cnt[st][t][ph][0];
          pa.prev = t > 0 ? &ctl->cnt[st][t - 1][0][0] : nullptr;
          pa.victim_any = &ctl->victim_any[st];
          if (c->use_bset) {
            Timer t2(c, s, RAPID_K_PROPOSE, st);
            const bool list = c->sweep_list_minb > 0 && P.st[st].b >= c->sweep_list_minb;
            launch_sweep(pa, pixel, P.st[st].smallb, list, c->sm_count, s);
            c->launches += list && !pixel ? 2 : 1;
          } else {
            {
              Timer t2(c, s, RAPID_K_PROPOSE, st);
              launch_scan(pa, has_tmap[st] ? tmaps[st].b : nullptr, c->scan_grid, s);
              c->launches++;
            }
            {
              Timer t2(c, s, RAPID_K_EVAL, st);
              launch_eval(pa, pixel, c->eval_grid, s);
              c->launches++;
            }
          }
          if (gated_sz) {
            Timer t2(c, s, RAPID_K_COMMIT, st);
            if (fused_snap) {
              const cudaError_t e = launch_commit_snap(pa, pixel, c->sm_count, s);
              if (e != cudaSuccess) return fail(c, RAPID_E_CUDA, std::string("cooperative launch k_commit<SNAP>: ") + cudaGetErrorString(e));
            } else {
              launch_commit(pa, pixel, c->sm_count * 8, s);  // latency-bound gathers: full occupancy
            }
            c->launches++;
          }
          if (stop_at(RAPID_STOP_PHASE, st, t, ph)) {
            if (gated_sz && !fused_snap) {  // fold K5's packed deltas: the stats read at the stop are whole
              SnapArgs sa{sp, K, c->stamp_base + (uint32_t)g, (long long)p->l_num, (long long)p->l_den};
              launch_snapshot(sa, grid_snap, s);
            }
            return RAPID_OK;
          }
        }
      }
    }
    {  // snapshot of the last phase's changes (merge round / prediction read it)
      Timer t2(c, s, RAPID_K_SNAPSHOT, st);
      if (g > 0 && !fused_snap) {
        SnapArgs sa{sp, K, c->stamp_base + (uint32_t)(g - 1), (long long)p->l_num, gated_sz ? (long long)p->l_den : 0ll};
        launch_snapshot(sa, grid_snap, s);
        c->launches++;
      }
    }
    if (p->size_mode == RAPID_SIZE_MERGE) {
      Timer tm(c, s, RAPID_K_MERGE, st);
      MergeArgs ma;
      ma.st = sd[st];
      ma.sp = sp;
      ma.B = B; ma.M = M; ma.K = K;
      ma.lam_pos = p->lambda_pos_q16;
      ma.lam_b = p->lambda_b_q16;
      ma.u_num = p->u_num; ma.u_den = p->u_den;
      ma.victim_any = &ctl->victim_any[st];
      ma.remap_pending = &ctl->remap_pending[st];
      ma.chunk = c->chunk;
      ma.total = &ctl->vtotal;
      ma.vlist = c->vlist;
      ma.hkeys = c->hkeys;
      ma.hvals = c->hvals;
      ma.hnext = c->hnext;
      ma.head = c->head;
      ma.hmask = c->hcap - 1;
      ma.worklist = use_work ? (const int32_t *)c->work.p : nullptr;
      ma.nwork = &ctl->nwork[st];
      ma.deg = c->deg;
      ma.deg_total = &ctl->deg_total;
      ma.candT = c->candT;
      ma.candV = c->candV;
      ma.mlock = c->mlock;
      ma.res = c->res;
      ma.candE = c->candE;
      ma.pairs = c->pairs;
      ma.npairs = &ctl->npairs;
      ma.flag = ctl->mflag;
      ma.bset = c->use_bset ? (const uint32_t *)c->bset.p : nullptr;
      ma.vtile = (uint8_t *)c->vtile.p;
      ma.vstamp = (uint8_t)(st + 1);
      ma.stage_info = &ctl->stage_info[st][0];
      const cudaError_t me = launch_merge_round(ma, has_tmap[st] ? tmaps[st].b : nullptr, c->tiles_grid, grid_k, s, &c->launches);
      if (me != cudaSuccess) return fail(c, RAPID_E_CUDA, std::string("cooperative launch k_merge_match: ") + cudaGetErrorString(me));
    }
    if (stop_at(RAPID_STOP_AFTER_MERGE, st, 0, 0)) {
      remap_in_place(st);
      return RAPID_OK;
    }
    if (st == 0 && mask != RAPID_MASK_OFF) {
      Timer tm(c, s, RAPID_K_PREDICT, st);
      SnapArgs sa{sp, K, 0u, (long long)p->l_num, gated_sz ? (long long)p->l_den : 0ll};
      launch_snapshot(sa, grid_snap, s);
      c->launches++;
      PredictArgs pr;
      pr.st = sd[st];
      pr.sp = sp;
      pr.B = B; pr.M = M; pr.K = K;
      pr.mask_rule = mask;
      pr.n_proto = (int)p->n_proto;
      for (int k = 0; k < 4; k++)
        for (int ch = 0; ch < 3; ch++) pr.proto[k][ch] = p->proto_rgb[k][ch];
      pr.tau2 = p->tau2;
      pr.remap_pending = &ctl->remap_pending[st];
      pr.chunk = c->chunk;
      pr.total = &ctl->atotal;
      pr.alist = c->alist;
      pr.y_model = (int)p->y_model;
      for (int k = 0; k < 5; k++) pr.feat_w[k] = p->feat_w_q16[k];
      pr.image = image;
      pr.H = H; pr.W = W;
      pr.b0x = T + P.o_b0x;
      pr.b0y = T + P.o_b0y;
      pr.scratch = c->rc;
      pr.hkeys = c->hkeys;
      pr.hmask = c->hcap - 1;
      launch_predict(pr, grid_k, s, &c->launches);
      if (stop_at(RAPID_STOP_AFTER_PREDICT, st, 0, 0)) {
        remap_in_place(st);
        return RAPID_OK;
      }
    }
  }
  {
    Timer tm(c, s, RAPID_K_FINAL, nst - 1);
    FinalArgs fa;
    fa.last = sd[nst - 1];
    fa.sp = sp;
    fa.B = B; fa.H = H; fa.W = W; fa.M = M;
    fa.bxp = T + P.o_bxp;
    fa.byp = T + P.o_byp;
    fa.remap_pending = &ctl->remap_pending[nst - 1];
    fa.labels = labels;
    const bool last_work = nst > 1 && tile_gate;
    fa.worklist = last_work ? (const int32_t *)c->work.p : nullptr;
    fa.nwork = &ctl->nwork[nst - 1];
    if (last_work && c->use_bset && g_adj_tma == 0 && p->size_mode == RAPID_SIZE_MERGE) {
      fa.vtile = (const uint8_t *)c->vtile.p;  // marked by the last stage's adjacency pass
      fa.vstamp = (uint8_t)nst;
    }
    launch_final(fa, P.st[nst - 1].b > 1, s);
    c->launches++;
  }
  return RAPID_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char *rapid_status_string(int st) {
  switch (st) {
    case RAPID_OK: return "ok";
    case RAPID_E_ARG: return "invalid argument";
    case RAPID_E_CAPACITY: return "capacity exceeded";
    case RAPID_E_RANGE: return "value out of the exact-arithmetic range";
    case RAPID_E_CUDA: return "CUDA error";
    case RAPID_E_OOM: return "out of device memory";
    case RAPID_E_INTEGRITY: return "RECOUNT integrity check failed";
    case RAPID_E_STATE: return "no segmentation has run";
    default: return "unknown status";
  }
}

const char *rapid_last_error(const rapid_ctx *c) { return c ? c->err.c_str() : "null ctx"; }

void rapid_free(rapid_ctx *c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto &g : c->gcache) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    for (cudaEvent_t e : g.owned) cudaEventDestroy(e);
  }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  for (cudaEvent_t e : c->hev)
    if (e) cudaEventDestroy(e);
  if (c->herr) cudaFreeHost(c->herr);
  for (DevBuf *b : {&c->himg2, &c->hlab2, &c->qkeys, &c->qcnt, &c->qsize, &c->qspb, &c->qacc})
    if (b->p) cudaFree(b->p);
  void *ptrs[] = {c->sums, c->rc, c->dsum, c->rec, c->init, c->out, c->remap, c->head,
                  c->vlist, c->alist, c->pairs, c->alive, c->active, c->victim, c->y, c->dirty,
                  c->deg, c->chunk, c->hkeys, c->candE, c->hvals, c->hnext, c->candT, c->ctl,
                  c->candV, c->mlock, c->res,
                  c->tab.p, c->bsum.p, c->maps[0].p, c->maps[1].p, c->props.p, c->work.p, c->cands.p, c->bset.p, c->vtile.p,
                  c->himg.p, c->hlab.p};
  for (void *q : ptrs)
    if (q) cudaFree(q);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
  cudaSetDevice(prev);
}

int rapid_init(rapid_ctx **out, int device, uint64_t max_pixels_total, uint64_t max_superpixels_total) {
  if (!out) return RAPID_E_ARG;
  *out = nullptr;
  if (max_pixels_total < 1 || max_superpixels_total < 1 || max_superpixels_total >= (1ull << 31) ||
      max_pixels_total >= (1ull << 32))
    return RAPID_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return RAPID_E_CUDA;
  rapid_ctx *c = new rapid_ctx();
  c->device = device;
  c->cap_px = max_pixels_total;
  c->cap_sp = max_superpixels_total;
  int rc = cuda_check(c, cudaSetDevice(device), "cudaSetDevice");
  if (rc) { delete c; return rc; }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  const size_t K = max_superpixels_total;
  size_t hc = 1024;
  while (hc < 12 * K + 1024) hc <<= 1;  // planar adjacency: <= 3K unordered pairs, 2 directions
  c->hcap = hc;
  if ((rc = dalloc(c, &c->sums, K * SUMW)) || (rc = dalloc(c, &c->rc, K * SUMW)) ||
      (rc = dalloc(c, &c->rec, K)) || (rc = dalloc(c, &c->init, K)) || (rc = dalloc(c, &c->out, K)) ||
      (rc = dalloc(c, &c->remap, K)) ||
      (rc = dalloc(c, &c->head, K)) || (rc = dalloc(c, &c->vlist, K)) || (rc = dalloc(c, &c->alist, K)) ||
      (rc = dalloc(c, &c->pairs, 2 * K)) || (rc = dalloc(c, &c->alive, K)) ||
      (rc = dalloc(c, &c->active, K)) || (rc = dalloc(c, &c->victim, K)) || (rc = dalloc(c, &c->y, K)) ||
      (rc = dalloc(c, &c->dirty, K + 4)) || (rc = dalloc(c, &c->deg, K + 1)) ||
      (rc = dalloc(c, &c->chunk, K / 1024 + 2)) || (rc = dalloc(c, &c->hkeys, hc)) ||
      (rc = dalloc(c, &c->hvals, hc)) || (rc = dalloc(c, &c->hnext, hc)) ||
      (rc = dalloc(c, &c->candT, hc)) || (rc = dalloc(c, &c->candE, 2 * hc)) ||
      (rc = dalloc(c, &c->candV, hc)) || (rc = dalloc(c, &c->mlock, K)) || (rc = dalloc(c, &c->res, K)) ||
      (rc = dalloc(c, &c->ctl, 1)) || (rc = dalloc(c, &c->dsum, K * 4))) {
    rapid_free(c);
    return rc;
  }
  cudaMemset(c->hkeys, 0xff, hc * 8);
  cudaMemset(c->hvals, 0, hc * 4);
  cudaMemset(c->dirty, 0, K * 4);
  cudaMemset(c->mlock, 0, K * 4);
  cudaMemset(c->res, 0xff, K * 4);
  cudaMemset(c->rc, 0, K * SUMW * 8);
  c->scan_grid = c->sm_count * scan_occupancy();
  c->eval_grid = c->sm_count * eval_occupancy();
  c->sweep_grid = c->sm_count * sweep_occupancy();
  if (const char *e = getenv("RAPID_SWEEP_GPW")) c->sweep_gpw = std::max(1, atoi(e));
  if (const char *e = getenv("RAPID_SWEEP_LIST")) c->sweep_list_minb = std::max(0, atoi(e));
  if (const char *e = getenv("RAPID_PACKED")) {
    c->packed = e[0] != '0';
    c->packed_force = e[0] == '1';
  }
  if (const char *e = getenv("RAPID_SNAP_CTAS")) c->snap_ctas = std::min(8, std::max(1, atoi(e)));
  if (const char *e = getenv("RAPID_PACKED_LIM")) c->packed_lim = std::max(0, atoi(e));
  if (const char *e = getenv("RAPID_SWEEP_TAIL")) c->sweep_tail = std::min(100, std::max(0, atoi(e)));
  if (const char *e = getenv("RAPID_FUSE_BSET")) c->fuse_bset = e[0] == '1';
  if (const char *e = getenv("RAPID_BSET_PARENT")) c->bset_parent = e[0] != '0';
  if (const char *e = getenv("RAPID_FUSE_SNAP")) c->fuse_snap = e[0] == '1';
  if (const char *e = getenv("RAPID_SWEEP_NO_SMALLB")) c->no_smallb = e[0] == '1';
  if (const char *e = getenv("RAPID_PDL")) g_pdl = e[0] == '1';
  if (const char *e = getenv("RAPID_SWEEP_UNI")) g_sweep_uni = e[0] != '0';
  if (const char *e = getenv("RAPID_ADJ_MINB8")) g_adj_minb8 = e[0] == '1';
  if (const char *e = getenv("RAPID_ADJ_ILP")) g_adj_ilp = atoi(e) >= 4 ? 4 : atoi(e) >= 2 ? 2 : 1;
  if (const char *e = getenv("RAPID_ADJ")) g_adj_tma = strcmp(e, "tma") == 0 ? 1 : 0;
  if (const char *e = getenv("RAPID_BSET_ROWS")) g_bset_rows = e[0] == '0' ? 0 : e[0] == '2' ? 2 : 1;
  c->tiles_grid = c->sm_count * tiles_occupancy();
  {
    const char *e = getenv("RAPID_SWEEP");
    c->use_bset = !(e && strcmp(e, "scan") == 0);
  }
  {
    const char *e = getenv("RAPID_NO_TMA");
    c->use_tma = !(e && e[0] == '1');
  }
  {
    const char *e = getenv("RAPID_NO_GRAPH");
    c->use_graph = !(e && e[0] == '1');
    e = getenv("RAPID_L2_PERSIST");
    c->l2_persist = e && e[0] == '1';
  }
  rc = cuda_check(c, cudaDeviceSynchronize(), "rapid_init");
  if (rc) {
    rapid_free(c);
    return rc;
  }
  *out = c;
  return RAPID_OK;
}

int rapid_segment(rapid_ctx *c, const uint8_t *image, int32_t H, int32_t W, const rapid_params *p,
                  int32_t *labels_out, void *stream) {
  if (!c) return RAPID_E_ARG;
  c->status = RAPID_OK;
  c->err.clear();
  if (!image || !labels_out) return fail(c, RAPID_E_ARG, "null image or labels");
  int rc = validate(c, H, W, p);
  if (rc) return rc;
  cudaSetDevice(c->device);
  if ((rc = build_plan(c, H, W, p))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  cudaGetLastError();
  if (c->use_graph && c->stop_kind == 0) {
    rapid_ctx::GraphKey k;
    memset(&k, 0, sizeof k);
    k.image = image;
    k.labels = labels_out;
    k.H = H;
    k.W = W;
    k.prof = c->prof;
    k.plan_gen = c->plan_gen;
    k.p = *p;
    memset(k.p.pad0_, 0, sizeof k.p.pad0_);  // the explicit padding never selects a graph
    memset(k.p.pad_, 0, sizeof k.p.pad_);
    rapid_ctx::GraphEntry *ent = nullptr;
    for (auto &g : c->gcache)
      if (memcmp(&k, &g.key, sizeof k) == 0) ent = &g;
    if (!ent) {
      if (c->gcache.size() == rapid_ctx::GRAPH_CACHE) {  // evict the least recently used
        auto old = std::min_element(c->gcache.begin(), c->gcache.end(),
                                    [](const rapid_ctx::GraphEntry &x, const rapid_ctx::GraphEntry &y) {
                                      return x.used < y.used;
                                    });
        cudaStreamSynchronize(c->last_stream);
        cudaDeviceSynchronize();
        if (old->exec) cudaGraphExecDestroy(old->exec);
        for (cudaEvent_t e : old->owned) cudaEventDestroy(e);
        c->gcache.erase(old);
      }
      if (!c->cap_stream) {
        if ((rc = cuda_check(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking), "capture stream")))
          return rc;
        if (c->l2_persist) {  // keep the per-superpixel sums (atomic targets) resident in L2
          int max_persist = 0, max_win = 0;
          cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
          cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
          const size_t bytes = std::min<size_t>((size_t)c->cap_sp * SUMW * 8, (size_t)max_win);
          if (max_persist > 0 && bytes > 0) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(bytes, (size_t)max_persist));
            cudaStreamAttrValue v{};
            v.accessPolicyWindow.base_ptr = c->sums;
            v.accessPolicyWindow.num_bytes = bytes;
            v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)max_persist / (float)bytes);
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(c->cap_stream, cudaStreamAttributeAccessPolicyWindow, &v);
            if (getenv("RAPID_VERBOSE"))
              fprintf(stderr, "rapid: L2 persisting window %zu B (max persist %d, max window %d)\n", bytes,
                      max_persist, max_win);
          }
          cudaGetLastError();
        }
      }
      if ((rc = cuda_check(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal),
                           "begin capture")))
        return rc;
      c->capturing = true;
      c->cap_owned.clear();
      rc = enqueue(c, image, H, W, p, labels_out, c->cap_stream);
      c->capturing = false;
      cudaGraph_t g = nullptr;
      const cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
      auto drop_events = [&]() {
        for (cudaEvent_t ev : c->cap_owned) cudaEventDestroy(ev);
        c->cap_owned.clear();
      };
      if (rc) {
        if (g) cudaGraphDestroy(g);
        drop_events();
        return rc;
      }
      if ((rc = cuda_check(c, e, "end capture"))) {
        drop_events();
        return rc;
      }
      if (c->l2_persist) {  // the capture stream's window, set on every kernel node explicitly
        cudaStreamAttrValue sv{};
        if (cudaStreamGetAttribute(c->cap_stream, cudaStreamAttributeAccessPolicyWindow, &sv) == cudaSuccess &&
            sv.accessPolicyWindow.num_bytes > 0) {
          size_t nn = 0;
          cudaGraphGetNodes(g, nullptr, &nn);
          std::vector<cudaGraphNode_t> nodes(nn);
          if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
          cudaKernelNodeAttrValue kv{};
          kv.accessPolicyWindow = sv.accessPolicyWindow;
          int nk = 0;
          for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel &&
                cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &kv) == cudaSuccess)
              nk++;
          }
          if (getenv("RAPID_VERBOSE")) fprintf(stderr, "rapid: access-policy window on %d kernel nodes\n", nk);
        }
        cudaGetLastError();
      }
      rapid_ctx::GraphEntry ne;
      const cudaError_t ei = cudaGraphInstantiate(&ne.exec, g, 0);
      cudaGraphDestroy(g);
      if ((rc = cuda_check(c, ei, "graph instantiate"))) {
        drop_events();
        return rc;
      }
      ne.key = k;
      ne.evs = c->evs;
      ne.owned = c->cap_owned;
      ne.launches = c->launches;
      c->cap_owned.clear();
      c->gcache.push_back(ne);
      ent = &c->gcache.back();
    }
    ent->used = ++c->gclock;
    c->evs = ent->evs;  // the profile of this call = the events of this graph
    c->launches = ent->launches;
    rc = cuda_check(c, cudaGraphLaunch(ent->exec, s), "graph launch");
  } else {
    rc = enqueue(c, image, H, W, p, labels_out, s);
  }
  c->last = *p;
  c->last_prof = c->prof;
  c->have_run = true;
  c->last_stream = s;
  if (rc) return rc;
  return cuda_check(c, cudaGetLastError(), "launch");
}

int rapid_segment_host(rapid_ctx *c, const uint8_t *image_host, int32_t H, int32_t W,
                       const rapid_params *p, int32_t *labels_host, void *stream) {
  if (!c) return RAPID_E_ARG;
  if (!image_host || !labels_host) return fail(c, RAPID_E_ARG, "null host buffer");
  int rc = validate(c, H, W, p);
  if (rc) return rc;
  cudaSetDevice(c->device);
  const size_t px = (size_t)p->batch * H * W;
  if ((rc = ensure(c, c->himg, px * 3)) || (rc = ensure(c, c->hlab, px * 4))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemcpyAsync(c->himg.p, image_host, px * 3, cudaMemcpyHostToDevice, s);
  rc = rapid_segment(c, (const uint8_t *)c->himg.p, H, W, p, (int32_t *)c->hlab.p, stream);
  if (rc) return rc;
  cudaMemcpyAsync(labels_host, c->hlab.p, px * 4, cudaMemcpyDeviceToHost, s);
  rc = cuda_check(c, cudaStreamSynchronize(s), "rapid_segment_host");
  if (rc) return rc;
  unsigned err = 0;
  cudaMemcpy(&err, &c->ctl->err, 4, cudaMemcpyDeviceToHost);
  return err ? fail(c, RAPID_E_INTEGRITY, "RECOUNT mismatch") : RAPID_OK;
}

int rapid_segment_host_stream(rapid_ctx *c, const uint8_t *const *images, int32_t *const *labels, int32_t n,
                              int32_t H, int32_t W, const rapid_params *p, void *stream) {
  if (!c) return RAPID_E_ARG;
  if (!images || !labels || n < 1) return fail(c, RAPID_E_ARG, "null buffer list or n < 1");
  for (int k = 0; k < n; k++)
    if (!images[k] || !labels[k]) return fail(c, RAPID_E_ARG, "null host buffer");
  int rc = validate(c, H, W, p);
  if (rc) return rc;
  cudaSetDevice(c->device);
  const size_t px = (size_t)p->batch * H * W;
  if ((rc = ensure(c, c->himg, px * 3)) || (rc = ensure(c, c->hlab, px * 4)) ||
      (rc = ensure(c, c->himg2, px * 3)) || (rc = ensure(c, c->hlab2, px * 4)))
    return rc;
  if (!c->h2d) {
    if ((rc = cuda_check(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking), "h2d stream")) ||
        (rc = cuda_check(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking), "d2h stream")))
      return rc;
    for (cudaEvent_t &e : c->hev)
      if ((rc = cuda_check(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "stream events"))) return rc;
    if ((rc = cuda_check(c, cudaMallocHost(&c->herr, 64 * sizeof(uint32_t)), "pinned flags"))) return rc;
  }
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *dimg[2] = {(uint8_t *)c->himg.p, (uint8_t *)c->himg2.p};
  int32_t *dlab[2] = {(int32_t *)c->hlab.p, (int32_t *)c->hlab2.p};
  cudaEvent_t *in_done = c->hev, *seg_done = c->hev + 2, *out_done = c->hev + 4;
  // every event starts "complete" so that the first two segmentations need not wait
  for (cudaEvent_t e : c->hev) cudaEventRecord(e, s);
  uint32_t err_any = 0;
  for (int k = 0; k < n; k++) {
    const int b = k & 1;
    // image k -> buffer b, once segmentation k-2 has read it
    cudaStreamWaitEvent(c->h2d, seg_done[b], 0);
    cudaMemcpyAsync(dimg[b], images[k], px * 3, cudaMemcpyHostToDevice, c->h2d);
    cudaEventRecord(in_done[b], c->h2d);
    // segment k once its image is in and the labels of k-2 have left buffer b
    cudaStreamWaitEvent(s, in_done[b], 0);
    cudaStreamWaitEvent(s, out_done[b], 0);
    if ((rc = rapid_segment(c, dimg[b], H, W, p, dlab[b], stream))) break;
    cudaMemcpyAsync(&c->herr[k & 63], &c->ctl->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(seg_done[b], s);
    // labels k -> host while k+1 is copied in and segmented
    cudaStreamWaitEvent(c->d2h, seg_done[b], 0);
    cudaMemcpyAsync(labels[k], dlab[b], px * 4, cudaMemcpyDeviceToHost, c->d2h);
    cudaEventRecord(out_done[b], c->d2h);
    if ((k & 63) == 63) {  // drain the pinned flag ring
      cudaStreamSynchronize(s);
      for (int j = 0; j < 64; j++) err_any |= c->herr[j];
    }
  }
  const int rs = cuda_check(c, cudaStreamSynchronize(s), "host stream segment");
  const int r2 = cuda_check(c, cudaStreamSynchronize(c->d2h), "host stream d2h");
  if (rc) return rc;
  if (rs) return rs;
  if (r2) return r2;
  for (int j = 0; j < (n & 63); j++) err_any |= c->herr[j];
  return err_any ? fail(c, RAPID_E_INTEGRITY, "RECOUNT mismatch") : RAPID_OK;
}

int rapid_quality(rapid_ctx *c, const int32_t *labels, const int32_t *gt, int32_t B, int32_t H, int32_t W,
                  int32_t M, int32_t eps, rapid_quality_result *out, void *stream) {
  if (!c) return RAPID_E_ARG;
  if (!labels || !gt || !out || B < 1 || H < 1 || W < 1 || M < 1 || eps < 0)
    return fail(c, RAPID_E_ARG, "rapid_quality: bad arguments");
  const uint64_t px = (uint64_t)B * H * W;
  if (px >= (1ull << 32) || (uint64_t)B * M >= (1ull << 31)) return fail(c, RAPID_E_RANGE, "rapid_quality: sizes");
  cudaSetDevice(c->device);
  // pair histogram: at least 2x the pixels of small inputs, 4x the superpixels of large ones
  size_t cap = 1024;
  const size_t want = std::min<size_t>(2 * px, std::max<size_t>(8 * (size_t)B * M, 1 << 20));
  while (cap < want && cap < (1ull << 26)) cap <<= 1;
  int rc;
  if ((rc = ensure(c, c->qkeys, cap * 8)) || (rc = ensure(c, c->qcnt, cap * 4)) ||
      (rc = ensure(c, c->qsize, (size_t)B * M * 4)) || (rc = ensure(c, c->qspb, px)) ||
      (rc = ensure(c, c->qacc, 5 * 8)))
    return rc;
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(c->qkeys.p, 0xff, cap * 8, s);
  cudaMemsetAsync(c->qcnt.p, 0, cap * 4, s);
  cudaMemsetAsync(c->qsize.p, 0, (size_t)B * M * 4, s);
  cudaMemsetAsync(c->qacc.p, 0, 5 * 8, s);
  QualityArgs a;
  a.labels = labels;
  a.gt = gt;
  a.B = B; a.H = H; a.W = W; a.M = M; a.eps = eps;
  a.keys = (unsigned long long *)c->qkeys.p;
  a.cnt = (uint32_t *)c->qcnt.p;
  a.cmask = cap - 1;
  a.size = (uint32_t *)c->qsize.p;
  a.spb = (uint8_t *)c->qspb.p;
  a.acc = (unsigned long long *)c->qacc.p;
  launch_quality(a, c->sm_count, s);
  unsigned long long acc[5] = {0, 0, 0, 0, 0};
  cudaMemcpyAsync(acc, a.acc, sizeof acc, cudaMemcpyDeviceToHost, s);
  if ((rc = cuda_check(c, cudaStreamSynchronize(s), "rapid_quality"))) return rc;
  if (acc[4] & 2ull) return fail(c, RAPID_E_ARG, "rapid_quality: a label outside [0, M) or a negative segment id");
  if (acc[4] & 1ull) return fail(c, RAPID_E_CAPACITY, "rapid_quality: too many (superpixel, segment) pairs");
  out->pixels = px;
  out->leak_px = acc[0];
  out->gt_boundary_px = acc[1];
  out->covered_px = acc[2];
  out->pairs = acc[3];
  out->ue = (double)acc[0] / (double)px;
  out->br = acc[1] ? (double)acc[2] / (double)acc[1] : 1.0;
  return RAPID_OK;
}

int rapid_stats(rapid_ctx *c, rapid_sp_stat *out, uint64_t capacity, rapid_run_info *info) {
  if (!c) return RAPID_E_ARG;
  if (!c->have_run) return fail(c, RAPID_E_STATE, "no segmentation has run");
  cudaSetDevice(c->device);
  int rc = cuda_check(c, cudaStreamSynchronize(c->last_stream), "rapid_stats sync");
  if (rc) return rc;
  const Plan &P = c->plan;
  const size_t K = (size_t)P.B * P.M;
  Ctl *h = new Ctl;
  cudaMemcpy(h, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost);
  if (out && capacity) {
    const size_t n = std::min<size_t>(K, capacity);
    std::vector<unsigned long long> sums(n * SUMW);
    std::vector<int32_t> init(n);
    std::vector<uint8_t> alive(n), active(n);
    std::vector<int8_t> y(n);
    cudaMemcpy(sums.data(), c->sums, n * SUMW * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(init.data(), c->init, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(alive.data(), c->alive, n, cudaMemcpyDeviceToHost);
    cudaMemcpy(active.data(), c->active, n, cudaMemcpyDeviceToHost);
    cudaMemcpy(y.data(), c->y, n, cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < n; k++) {
      rapid_sp_stat &o = out[k];
      const long long *sv = (const long long *)&sums[k * SUMW];
      o.n = sv[0]; o.sum_r = sv[1]; o.sum_g = sv[2]; o.sum_b = sv[3]; o.sum_x = sv[4]; o.sum_y = sv[5];
      const double nn = (double)o.n;
      o.mean_r = o.n ? (double)o.sum_r / nn : 0.0;
      o.mean_g = o.n ? (double)o.sum_g / nn : 0.0;
      o.mean_b = o.n ? (double)o.sum_b / nn : 0.0;
      o.mean_x = o.n ? (double)o.sum_x / nn : 0.0;
      o.mean_y = o.n ? (double)o.sum_y / nn : 0.0;
      o.init_size = init[k];
      o.alive = (int8_t)alive[k];
      o.active = (int8_t)active[k];
      o.y = y[k];
      o.pad_ = 0;
    }
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->status = h->err ? RAPID_E_INTEGRITY : RAPID_OK;
    info->batch = P.B; info->H = P.H; info->W = P.W; info->n_superpixels = P.M;
    info->n_stages = P.nst; info->sweeps = c->last.sweeps;
    info->grid_rows = P.rows; info->grid_cols = P.cols;
    for (int s = 0; s < P.nst; s++) {
      info->stage_nbx[s] = P.st[s].nbx;
      info->stage_nby[s] = P.st[s].nby;
      info->stage_tiles[s] = (uint64_t)P.st[s].tiles_x * P.st[s].tiles_y * P.B;
      const bool work = s > 0 && (c->last.mask_rule == RAPID_MASK_CLASS || c->last.mask_rule == RAPID_MASK_BSP);
      info->stage_active_tiles[s] = work ? h->nwork[s] : info->stage_tiles[s];
      info->stage_victims[s] = h->stage_info[s][0];
      info->stage_merges[s] = h->stage_info[s][1];
      uint64_t run = 0;
      for (uint32_t t = 0; t < c->last.sweeps; t++) {
        run++;
        uint64_t com = 0;
        for (int ph = 0; ph < 4; ph++) com += h->cnt[s][t][ph][RAPID_C_COMMIT];
        if (com == 0) break;
      }
      info->stage_sweeps_run[s] = run;
      if (c->last_prof == 2)
        info->stage_window_blocks[s] =
            work ? h->stage_info[s][2] : (uint64_t)P.st[s].nbx * P.st[s].nby * P.B;
    }
    memcpy(info->phase, h->cnt, sizeof(info->phase));
    std::vector<uint8_t> alive(K), active(K);
    cudaMemcpy(alive.data(), c->alive, K, cudaMemcpyDeviceToHost);
    cudaMemcpy(active.data(), c->active, K, cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < K; k++) {
      info->alive += alive[k];
      info->active += alive[k] && active[k];
    }
  }
  const int st = h->err ? RAPID_E_INTEGRITY : RAPID_OK;
  delete h;
  rc = cuda_check(c, cudaGetLastError(), "rapid_stats");
  if (rc) return rc;
  return st ? fail(c, st, "RECOUNT mismatch") : RAPID_OK;
}

int rapid_set_profiling(rapid_ctx *c, int enable) {
  if (!c) return RAPID_E_ARG;
  c->prof = enable < 0 ? 0 : (enable > 3 ? 1 : enable);
  return RAPID_OK;
}

int rapid_get_profile(rapid_ctx *c, rapid_profile *out) {
  if (!c || !out) return RAPID_E_ARG;
  if (!c->have_run) return fail(c, RAPID_E_STATE, "no segmentation has run");
  cudaSetDevice(c->device);
  int rc = cuda_check(c, cudaStreamSynchronize(c->last_stream), "profile sync");
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  for (const ProfEv &e : c->evs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) != cudaSuccess) ms = 0.f;
    out->launches[e.cls][e.stage]++;
    out->ms[e.cls][e.stage] += ms;
  }
  out->total_launches = (uint64_t)c->launches;
  cudaGetLastError();  // elapsed-time failures are not sticky; do not leak them into later calls
  return RAPID_OK;
}

int rapid_debug_stop(rapid_ctx *c, int kind, int stage, int sweep, int phase) {
  if (!c) return RAPID_E_ARG;
  c->stop_kind = kind;
  c->stop_stage = stage;
  c->stop_sweep = sweep;
  c->stop_phase = phase;
  return RAPID_OK;
}

int rapid_debug_map(rapid_ctx *c, int32_t *host, uint64_t capacity, int32_t *nbx, int32_t *nby) {
  if (!c || !host) return RAPID_E_ARG;
  if (!c->stopped || !c->stop_map) return fail(c, RAPID_E_STATE, "no debug stop reached");
  cudaSetDevice(c->device);
  int rc = cuda_check(c, cudaStreamSynchronize(c->last_stream), "debug sync");
  if (rc) return rc;
  const size_t n = (size_t)c->stop_nbx * c->stop_nby * c->plan.B;
  if (capacity < n) return fail(c, RAPID_E_CAPACITY, "debug map capacity");
  rc = cuda_check(c, cudaMemcpy(host, c->stop_map, n * 4, cudaMemcpyDeviceToHost), "debug map copy");
  if (nbx) *nbx = c->stop_nbx;
  if (nby) *nby = c->stop_nby;
  return rc;
}

}  // extern "C"
