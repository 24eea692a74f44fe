// kernels.cuh — argument blocks and launch wrappers of the RAPID sm_100a kernels.
#pragma once
#include "common.cuh"

namespace rapid {

// ---- K4 / K5: one parity phase (propose, commit) --------------------------------------
struct PhaseArgs {
  StageDev st;
  SpDev sp;
  const uint8_t *image;
  int32_t H, W, B, M;
  int32_t cx, cy;            // phase colour (A5)
  int32_t gating;            // 0 off, 1 active[A] (CLASS/BSP), 2 Eq. 7 (EQ7)
  int32_t size_mode;         // RAPID_SIZE_*
  long long l_num, l_den;
  long long lam_pos, lam_b;  // Q16
  const int32_t *worklist;   // null: every tile of the stage
  const unsigned int *nwork; // device count of the worklist
  uint4 *cands;              // K4a -> K4b candidate list (2 x uint4 per entry)
  unsigned long long *cand_count;
  uint4 *props;              // proposals {stage-map index, A, B, packed RGB (pixel stage)}
  unsigned long long *prop_count;
  uint32_t stamp;            // phase index (non-zero)
  unsigned long long *cnt;        // [NCNT] counters of this phase
  const unsigned long long *prev; // counters of the previous sweep (phase 0), or null
  uint32_t *victim_any;
  uint32_t *bset;            // boundary sets of the stage (null: full-scan path K4a/K4b)
  int32_t gpw;               // k_sweep: word groups per warp to aim for (sizes the groups)
  int32_t tail_pct;          // k_sweep: % of the words dealt in quarter-size groups at the end
  unsigned int *wq;          // k_sweep: work-queue counter of this phase (zeroed per call)
  uint32_t *list;            // k_bset_list -> k_sweep<LIST>: the phase's set bits (word << 5 | bit)
  unsigned int *list_count;  // their number (zeroed per call)
};

struct SnapArgs {
  SpDev sp;
  int32_t K;
  uint32_t stamp;             // 0: refresh all; else only the superpixels marked in the dirty byte map
  long long l_num, l_den;     // size floor l (the outflow budget rem[] of the next phase)
  bool full_flags = false;    // dirty refresh that reads InitSize and flags from their tables
                              // (stage start after a merge round) instead of the old record
};

struct MergeArgs {
  StageDev st;
  SpDev sp;
  int32_t B, M, K;
  long long lam_pos, lam_b;
  long long u_num, u_den;
  uint32_t *victim_any;      // this stage's flag
  uint32_t *remap_pending;   // this stage's flag (out)
  // compaction scratch
  unsigned int *chunk;       // per-chunk counts -> offsets
  unsigned int *total;       // number of victims
  int32_t *vlist;            // ordered victims
  uint8_t *vtile;            // per stage tile: = vstamp if it holds a victim's boundary block (or null)
  uint8_t vstamp;
  // adjacency hash
  unsigned long long *hkeys;
  unsigned int *hvals;
  int32_t *hnext;
  int32_t *head;             // [K]
  unsigned long long hmask;
  const int32_t *worklist;   // active tiles of this stage (null: every tile)
  const unsigned int *nwork;
  // candidates
  unsigned int *deg;         // [victims] -> offsets (in place scan)
  unsigned int *deg_total;
  int32_t *candT;            // candidate target (global id), -1 = infeasible / resolved
  int32_t *candV;            // candidate's victim
  unsigned long long *candE; // dE_m as int128 (hi, lo)
  uint32_t *mlock;           // [K] matched flags (zero outside the round)
  uint32_t *res;             // [K] reservations (~0 outside the round)
  int32_t *pairs;            // merges (A, T)
  unsigned int *npairs;
  unsigned long long *stage_info; // [4]: victims, merges, active tiles, -
  unsigned int *flag;        // [2] cooperative match: pending-edge flags (zero outside)
  const uint32_t *bset;      // boundary sets of the stage (null: scan every block)
};

// ---- merge adjacency hash (open addressing, (victim, neighbour) -> shared edge length)
__device__ __forceinline__ unsigned long long hmix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
constexpr unsigned long long HEMPTY = ~0ull;

__device__ __forceinline__ void hash_add(const MergeArgs &a, int V, int T, unsigned e) {
  const unsigned long long key = ((unsigned long long)(unsigned)V << 32) | (unsigned)T;
  unsigned long long h = hmix(key) & a.hmask;
  while (true) {
    // most calls find an existing key: a plain (volatile) read avoids contended CAS
    const unsigned long long seen = *reinterpret_cast<volatile unsigned long long *>(&a.hkeys[h]);
    if (seen == key) {
      atomicAdd(&a.hvals[h], e);
      return;
    }
    if (seen != HEMPTY) {
      h = (h + 1) & a.hmask;
      continue;
    }
    const unsigned long long old = atomicCAS(&a.hkeys[h], HEMPTY, key);
    if (old == HEMPTY) {
      atomicAdd(&a.hvals[h], e);
      a.hnext[h] = atomicExch(&a.head[V], (int)h);
      return;
    }
    if (old == key) {
      atomicAdd(&a.hvals[h], e);
      return;
    }
    h = (h + 1) & a.hmask;
  }
}

struct PredictArgs {
  StageDev st;
  SpDev sp;
  int32_t B, M, K;
  int32_t mask_rule, n_proto;
  int32_t proto[4][3];
  long long tau2;
  const uint32_t *remap_pending;
  unsigned int *chunk;
  unsigned int *total;
  int32_t *alist;
  // f2 feature model (y_model == 1): P:271 features, A31
  int32_t y_model;
  long long feat_w[5];           // bias, w1..w4 (Q16.16)
  const uint8_t *image;
  int32_t H, W;
  const int32_t *b0x, *b0y;      // pixel column / row -> stage-0 block
  unsigned long long *scratch;   // [K][SUMW] zeroed scratch (the RECOUNT buffer)
  unsigned long long *hkeys;     // the merge hash keys (EMPTY outside merge rounds)
  unsigned long long hmask;
};

struct TransArgs {
  StageDev prev, next;
  SpDev sp;
  int32_t B, M;
  const uint32_t *remap_pending;
  int32_t gate;              // 1: build the active-tile worklist of `next`
  int32_t *worklist;
  unsigned int *nwork;
  uint32_t *bset;            // dyadic path: also write the boundary sets of `next` (else null)
  int32_t gating;            // static gate of the boundary sets (as PhaseArgs::gating)
};

struct InitArgs {
  StageDev st0;              // stage 0 (map, geometry, packed sums)
  SpDev sp;
  const uint8_t *image;
  int32_t H, W, B, M, K;
  int32_t rows, cols;
  const int32_t *X, *Y;      // cell boundaries (cols+1, rows+1)
  const int32_t *cellx, *celly; // cell index of each stage-0 block column / row
};

struct RecountArgs {
  StageDev st;
  SpDev sp;
  const uint8_t *image;
  int32_t H, W, B, M, K;
  unsigned long long *rc;    // [K][SUMW] recount scratch (zeroed)
  uint32_t *err;
};

struct FinalArgs {
  StageDev last;
  SpDev sp;
  int32_t B, H, W, M;
  const int32_t *bxp, *byp;  // block column / row of each pixel column / row
  const uint32_t *remap_pending;
  int32_t *labels;           // [B][H][W]
  const int32_t *worklist;   // remap pass: active tiles of `last` (null: every tile)
  const unsigned int *nwork;
  const uint8_t *vtile = nullptr;  // tiles marked by the last merge round's adjacency pass (or null)
  uint8_t vstamp = 0;
};

// ---- f4 quality metrics (quality.cu)
struct QualityArgs {
  const int32_t *labels, *gt;
  int32_t B, H, W, M, eps;
  unsigned long long *keys;  // [cap] pair keys ((img*M + sp) << 32 | gt), QEMPTY = free
  uint32_t *cnt;             // [cap] pair counts
  unsigned long long cmask;  // cap - 1
  uint32_t *size;            // [B*M] superpixel sizes
  uint8_t *spb;              // [B*H*W] superpixel-boundary flags
  unsigned long long *acc;   // [5] leak, gt boundary, covered, pairs, error flags
};

// launch wrappers (all enqueue on `s`)
void launch_init_sp(const InitArgs &a, cudaStream_t s);
// literal: f3 literal image pyramid (A32): colour data = area x rounded level mean
void launch_pyramid_leaf(const StageDev &st, const uint8_t *image, int H, int W, int B,
                         uint64_t *bsum, bool literal, cudaStream_t s);
void launch_pyramid_up(const StageDev &parent, const StageDev &child, int B, uint64_t *bsum, bool literal,
                       cudaStream_t s);
// b = 2 leaf fused with its b = 4 parent (uniform dyadic stages); false when not applicable
bool launch_pyramid_leaf24(const StageDev &st, const StageDev &up, const uint8_t *image, int H, int W, int B,
                           uint64_t *bsum, uint64_t *bsum_up, bool literal, cudaStream_t s);
void launch_init_map0(const InitArgs &a, cudaStream_t s);
void launch_stats0(const InitArgs &a, cudaStream_t s);
// ------------------------------------------------------------------ K3: snapshot (device side)
#ifndef RAPID_FULLREC
#define RAPID_FULLREC 0
#endif
constexpr bool kFullRec = RAPID_FULLREC;
__device__ __forceinline__ Rec make_rec(const SpDev &sp, int k, bool full = true) {
  // gathers with a 64-B L2 fill (ld64_*, common.cuh); coherent: the fused commit + snapshot
  // kernel reads sums its own atomics wrote
  const ulonglong2 s01 = ld64_v2u64(sp.sums + (size_t)k * SUMW), s23 = ld64_v2u64(sp.sums + (size_t)k * SUMW + 2);
  const ulonglong2 s45 = ld64_v2u64(sp.sums + (size_t)k * SUMW + 4);
  unsigned long long s[6] = {s01.x, s01.y, s23.x, s23.y, s45.x, s45.y};
  if (sp.dsum != nullptr) {  // fold K5's packed deltas of the last phase into the sums and clear them
    unsigned long long *q = sp.dsum + (size_t)k * 4;
    const ulonglong2 e01 = ld64_v2u64(q), e2 = ld64_v2u64(q + 2);
    if ((e01.x | e01.y | e2.x) != 0ull) {
      const unsigned long long e[3] = {e01.x, e01.y, e2.x};
#pragma unroll
      for (int w = 0; w < 3; w++) {
        const long long lo = (long long)(int32_t)(uint32_t)e[w];
        const long long hi = (long long)(e[w] - (unsigned long long)lo) >> 32;
        s[2 * w] += (unsigned long long)lo;
        s[2 * w + 1] += (unsigned long long)hi;
      }
      unsigned long long *t = sp.sums + (size_t)k * SUMW;
      *reinterpret_cast<ulonglong2 *>(t) = make_ulonglong2(s[0], s[1]);
      *reinterpret_cast<ulonglong2 *>(t + 2) = make_ulonglong2(s[2], s[3]);
      *reinterpret_cast<ulonglong2 *>(t + 4) = make_ulonglong2(s[4], s[5]);
      *reinterpret_cast<ulonglong2 *>(q) = make_ulonglong2(0ull, 0ull);
      q[2] = 0ull;
    }
  }
  const unsigned long long n = s[0];
  Rec r;
  r.n = (int32_t)n;
  uint32_t flags;
  if (full) {
    r.init = (int32_t)ld64_u32(sp.init + k);
    flags = ld64_u8(sp.alive + k) | (ld64_u8(sp.active + k) << 1) |
            ((uint32_t)((int)(int8_t)ld64_u8(sp.y + k) + 1) << 2);
  } else {
    // inside a stage's phase loop InitSize and the alive / active / y flags do not change (merges
    // and prediction come after the stage's last snapshot, and every stage starts with a full
    // refresh): one 32-B sector of the previous record instead of four flag-table gathers
    const int4 o0 = ld64_v4(&sp.rec[k]), o1 = ld64_v4(reinterpret_cast<const int4 *>(&sp.rec[k]) + 1);
    r.init = o1.y;
    flags = (uint32_t)o0.w >> 16;
  }
  uint32_t c0 = 0, c1 = 0, c2 = 0;
  int32_t mx = 0, my = 0;
  if (n > 0) {
    const unsigned long long twon = 2 * n;
    // round-half-up(2^F S / n) = floor((2^(F+1) S + n) / 2n)  (A24).  Exact quotient from a
    // double reciprocal estimate (relative error < 2^-50, quotients < 2^25, so the estimate is
    // within one of the quotient) and one integer correction step each way.
    const double rcp = 1.0 / (double)twon;
    auto qdiv = [&](unsigned long long num) -> unsigned long long {
      long long q = (long long)((double)num * rcp);
      long long r = (long long)(num - (unsigned long long)q * twon);
      if (r < 0) { q--; r += (long long)twon; }
      if (r >= (long long)twon) q++;
      return (unsigned long long)q;
    };
    // A33: a colour sum outside [0, 255 n] (only the literal pyramid's synthesised data makes
    // one, f3) gives a mean clamped to the intensity range
    auto cmean = [&](unsigned long long sc) -> uint32_t {
      if ((long long)sc < 0) return 0u;
      if (sc > 255ull * n) return 255u << FRAC;
      return (uint32_t)qdiv((sc << (FRAC + 1)) + n);
    };
    c0 = cmean(s[1]);
    c1 = cmean(s[2]);
    c2 = cmean(s[3]);
    mx = (int32_t)qdiv((s[4] << (FRAC + 1)) + n);
    my = (int32_t)qdiv((s[5] << (FRAC + 1)) + n);
  }
  r.mux = mx;
  r.muy = my;
  r.cq01 = c0 | (c1 << 16);
  r.cq2f = c2 | (flags << 16);
  r.pad0 = r.pad1 = 0;
  sp.rec[k] = r;
  return r;
}

// O6' budget of the next phase (A19): A's proposals commit iff their total outflow o keeps
// (n_snap - o) l_den >= l_num InitSize, i.e. o <= rem = floor((n_snap l_den - l_num InitSize) / l_den);
// K4 subtracts each proposal from rem[A], so K5 accepts A's proposals iff rem[A] >= 0 after K4
__device__ __forceinline__ int32_t outflow_budget(const Rec &r, long long l_num, long long l_den) {
  if (l_den <= 0) return 0;  // (size mode NONE: no budget)
  const long long S = (long long)r.n * l_den - l_num * (long long)r.init;
  if ((l_den & (l_den - 1)) == 0) return (int32_t)(S >> (63 - __clzll(l_den)));  // floor, power of 2
  long long q = S / l_den;
  if (q * l_den > S) q--;  // floor for negative S
  return (int32_t)q;
}

// Full refresh (stamp 0) or only the superpixels marked in the dirty byte map (set by the commits
// of the previous phase with plain stores), by warps wid = 0 .. nw-1.  A warp takes 128
// consecutive superpixels (lane l reads the 4 bytes of superpixels 4l .. 4l+3 as one word and
// clears it), compacts the marked ones and refreshes them 32 at a time (one record per lane).
// Also run at the end of the commit kernel (after a grid barrier).
__device__ __forceinline__ void snapshot_warps(const SnapArgs &a, int wid, int nw) {
  const int lane = lane_id();
  const int n4 = (a.K + 3) >> 2;
  const int nchunks = (n4 + 31) >> 5;
  for (int ch = wid; ch < nchunks; ch += nw) {
    const int i = ch * 32 + lane;  // 4-superpixel slice: superpixels 4i .. 4i+3
    unsigned m = 0;
    if (i < n4) {
      uint32_t *wp = a.sp.dirty + i;
      const uint32_t wv = *wp;
      if (a.stamp == 0u) {
#pragma unroll
        for (int j = 0; j < 4; j++)
          if (4 * i + j < a.K) m |= 1u << j;
      } else {
        m = (unsigned)((wv & 0xffu) != 0u) | ((unsigned)((wv & 0xff00u) != 0u) << 1) |
            ((unsigned)((wv & 0xff0000u) != 0u) << 2) | ((unsigned)((wv & 0xff000000u) != 0u) << 3);
      }
      if (wv != 0u) *wp = 0u;
    }
    unsigned incl = __popc(m);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned total = __shfl_sync(FULL, incl, 31);
    for (unsigned rb = 0; rb < total; rb += 32) {
      const unsigned k = rb + lane;
      int j = 0;  // source lane: #lanes with incl <= k
#pragma unroll
      for (int h = 16; h > 0; h >>= 1) {
        const unsigned v = __shfl_sync(FULL, incl, j + h - 1);
        if (v <= k) j += h;
      }
      const unsigned mj = __shfl_sync(FULL, m, j);
      unsigned r = k - (__shfl_sync(FULL, incl, j) - __popc(mj));
      if (k < total) {
        int bit = 0;  // r-th set bit of the 4-bit mask
        unsigned mm = mj;
        while (r) {
          mm &= mm - 1;
          r--;
        }
        bit = __ffs(mm) - 1;
        const int k = 4 * (ch * 32 + j) + bit;
        const Rec r = make_rec(a.sp, k, a.stamp == 0u || a.full_flags || kFullRec);
        // the outflow budget of the next phase starts full: every superpixel whose rem[] the
        // last phase lowered (every proposal's source) was marked dirty by K4 or K5
        a.sp.out[k] = outflow_budget(r, a.l_num, a.l_den);
        // K5's packed-delta condition: flag (plain store, sticky for the call) any snapshot size
        // above the call's limit; every record written since the call's first (full) refresh
        // went through here
        if (r.n > a.sp.nlim) *a.sp.big = 1u;
      }
    }
  }
}

void launch_snapshot(const SnapArgs &a, int grid, cudaStream_t s);

// Launch with the programmatic-stream-serialization attribute when g_pdl is set (the kernel must
// begin with pdl_wait_and_trigger()); a plain stream-ordered launch otherwise.
extern bool g_pdl;
extern int g_adj_tma;
extern int g_adj_ilp;
extern int g_adj_minb8;
extern int g_sweep_uni;
extern int g_bset_rows;
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = g_pdl ? at : nullptr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
}
// K4a: tmap = TMA descriptor of the stage map (CUtensorMap*), or null for the LDG loader
void launch_scan(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s);
void launch_eval(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s);
void launch_commit(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s);
cudaError_t launch_commit_snap(const PhaseArgs &a, bool pixel, int sm_count, cudaStream_t s);
// boundary-set sweep: K4 build (once per stage) and the fused bitset-driven sweep
void launch_bset_build(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s);
// list: a block stage's per-phase candidate list (k_bset_list, then k_sweep<LIST>)
void launch_sweep(const PhaseArgs &a, bool pixel, bool smallb, bool list, int sm_count, cudaStream_t s);
int sweep_occupancy();
int scan_occupancy();
int eval_occupancy();
constexpr int CAND_SLACK_PER_WARP = 64;  // chunked reservations: unused tail per scanning warp
// encode a 3-D TMA descriptor {nbx, nby, B} of int32 with box {TX+4, TY+2, 1};
// false when nbx*4 is not a multiple of 16 B (the LDG loader is used then)
bool make_label_tmap(void *tmap64B, int32_t *base, int nbx, int nby, int B);
cudaError_t launch_merge_round(const MergeArgs &a, const void *tmap, int tgrid, int grid, cudaStream_t s,
                        int *nlaunch);
bool launch_merge_adjacency_tma(const MergeArgs &a, const void *tmap, int grid, cudaStream_t s);
int tiles_occupancy();
void launch_quality(const QualityArgs &a, int sms, cudaStream_t s);
void launch_predict(const PredictArgs &a, int grid, cudaStream_t s, int *nlaunch);
// returns true when it also wrote the boundary sets of `next` (dyadic path with a.bset)
bool launch_transition(const TransArgs &a, cudaStream_t s);
// boundary sets of a dyadic uniform stage from its parents' map (after the transition wrote the
// child worklist); false when the stages are not dyadic uniform
bool launch_bset_dyadic(const TransArgs &a, int sms, cudaStream_t s);
void launch_recount(const RecountArgs &a, bool pixel, int grid, cudaStream_t s, int *nlaunch);
void launch_final(const FinalArgs &a, bool upsample, cudaStream_t s);
void launch_count_window(const StageDev &st, const SpDev &sp, int B, int M, unsigned long long *out,
                         cudaStream_t s);

}  // namespace rapid
