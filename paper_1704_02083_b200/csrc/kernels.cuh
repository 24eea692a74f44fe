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
  uint32_t stamp;            // dirty stamp of this phase (superpixels whose sums change)
  unsigned long long *cnt;        // [NCNT] counters of this phase
  const unsigned long long *prev; // counters of the previous sweep (phase 0), or null
  uint32_t *victim_any;
  uint32_t *bset;            // boundary sets of the stage (null: full-scan path K4a/K4b)
  int32_t gpw;               // k_sweep: word groups per warp to aim for (sizes the groups)
  unsigned int *wq;          // k_sweep: work-queue counter of this phase (zeroed per call)
};

struct SnapArgs {
  SpDev sp;
  int32_t K;
  uint32_t stamp;             // 0: refresh all; else only superpixels with dirty == stamp
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
void launch_snapshot(const SnapArgs &a, int grid, cudaStream_t s);
// K4a: tmap = TMA descriptor of the stage map (CUtensorMap*), or null for the LDG loader
void launch_scan(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s);
void launch_eval(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s);
void launch_commit(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s);
// boundary-set sweep: K4 build (once per stage) and the fused bitset-driven sweep
void launch_bset_build(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s);
void launch_sweep(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s);
int sweep_occupancy();
int scan_occupancy();
int eval_occupancy();
constexpr int CAND_SLACK_PER_WARP = 64;  // chunked reservations: unused tail per scanning warp
// encode a 3-D TMA descriptor {nbx, nby, B} of int32 with box {TX+4, TY+2, 1};
// false when nbx*4 is not a multiple of 16 B (the LDG loader is used then)
bool make_label_tmap(void *tmap64B, int32_t *base, int nbx, int nby, int B);
void launch_merge_round(const MergeArgs &a, const void *tmap, int tgrid, int grid, cudaStream_t s,
                        int *nlaunch);
bool launch_merge_adjacency_tma(const MergeArgs &a, const void *tmap, int grid, cudaStream_t s);
int tiles_occupancy();
void launch_quality(const QualityArgs &a, int sms, cudaStream_t s);
void launch_predict(const PredictArgs &a, int grid, cudaStream_t s, int *nlaunch);
// returns true when it also wrote the boundary sets of `next` (dyadic path with a.bset)
bool launch_transition(const TransArgs &a, cudaStream_t s);
void launch_recount(const RecountArgs &a, bool pixel, int grid, cudaStream_t s, int *nlaunch);
void launch_final(const FinalArgs &a, bool upsample, cudaStream_t s);
void launch_count_window(const StageDev &st, const SpDev &sp, int B, int M, unsigned long long *out,
                         cudaStream_t s);

}  // namespace rapid
