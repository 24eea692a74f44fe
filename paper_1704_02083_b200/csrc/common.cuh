// common.cuh — device-side data layout shared by the RAPID kernels (sm_100a).
// Product code: never includes or links anything under oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rapid {

constexpr int FRAC = 8;          // F: fractional bits of the snapshot means (DESIGN §2 A24)
constexpr int TX = 64;           // sweep tile width in blocks
constexpr int TY = 16;           // sweep tile height in blocks
constexpr int PROP_THREADS = 256;// one candidate per thread: (TX/2)*(TY/2) = 256
constexpr unsigned FULL = 0xffffffffu;
constexpr int NCNT = 6;          // per-phase counters (RAPID_C_*)
constexpr int MAXS = 12;
constexpr int MAXSW = 64;

// stats record of a superpixel: 8 x int64 (n, r, g, b, x, y, pad, pad); 64-B aligned
constexpr int SUMW = 8;

// Snapshot record: one 32-B sector per superpixel, refreshed before every phase
// (frozen per-phase means, DESIGN §2 A4).  cq/mu are round-half-up(2^F * mean).
struct __align__(16) Rec {
  int32_t mux, muy;   // position means, 2^F units (< 2^24)
  uint32_t cq01;      // cq_r | cq_g << 16 (each <= 255*2^8)
  uint32_t cq2f;      // cq_b | flags << 16
  int32_t n;          // size at snapshot
  int32_t init;       // InitSize
  int32_t pad0, pad1;
};
// flags
constexpr uint32_t F_ALIVE = 1u, F_ACTIVE = 2u;
// y is stored as (y + 1) in bits 2..3

// Division by a runtime-constant divisor d >= 1 for n < 2^31: with s = ceil(log2 d) and
// m = ceil(2^(31+s) / d) (< 2^32), floor(n/d) = umulhi(n, m) >> (s-1)  (error n*e < 2^(31+s)).
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d <= 1) return f;
  uint32_t s = 0;
  while ((1ull << s) < d) s++;
  f.m = (uint32_t)(((1ull << (31 + s)) + d - 1) / d);
  f.s = s - 1;
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
  return f.d <= 1 ? n : (__umulhi(n, f.m) >> f.s);
}
// Division of any n < 2^32 by d in [1, 2^32): with M = ceil(2^64 / d) (d >= 2),
// floor(n/d) = umul64hi(n, M), since n (M - 2^64/d) / 2^64 < 2^-32 <= 1/d.
struct FastDivU {
  unsigned long long M;
  uint32_t d;
};
inline FastDivU make_fastdivu(uint32_t d) {
  FastDivU f{0ull, d};
  if (d >= 2) f.M = ~0ull / d + 1ull;
  return f;
}
__device__ __forceinline__ uint32_t fdivu(uint32_t n, const FastDivU &f) {
  return f.d <= 1 ? n : (uint32_t)__umul64hi((unsigned long long)n, f.M);
}

struct StageDev {
  int32_t nbx, nby, b;
  int32_t uniform;               // 1: every block is b x b with xs[i] = i*b, ys[j] = j*b
  int32_t tiles_x, tiles_y;      // sweep tiles per image
  FastDiv fd_tx, fd_ty;          // division by tiles_x / tiles_y
  FastDivU fd_nbx, fd_nper;      // division by nbx / nbx * nby (block index -> img, gy, gx)
  const int32_t *xs, *ys;        // block boundaries (nbx+1, nby+1)
  const int32_t *px, *py;        // parent block index in stage s-1 (s > 0)
  const int32_t *cxs, *cys;      // first child index in stage s+1 (nbx+1, nby+1)
  const uint64_t *bsum;          // packed colour sums r | g<<21 | b<<42 (b > 1), else null;
  int32_t bsum32;                // 1: uniform b = 2 stage, sums stored as u32 r | g<<10 | b<<20 (<= 1020 each)
  int32_t *map;                  // stage label map [B][nby][nbx], per-image local ids
};

struct SpDev {
  unsigned long long *sums;  // [K][SUMW]
  Rec *rec;                  // [K]
  int32_t *init;             // [K]
  uint8_t *alive, *active;   // [K]
  int8_t *y;                 // [K]
  uint8_t *victim;           // [K]
  int32_t *out;              // [K] rem: outflow budget left in the current phase (O6', A19)
  uint32_t *dirty;           // byte map [K] (as words): superpixels whose sums (or budget) changed this phase
  int32_t *remap;            // [K]
  // K5's packed per-phase stats deltas: [K][4] u64, three words of two signed 32-bit fields
  // {n, r}, {g, b}, {x, y} (two's complement, summed modulo 2^64), folded into sums by K3 and
  // zero outside a phase; used while every snapshot size is <= the stage's limit
  unsigned long long *dsum;   // null: K5 always updates the sums directly
  unsigned int *big;          // set by K3 once a snapshot size exceeds nlim (sticky for the call)
  int32_t nlim;               // the call's size limit: the smallest stage limit
};

struct RecV {
  long long c0, c1, c2, mx, my;
};
__device__ __forceinline__ RecV rec_vals(const Rec &r) {
  RecV v;
  v.c0 = r.cq01 & 0xffffu;
  v.c1 = r.cq01 >> 16;
  v.c2 = r.cq2f & 0xffffu;
  v.mx = r.mux;
  v.my = r.muy;
  return v;
}

// Exact early exit (DESIGN §2 A25): a sweep with zero commits leaves labels and sums
// unchanged, so every later sweep of the stage would repeat it identically.
__device__ __forceinline__ bool sweep_skipped(const unsigned long long *prev) {
  if (prev == nullptr) return false;
  return (prev[0 * NCNT + 4] + prev[1 * NCNT + 4] + prev[2 * NCNT + 4] + prev[3 * NCNT + 4]) == 0ull;
}

// Yokoi 4-connectivity number == 1 on the 8-ring (N,NE,E,SE,S,SW,W,NW = bits 0..7):
// C4 = sum_{k in N,E,S,W} x_k (1 - x_{k+1} x_{k+2})   (E_topo; DESIGN A9)
__device__ __forceinline__ bool simple_point(unsigned m) {
  const unsigned r = m | (m << 8);  // ring wrap
  unsigned c = 0;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const unsigned xk = (r >> k) & 1u, x1 = (r >> (k + 1)) & 1u, x2 = (r >> (k + 2)) & 1u;
    c += xk & ~(x1 & x2) & 1u;
  }
  return c == 1u;
}

// position of the r-th set bit (0-based) of w; r < popc(w)
__device__ __forceinline__ unsigned nth_set_bit(uint32_t w, unsigned r) {
  unsigned pos = 0;
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {
    const unsigned lo = __popc(w & ((1u << h) - 1u));
    if (r >= lo) {
      r -= lo;
      pos += h;
      w >>= h;
    }
  }
  return pos;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Programmatic dependent launch (phase-loop kernels, RAPID_PDL): wait until the previous kernel
// in the stream has completed and its writes are visible (a no-op without a PDL launch), then
// let the next kernel's CTAs be launched while this one runs (they block in their own wait).
__device__ __forceinline__ void pdl_wait_and_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Warp-aggregated delta update of the six int64 sums of superpixel `key` (north star (d)):
// __match_any_sync groups the lanes by key, every group is reduced at once with REDUX
// (__reduce_add_sync on 16-bit halves: each d[f] is in [0, 2^47), so no 32-bit partial sum
// overflows), and each group's leader issues fire-and-forget int64 atomics.  Integer
// atomics are order-independent, so the result is deterministic.  The leader also marks the
// superpixel dirty (the next snapshot refreshes marked records only).
// Must be called by all 32 lanes (uniform control flow).
// Runs of adjacent lanes with equal keys (invalid lanes get unique keys): run start of this
// lane and whether it ends its run.  Full-mask intrinsics only (a per-group mask makes the
// compiler emit a divergent slow path).
struct WarpRun {
  int start;
  bool end;
};
__device__ __forceinline__ WarpRun warp_runs(bool valid, int key) {
  const int lane = lane_id();
  const int k = valid ? key : -1 - lane;
  const int kp = __shfl_up_sync(FULL, k, 1);
  const bool st = lane == 0 || kp != k;
  const unsigned sm = __ballot_sync(FULL, st);
  WarpRun r;
  r.start = 31 - __clz(sm & ((2u << lane) - 1u));
  r.end = lane == 31 || ((sm >> (lane + 1)) & 1u);
  return r;
}

// Streaming (evict-first) loads that ask L2 for a 64-B fill: without the prefetch-size
// qualifier an isolated load fetches 128 B from DRAM on this B200 (measured,
// tools/micro/dram_granularity.cu: 128 B per scattered 4-B load by default, 64 B with
// .L2::64B), which doubles the traffic of sparse 3x3 windows.
__device__ __forceinline__ int ld_stream64(const int32_t *p) {
  int v;
  asm("ld.global.cs.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream64(const uint32_t *p) {
  uint32_t v;
  asm("ld.global.cs.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream64(const uint8_t *p) {
  uint32_t v;
  asm("ld.global.cs.L2::64B.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_stream64(const unsigned long long *p) {
  unsigned long long v;
  asm("ld.global.cs.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// The same 64-B fill for gathers of the per-superpixel tables (records, sums, flags): coherent
// loads (the table may have been written earlier in the same kernel), and non-coherent
// read-only ones (.nc) where the kernel never writes it.
__device__ __forceinline__ int4 ld64_v4(const void *p) {
  int4 v;
  asm("ld.global.L2::64B.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ldnc64_v4(const void *p) {
  int4 v;
  asm("ld.global.nc.L2::64B.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong2 ld64_v2u64(const void *p) {
  ulonglong2 v;
  asm("ld.global.L2::64B.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld64_u32(const void *p) {
  uint32_t v;
  asm("ld.global.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld64_u8(const void *p) {
  uint32_t v;
  asm("ld.global.L2::64B.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldnc64_u32(const void *p) {
  uint32_t v;
  asm("ld.global.nc.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ Rec ldnc64_rec(const Rec *p) {
  const int4 a = ldnc64_v4(p), b = ldnc64_v4(reinterpret_cast<const int4 *>(p) + 1);
  Rec r;
  r.mux = a.x; r.muy = a.y; r.cq01 = (uint32_t)a.z; r.cq2f = (uint32_t)a.w;
  r.n = b.x; r.init = b.y; r.pad0 = b.z; r.pad1 = b.w;
  return r;
}

// int64 atomic add that asks L2 to keep the line (evict_last): the per-superpixel sums are
// the atomic targets of every phase and must not be displaced by the streaming label reads
__device__ __forceinline__ void red_add_keep(unsigned long long *p, unsigned long long v) {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ void mark_dirty(uint32_t *dirty, int key) {
  reinterpret_cast<uint8_t *>(dirty)[key] = 1u;  // byte map: a plain store, no atomic
}

// One aggregated stats delta: six int64 REDs on the sums, or (dsum) three on the packed
// per-phase delta words {n, r}, {g, b}, {x, y} — lo + hi * 2^32 modulo 2^64, so that negation
// and every sum of packed words stay packed; exact while each field's phase total fits int32
__device__ __forceinline__ void red_sums(const long long tot[6], int key, bool negate,
                                         unsigned long long *sums, unsigned long long *dsum) {
  if (dsum != nullptr) {
    unsigned long long *q = dsum + (size_t)key * 4;
#pragma unroll
    for (int w = 0; w < 3; w++) {
      const unsigned long long v =
          (unsigned long long)tot[2 * w] + ((unsigned long long)tot[2 * w + 1] << 32);
      red_add_keep(&q[w], negate ? 0ull - v : v);
    }
  } else {
    unsigned long long *q = sums + (size_t)key * SUMW;
#pragma unroll
    for (int f = 0; f < 6; f++) red_add_keep(&q[f], (unsigned long long)(negate ? -tot[f] : tot[f]));
  }
}

__device__ __forceinline__ void agg_sums(bool valid, int key, const long long d[6], bool negate,
                                         unsigned long long *sums, uint32_t *dirty,
                                         unsigned long long *dsum = nullptr) {
  if (__ballot_sync(FULL, valid) == 0u) return;  // warp-uniform
  const WarpRun run = warp_runs(valid, key);
  const int lane = lane_id();
  // segmented inclusive scan over each run: n, r, g, b fit 32 bits (block <= 64^2 pixels),
  // position sums need 64 bits
  unsigned v0 = valid ? (unsigned)d[0] : 0u, v1 = valid ? (unsigned)d[1] : 0u;
  unsigned v2 = valid ? (unsigned)d[2] : 0u, v3 = valid ? (unsigned)d[3] : 0u;
  long long v4 = valid ? d[4] : 0, v5 = valid ? d[5] : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t0 = __shfl_up_sync(FULL, v0, o), t1 = __shfl_up_sync(FULL, v1, o);
    const unsigned t2 = __shfl_up_sync(FULL, v2, o), t3 = __shfl_up_sync(FULL, v3, o);
    const long long t4 = __shfl_up_sync(FULL, v4, o), t5 = __shfl_up_sync(FULL, v5, o);
    if (lane - o >= run.start) {
      v0 += t0; v1 += t1; v2 += t2; v3 += t3; v4 += t4; v5 += t5;
    }
  }
  if (valid && run.end) {
    const long long tot[6] = {(long long)v0, (long long)v1, (long long)v2, (long long)v3, v4, v5};
    red_sums(tot, key, negate, sums, dsum);
    if (dirty != nullptr) mark_dirty(dirty, key);
  }
}

// Packed variant for blocks of at most 4 x 4 pixels (b <= 4): one move's data and any 32-lane
// run sum fit two 64-bit words without a field overflowing into the next — n (10 bits;
// <= 16 x 32), colour sums (18 bits each; <= 255 x 16 x 32), position sums (26 bits each;
// <= 2^20 x 32) — so the segmented scan moves 2 words instead of 6.
__device__ __forceinline__ void agg_sums_small(bool valid, int key, const long long d[6], bool negate,
                                               unsigned long long *sums, uint32_t *dirty,
                                               unsigned long long *dsum = nullptr) {
  if (__ballot_sync(FULL, valid) == 0u) return;  // warp-uniform
  const int lane = lane_id();
  unsigned long long u0 = 0, u1 = 0;
  if (valid) {
    u0 = (unsigned long long)d[0] | ((unsigned long long)d[1] << 10) | ((unsigned long long)d[2] << 28) |
         ((unsigned long long)d[3] << 46);
    u1 = (unsigned long long)d[4] | ((unsigned long long)d[5] << 26);
  }
  // runs of adjacent lanes with equal keys (the usual case: a warp's moves come from a few
  // boundary stretches) are summed by a segmented scan; the run ends holding the totals are
  // then grouped by key (runs of one key that are not adjacent) and the group's lowest run end
  // gathers the others' words with shuffles (iterations = largest group - 1, usually 0)
  const WarpRun run = warp_runs(valid, key);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t0 = __shfl_up_sync(FULL, u0, o), t1 = __shfl_up_sync(FULL, u1, o);
    if (lane - o >= run.start) {
      u0 += t0;
      u1 += t1;
    }
  }
  const bool rend = valid && run.end;
  const unsigned grp = __match_any_sync(FULL, rend ? key : -1 - lane);
  const bool leader = rend && (__ffs(grp) - 1) == lane;
  unsigned rem = leader ? grp & ~(1u << lane) : 0u;
  const unsigned long long v0 = u0, v1 = u1;
  while (__any_sync(FULL, rem != 0u)) {
    const int src = rem ? __ffs(rem) - 1 : lane;
    const unsigned long long t0 = __shfl_sync(FULL, v0, src), t1 = __shfl_sync(FULL, v1, src);
    if (rem) {
      u0 += t0;
      u1 += t1;
      rem &= rem - 1;
    }
  }
  if (leader) {
    const long long tot[6] = {(long long)(u0 & 0x3FFull), (long long)((u0 >> 10) & 0x3FFFFull),
                              (long long)((u0 >> 28) & 0x3FFFFull), (long long)(u0 >> 46),
                              (long long)(u1 & 0x3FFFFFFull), (long long)(u1 >> 26)};
    red_sums(tot, key, negate, sums, dsum);
    if (dirty != nullptr) mark_dirty(dirty, key);
  }
}

// Warp-aggregated int32 add (proposal outflow per source superpixel); |v| < 2^16.
__device__ __forceinline__ void agg_add_i32(bool valid, int key, int v, int32_t *arr) {
  if (__ballot_sync(FULL, valid) == 0u) return;  // warp-uniform
  const WarpRun run = warp_runs(valid, key);
  const int lane = lane_id();
  int s = valid ? v : 0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, s, o);
    if (lane - o >= run.start) s += t;
  }
  if (valid && run.end) atomicAdd(&arr[key], s);
}

// packed colour sums of block idx in the u64 layout r | g<<21 | b<<42 (from either storage)
__device__ __forceinline__ uint64_t widen_bsum32(uint32_t v) {
  return (uint64_t)(v & 0x3FFu) | ((uint64_t)((v >> 10) & 0x3FFu) << 21) | ((uint64_t)(v >> 20) << 42);
}
__device__ __forceinline__ uint64_t bsum_at(const StageDev &st, size_t idx) {
  return st.bsum32 ? widen_bsum32(reinterpret_cast<const uint32_t *>(st.bsum)[idx]) : st.bsum[idx];
}
__device__ __forceinline__ uint32_t narrow_bsum32(uint64_t pk) {
  return (uint32_t)(pk & 0x3FFull) | ((uint32_t)((pk >> 21) & 0x3FFull) << 10) | ((uint32_t)((pk >> 42) & 0x3FFull) << 20);
}

// Block data of a block at stage `st`: n, colour sums, position sums (x = column).
// Positions are closed-form sums over the block rectangle at full resolution (Eq. 8 exact).
__device__ __forceinline__ void block_data_blk(const StageDev &st, int img, int gx, int gy,
                                               long long d[6]) {
  const long long x0 = st.xs[gx], x1 = st.xs[gx + 1];
  const long long y0 = st.ys[gy], y1 = st.ys[gy + 1];
  const long long w = x1 - x0, h = y1 - y0;
  const uint64_t pk = bsum_at(st, ((size_t)img * st.nby + gy) * st.nbx + gx);
  d[0] = w * h;
  d[1] = (long long)(pk & 0x1FFFFFull);
  d[2] = (long long)((pk >> 21) & 0x1FFFFFull);
  d[3] = (long long)(pk >> 42);
  d[4] = h * ((w * (2 * x0 + w - 1)) / 2);
  d[5] = w * ((h * (2 * y0 + h - 1)) / 2);
}

__device__ __forceinline__ void block_data_pix(const uint8_t *image, int H, int W, int img, int gx,
                                               int gy, long long d[6]) {
  const uint8_t *p = image + (((size_t)img * H + gy) * W + gx) * 3;
  d[0] = 1;
  d[1] = p[0];
  d[2] = p[1];
  d[3] = p[2];
  d[4] = gx;
  d[5] = gy;
}

}  // namespace rapid
