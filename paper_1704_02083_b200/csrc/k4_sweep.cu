// sweep.cu — K4 (parity-phase boundary sweep, "propose") and K5 (commit) on sm_100a.
//
// One launch = one phase c = (cx, cy) of one sweep (DESIGN §2 A5/A6): every block of colour
// c in the stage map is tested in parallel against frozen per-phase means (A4):
//   boundary (Eq. 2) -> gate (Eq. 7 / prediction) -> simple point (E_topo)
//   -> Eq. 3 argmin over the distinct 4-neighbour labels of the Eq. 1 energy difference
//   -> size gate (E_size P:68 / RAPID l.19) -> commit or proposal.
//
// Structure (persistent, warp-specialised CTAs over the tile worklist; 8+1 warps):
//   * A producer lane streams (TY+2) x (TX+8) label tiles (1-block halo, 16-B aligned box)
//     with TMA (cp.async.bulk.tensor.3d) into a 4-stage shared-memory ring; full/empty
//     mbarriers hand the stages to the 8 consumer warps.  Maps whose row pitch is not a
//     multiple of 16 B use a per-warp LDG loader instead.
//   * Pass 1 (shared memory only): each consumer warp owns one candidate row of the tile
//     (32 blocks of the phase colour): boundary + 3x3 simple-point test; boundary blocks go
//     to the warp's own queue with their 4-neighbour labels.
//   * Pass 2 (whenever the warp queue holds >= 32 entries, and at the end): full-warp
//     evaluation — gate, colour gather, 32-B snapshot records of A and its neighbours (L2),
//     integer/int128 energy, argmin, size gate — then warp-aggregated int64 atomics
//     (size_mode NONE: commit in place) or proposals (HARD/MERGE).  No CTA-wide barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace rapid {

typedef __int128 i128;

// The TMA box starts HX = 4 blocks left of the tile: the inner coordinate of a tile load
// must be 16-B aligned (measured: x = -1 faults, x = -4 loads); width TX + 8 = 72 int32.
constexpr int HX = 4;
constexpr int BOXW = TX + 2 * HX;  // 72 int32 = 288 B
constexpr int BOXH = TY + 2;       // 18
constexpr int NSTAGE = 6;
constexpr unsigned TILE_BYTES = BOXH * BOXW * 4;
constexpr int STAGE_INTS = (BOXH * BOXW + 31) / 32 * 32;  // each TMA destination 128-B aligned

struct QE {         // queued boundary candidate (32 B)
  uint32_t pos;     // gx | gy << 16
  uint32_t imgt;    // img | topo_ok << 31
  int32_t A;
  int32_t n[4];     // N, E, S, W labels (-1: none)
  int32_t pad;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(m))
      : "memory");
}

// 2^(-16) x the oracle's weighted dE (same sign, same order): exact Eq. 1 difference of
// relabelling a pixel set with data d from A to B under the frozen quantised means.
__device__ __forceinline__ i128 delta_e(const RecV &ra, const RecV &rb, const long long d[6],
                                        long long dB2, long long lam_pos, long long lam_b) {
  const long long n = d[0];
  const long long dC = (rb.c0 - ra.c0) * (n * (rb.c0 + ra.c0) - (d[1] << (FRAC + 1))) +
                       (rb.c1 - ra.c1) * (n * (rb.c1 + ra.c1) - (d[2] << (FRAC + 1)));
  const i128 dCw = (i128)dC + (i128)((rb.c2 - ra.c2) * (n * (rb.c2 + ra.c2) - (d[3] << (FRAC + 1))));
  const long long dP = (rb.mx - ra.mx) * (n * (rb.mx + ra.mx) - (d[4] << (FRAC + 1))) +
                       (rb.my - ra.my) * (n * (rb.my + ra.my) - (d[5] << (FRAC + 1)));
  return (dCw << 16) + (i128)lam_pos * (i128)dP + ((i128)(lam_b * dB2) << 16);
}

struct Cnt {
  unsigned cand = 0, topo = 0, prop = 0, srej = 0, commit = 0;
};

// ------------------------------------------------------------------ pass 2 (one warp)
// Evaluates up to 32 queued candidates, one per lane: gate, colour, snapshot records,
// integer energy, Eq. 3 argmin, size gate; then commits (NONE) or emits proposals.
template <bool PIXEL, bool GATED>
__device__ __forceinline__ void eval_warp(const PhaseArgs &a, const QE *q, int n, Cnt &c) {
  const int lane = lane_id();
  const int nbx = a.st.nbx, nby = a.st.nby;
  const bool valid = lane < n;
  bool cand = false, topo = false, prop = false, srej = false;
  int A = 0, Bm = 0, kb = 0, gx = 0, gy = 0, img = 0;
  uint32_t rgb = 0;
  long long d[6] = {0, 0, 0, 0, 0, 0};
  if (valid) {
    const QE e = q[lane];
    gx = (int)(e.pos & 0xffffu);
    gy = (int)(e.pos >> 16);
    img = (int)(e.imgt & 0x7fffffffu);
    const bool topo_ok = (e.imgt >> 31) != 0;
    kb = img * a.M;
    A = e.A;
    bool gate = true;
    if (a.gating == 1) {
      gate = a.sp.active[kb + A] != 0;
    } else if (a.gating == 2) {  // Eq. 7 at block level
      const int8_t yA = a.sp.y[kb + A];
      gate = false;
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (e.n[k] >= 0 && e.n[k] != A && a.sp.y[kb + e.n[k]] != yA) gate = true;
    }
    cand = gate;
    if (gate && topo_ok) {
      topo = true;
      long long ew[4];
      if (PIXEL) {
        const uint8_t *p = a.image + (((size_t)img * a.H + gy) * a.W + gx) * 3;
        const uint32_t r = p[0], g = p[1], b = p[2];
        rgb = r | (g << 8) | (b << 16);
        d[0] = 1; d[1] = r; d[2] = g; d[3] = b; d[4] = gx; d[5] = gy;
        ew[0] = ew[1] = ew[2] = ew[3] = 1;
      } else {
        block_data_blk(a.st, img, gx, gy, d);
        const long long bw = a.st.xs[gx + 1] - a.st.xs[gx], bh = a.st.ys[gy + 1] - a.st.ys[gy];
        ew[0] = bw; ew[1] = bh; ew[2] = bw; ew[3] = bh;
      }
      // issue every record load before any use (memory-level parallelism)
      const Rec recA = a.sp.rec[kb + A];
      Rec rn[4];
      bool use[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int B = e.n[k];
        bool u = B >= 0 && B != A;
#pragma unroll
        for (int r = 0; r < k; r++) u &= (e.n[r] != B);
        use[k] = u;
        if (u) rn[k] = a.sp.rec[kb + B];
      }
      const RecV ra = rec_vals(recA);
      bool have = false;
      i128 bestE = 0;
      int bestB = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (!use[k]) continue;
        const int B = e.n[k];
        long long dB2 = 0;
#pragma unroll
        for (int r = 0; r < 4; r++)
          if (e.n[r] >= 0) dB2 += ew[r] * ((long long)(e.n[r] != B) - (long long)(e.n[r] != A));
        const i128 E = delta_e(ra, rec_vals(rn[k]), d, 2 * dB2, a.lam_pos, a.lam_b);
        if (!have || E < bestE || (E == bestE && B < bestB)) {
          have = true;
          bestE = E;
          bestB = B;
        }
      }
      if (have && bestE < 0) {
        if (a.size_mode != 0 &&
            ((long long)recA.n - d[0]) * a.l_den < a.l_num * (long long)recA.init) {
          srej = true;  // A12: the desired move would leave A below l * InitSize
          if (a.size_mode == 2) {
            a.sp.victim[kb + A] = 1;
            *a.victim_any = 1u;
          }
        } else {
          prop = true;
          Bm = bestB;
        }
      }
    }
  }
  c.cand += __popc(__ballot_sync(FULL, cand));
  c.topo += __popc(__ballot_sync(FULL, topo));
  c.srej += __popc(__ballot_sync(FULL, srej));
  const unsigned pm = __ballot_sync(FULL, prop);
  c.prop += __popc(pm);
  if (pm) {
    const size_t idx = ((size_t)img * nby + gy) * nbx + gx;
    if (!GATED) {  // size_mode NONE: no budget to check, commit in place
      if (prop) a.st.map[idx] = Bm;
      agg_sums(prop, kb + A, d, true, a.sp.sums, a.sp.dirty, a.stamp);
      agg_sums(prop, kb + Bm, d, false, a.sp.sums, a.sp.dirty, a.stamp);
      c.commit += __popc(pm);
    } else {
      agg_add_i32(prop, kb + A, (int)d[0], a.sp.out);
      unsigned long long pb = 0;
      if (lane == 0) pb = atomicAdd(a.prop_count, (unsigned long long)__popc(pm));
      pb = __shfl_sync(FULL, pb, 0);
      if (prop)
        a.props[pb + __popc(pm & lanemask_lt())] = make_uint4((unsigned)idx, (unsigned)A, (unsigned)Bm, rgb);
    }
  }
}

// Pass 1 for one warp: the 32 candidates of one tile row.  T[r][c] = label at
// (gx0 + c - 1, gy - 1 + r) for the warp's candidate row gy; -1 = outside the image.
// Boundary blocks are appended to the warp queue (returns the new queue length).
__device__ __forceinline__ int pass1_row(const int32_t (*T)[BOXW], int li, int gx, int gy, int img,
                                         bool inside, QE *wq, int qn) {
  bool bnd = false, topo_ok = false;
  int A = -1, n0 = -1, n1 = -1, n2 = -1, n3 = -1;
  if (inside) {
    A = T[1][li + 1];
    n0 = T[0][li + 1];  // N
    n1 = T[1][li + 2];  // E
    n2 = T[2][li + 1];  // S
    n3 = T[1][li];      // W
    bnd = (n0 >= 0 && n0 != A) | (n1 >= 0 && n1 != A) | (n2 >= 0 && n2 != A) | (n3 >= 0 && n3 != A);
    if (bnd) {
      const unsigned m = (unsigned)(n0 == A) | ((unsigned)(T[0][li + 2] == A) << 1) |
                         ((unsigned)(n1 == A) << 2) | ((unsigned)(T[2][li + 2] == A) << 3) |
                         ((unsigned)(n2 == A) << 4) | ((unsigned)(T[2][li] == A) << 5) |
                         ((unsigned)(n3 == A) << 6) | ((unsigned)(T[0][li] == A) << 7);
      topo_ok = simple_point(m);
    }
  }
  const unsigned bm = __ballot_sync(FULL, bnd);
  if (bnd) {
    int4 *dst = reinterpret_cast<int4 *>(&wq[qn + __popc(bm & lanemask_lt())]);
    dst[0] = make_int4((int)((uint32_t)gx | ((uint32_t)gy << 16)),
                       (int)((uint32_t)img | (topo_ok ? 0x80000000u : 0u)), A, n0);
    dst[1] = make_int4(n1, n2, n3, 0);
  }
  return qn + __popc(bm);
}

// Drain full 32-entry rounds of the warp queue (or everything when `all`).
template <bool PIXEL, bool GATED>
__device__ __forceinline__ int drain(const PhaseArgs &a, QE *wq, int qn, bool all, Cnt &c) {
  const int lane = lane_id();
  while (qn >= 32 || (all && qn > 0)) {
    __syncwarp();
    eval_warp<PIXEL, GATED>(a, wq, qn < 32 ? qn : 32, c);
    __syncwarp();
    const int rest = qn > 32 ? qn - 32 : 0;
    int4 v0 = make_int4(0, 0, 0, 0), v1 = v0;
    if (lane < rest) {
      const int4 *src = reinterpret_cast<const int4 *>(&wq[32 + lane]);
      v0 = src[0];
      v1 = src[1];
    }
    __syncwarp();
    if (lane < rest) {
      int4 *dst = reinterpret_cast<int4 *>(&wq[lane]);
      dst[0] = v0;
      dst[1] = v1;
    }
    __syncwarp();
    qn = rest;
  }
  return qn;
}

// ------------------------------------------------------------------ K4
// Warp-specialised persistent kernel: warp NWARP (one lane) produces TMA tile loads into an
// NSTAGE ring (full/empty mbarriers); warps 0..NWARP-1 each own one candidate row of the
// tile (pass 1) and their own candidate queue (pass 2).  No CTA-wide barrier in the loop.
constexpr int NWARP = TY / 2;  // 8 consumer warps
constexpr int WQCAP = 64;
constexpr int K4_THREADS = (NWARP + 1) * 32;

template <bool PIXEL, bool GATED, bool USE_TMA>
#ifndef K4_MIN_BLOCKS
#define K4_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(K4_THREADS, K4_MIN_BLOCKS) k_sweep(const PhaseArgs a,
                                                      const __grid_constant__ CUtensorMap tmap) {
  if (sweep_skipped(a.prev)) return;
  __shared__ __align__(128) int32_t buf[NSTAGE][STAGE_INTS];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
  __shared__ int4 s_info[NSTAGE];  // gx0, gy0, img, border
  __shared__ __align__(16) QE q[NWARP][WQCAP];
  // LDG loader: private 3-row windows per warp, carved from the (then unused) TMA ring
  int32_t(*wrow)[3][BOXW] = reinterpret_cast<int32_t(*)[3][BOXW]>(&buf[0][0]);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nbx = a.st.nbx, nby = a.st.nby;
  const int tiles_x = a.st.tiles_x, tiles_y = a.st.tiles_y;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(tiles_x * tiles_y) * (unsigned)a.B;

  if (threadIdx.x == 0 && USE_TMA) {
    for (int s = 0; s < NSTAGE; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NWARP) {  // ---- producer warp: 32 tiles decoded in parallel, lane 0 issues
    if (!USE_TMA) return;
    for (unsigned kb = 0; blockIdx.x + kb * gridDim.x < ntiles; kb += 32) {
      const unsigned wl = blockIdx.x + (kb + lane) * gridDim.x;
      int4 inf = make_int4(0, 0, 0, 0);
      if (wl < ntiles) {
        const uint32_t t = a.worklist ? (uint32_t)a.worklist[wl] : wl;
        const uint32_t r = fdiv(t, a.st.fd_tx), img = fdiv(r, a.st.fd_ty);
        const int gx0 = (int)(t - r * (uint32_t)tiles_x) * TX, gy0 = (int)(r - img * (uint32_t)tiles_y) * TY;
        const int border = (gx0 == 0 || gy0 == 0 || gx0 + TX + 1 > nbx || gy0 + TY + 1 > nby) ? 1 : 0;
        inf = make_int4(gx0, gy0, (int)img, border);
      }
      for (int j = 0; j < 32; j++) {
        const unsigned k = kb + j;
        if (blockIdx.x + k * gridDim.x >= ntiles) break;  // warp-uniform
        int4 v;
        v.x = __shfl_sync(FULL, inf.x, j);
        v.y = __shfl_sync(FULL, inf.y, j);
        v.z = __shfl_sync(FULL, inf.z, j);
        v.w = __shfl_sync(FULL, inf.w, j);
        if (lane == 0) {
          const int st = (int)(k % NSTAGE);
          if (k >= NSTAGE) mbar_wait(&empty[st], ((k / NSTAGE) - 1) & 1u);
          s_info[st] = v;
          fence_proxy_async();
          mbar_expect_tx(&full[st], TILE_BYTES);
          tma_load_3d(&buf[st][0], &tmap, v.x - HX, v.y - 1, v.z, &full[st]);
        }
        __syncwarp();
      }
    }
    return;
  }

  // ---- consumers
  const int li = 2 * lane + a.cx;     // candidate column within the tile
  const int lr = 2 * warp + a.cy;     // candidate row within the tile
  QE *wq = q[warp];
  int qn = 0;
  Cnt c;
  for (unsigned k = 0;; k++) {
    const unsigned w = blockIdx.x + k * gridDim.x;
    if (w >= ntiles) break;
    const int st = (int)(k % NSTAGE);
    int gx0, gy0, img, border;
    const int32_t(*T)[BOXW];
    if (USE_TMA) {
      mbar_wait(&full[st], (k / NSTAGE) & 1u);
      const int4 inf = s_info[st];
      gx0 = inf.x; gy0 = inf.y; img = inf.z; border = inf.w;
      int32_t *rows = buf[st] + lr * BOXW;  // smem rows lr .. lr+2 = gy-1 .. gy+1
      if (border) {  // TMA zero-fills outside the image; 0 is a label: mark "no block"
        for (int idx = lane; idx < 3 * BOXW; idx += 32) {
          const int r = idx / BOXW, cc = idx - r * BOXW;
          const int y = gy0 + lr - 1 + r, x = gx0 + cc - HX;
          if (x < 0 || x >= nbx || y < 0 || y >= nby) rows[idx] = -1;
        }
        __syncwarp();
      }
      T = reinterpret_cast<const int32_t(*)[BOXW]>(rows + (HX - 1));
    } else {
      const uint32_t t = a.worklist ? (uint32_t)a.worklist[w] : w;
      const uint32_t r = fdiv(t, a.st.fd_tx), im = fdiv(r, a.st.fd_ty);
      img = (int)im;
      gx0 = (int)(t - r * (uint32_t)tiles_x) * TX;
      gy0 = (int)(r - im * (uint32_t)tiles_y) * TY;
      const int32_t *map = a.st.map + (size_t)img * nby * nbx;
      __syncwarp();
      int32_t v[(3 * BOXW + 31) / 32];
#pragma unroll
      for (int u = 0; u < (3 * BOXW + 31) / 32; u++) {
        const int idx = lane + 32 * u;
        const int rr = idx / BOXW, cc = idx - rr * BOXW;
        const int y = gy0 + lr - 1 + rr, x = gx0 + cc - HX;
        v[u] = (idx < 3 * BOXW && x >= 0 && x < nbx && y >= 0 && y < nby) ? map[(size_t)y * nbx + x] : -1;
      }
#pragma unroll
      for (int u = 0; u < (3 * BOXW + 31) / 32; u++) {
        const int idx = lane + 32 * u;
        if (idx < 3 * BOXW) (&wrow[warp][0][0])[idx] = v[u];
      }
      __syncwarp();
      T = reinterpret_cast<const int32_t(*)[BOXW]>(&wrow[warp][0][0] + (HX - 1));
    }
    const int gx = gx0 + li, gy = gy0 + lr;
    qn = pass1_row(T, li, gx, gy, img, gx < nbx && gy < nby, wq, qn);
    __syncwarp();
    if (USE_TMA && lane == 0) mbar_arrive(&empty[st]);
    qn = drain<PIXEL, GATED>(a, wq, qn, false, c);
  }
  drain<PIXEL, GATED>(a, wq, qn, true, c);
  if (lane == 0) {
    if (c.cand) atomicAdd(&a.cnt[0], (unsigned long long)c.cand);
    if (c.topo) atomicAdd(&a.cnt[1], (unsigned long long)c.topo);
    if (c.prop) atomicAdd(&a.cnt[2], (unsigned long long)c.prop);
    if (c.srej) atomicAdd(&a.cnt[3], (unsigned long long)c.srej);
    if (c.commit) atomicAdd(&a.cnt[4], (unsigned long long)c.commit);
  }
}

// ------------------------------------------------------------------ K5: commit
template <bool PIXEL>
__global__ void __launch_bounds__(256) k_commit(const PhaseArgs a) {
  if (sweep_skipped(a.prev)) return;
  const unsigned long long n = *a.prop_count;
  const size_t nper = (size_t)a.st.nbx * a.st.nby;
  unsigned c_commit = 0, c_rej = 0;
  for (unsigned long long base = blockIdx.x * 256ull; base < n; base += gridDim.x * 256ull) {
    const unsigned long long i = base + threadIdx.x;
    const bool valid = i < n;
    bool ok = false, rej = false;
    int A = 0, B = 0, kb = 0;
    long long d[6] = {0, 0, 0, 0, 0, 0};
    if (valid) {
      const uint4 pr = a.props[i];
      const size_t idx = pr.x;
      A = (int)pr.y;
      B = (int)pr.z;
      const int img = (int)(idx / nper);
      const size_t r = idx - (size_t)img * nper;
      const int gy = (int)(r / a.st.nbx), gx = (int)(r - (size_t)gy * a.st.nbx);
      kb = img * a.M;
      const Rec ra = a.sp.rec[kb + A];
      // O6' all-or-nothing budget: the total proposed outflow must keep A >= l * InitSize (A19)
      ok = !(((long long)ra.n - (long long)a.sp.out[kb + A]) * a.l_den < a.l_num * (long long)ra.init);
      if (ok) {
        if (PIXEL) {
          d[0] = 1; d[1] = pr.w & 0xffu; d[2] = (pr.w >> 8) & 0xffu; d[3] = (pr.w >> 16) & 0xffu;
          d[4] = gx; d[5] = gy;
        } else {
          block_data_blk(a.st, img, gx, gy, d);
        }
        a.st.map[idx] = B;
      } else {
        rej = true;
        if (a.size_mode == 2) {
          a.sp.victim[kb + A] = 1;
          *a.victim_any = 1u;
        }
      }
    }
    agg_sums(ok, kb + A, d, true, a.sp.sums, a.sp.dirty, a.stamp);
    agg_sums(ok, kb + B, d, false, a.sp.sums, a.sp.dirty, a.stamp);
    c_commit += __popc(__ballot_sync(FULL, ok));
    c_rej += __popc(__ballot_sync(FULL, rej));
  }
  if (lane_id() == 0) {
    if (c_commit) atomicAdd(&a.cnt[4], (unsigned long long)c_commit);
    if (c_rej) atomicAdd(&a.cnt[5], (unsigned long long)c_rej);
  }
}

// ------------------------------------------------------------------ host side
bool make_label_tmap(void *tmap64B, int32_t *base, int nbx, int nby, int B) {
  if (((size_t)nbx * 4) % 16 != 0) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)nbx, (cuuint64_t)nby, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)nbx * 4, (cuuint64_t)nbx * nby * 4};
  const cuuint32_t box[3] = {(cuuint32_t)BOXW, (cuuint32_t)BOXH, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode((CUtensorMap *)tmap64B, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, base, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool P, bool G, bool T>
static int occ() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep<P, G, T>, K4_THREADS, 0);
  return nb < 1 ? 1 : nb;
}

int propose_occupancy(bool pixel, bool gated) {
  return pixel ? (gated ? occ<true, true, true>() : occ<true, false, true>())
               : (gated ? occ<false, true, true>() : occ<false, false, true>());
}

void launch_propose(const PhaseArgs &a, const void *tmap, bool pixel, int grid, cudaStream_t s) {
  const bool gated = a.size_mode != 0;
  static CUtensorMap dummy;
  const CUtensorMap &m = tmap ? *(const CUtensorMap *)tmap : dummy;
  if (tmap) {
    if (pixel && gated) k_sweep<true, true, true><<<grid, K4_THREADS, 0, s>>>(a, m);
    else if (pixel) k_sweep<true, false, true><<<grid, K4_THREADS, 0, s>>>(a, m);
    else if (gated) k_sweep<false, true, true><<<grid, K4_THREADS, 0, s>>>(a, m);
    else k_sweep<false, false, true><<<grid, K4_THREADS, 0, s>>>(a, m);
  } else {
    if (pixel && gated) k_sweep<true, true, false><<<grid, K4_THREADS, 0, s>>>(a, m);
    else if (pixel) k_sweep<true, false, false><<<grid, K4_THREADS, 0, s>>>(a, m);
    else if (gated) k_sweep<false, true, false><<<grid, K4_THREADS, 0, s>>>(a, m);
    else k_sweep<false, false, false><<<grid, K4_THREADS, 0, s>>>(a, m);
  }
}

void launch_commit(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s) {
  if (pixel) k_commit<true><<<grid, 256, 0, s>>>(a);
  else k_commit<false><<<grid, 256, 0, s>>>(a);
}

}  // namespace rapid
