// sweep.cu — the parity-phase boundary sweep on sm_100a: K4a scan, K4b evaluate, K5 commit.
//
// One phase c = (cx, cy) of one sweep (DESIGN §2 A5/A6) tests every block of colour c of the
// stage map in parallel against frozen per-phase means (A4):
//   boundary (Eq. 2) -> gate (Eq. 7 / prediction) -> simple point (E_topo)
//   -> Eq. 3 argmin over the distinct 4-neighbour labels of the Eq. 1 energy difference
//   -> size gate (E_size P:68 / RAPID l.19) -> commit or proposal.
//
// K4a  k_scan (streaming, HBM-bound): persistent warp-specialised CTAs over the tile
//      worklist.  A producer lane streams (TY+2) x (TX+8) label tiles (1-block halo,
//      16-B aligned box) with TMA (cp.async.bulk.tensor.3d) into an NSTAGE shared-memory
//      ring; full/empty mbarriers hand the stages to 8 consumer warps, one candidate row
//      (32 blocks of the phase colour) each.  Consumers test boundary + 3x3 simple point in
//      shared memory, gate the boundary blocks, and append the survivors — with their 4
//      neighbour labels — to a compact global candidate list (per-warp chunk reservations).
//      Maps whose row pitch is not a multiple of 16 B use a per-warp LDG loader.
// K4b  k_eval (gather-bound, full occupancy): one candidate per thread — colour, 32-B
//      snapshot records of A and its neighbours (L2), int64/int128 energy, argmin, size
//      gate — then warp-aggregated int64 atomics (size_mode NONE: commit in place) or
//      proposals (HARD/MERGE).
// K5   k_commit: all-or-nothing size budget per source superpixel (A19), label writes,
//      warp-aggregated stats deltas.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

#include <algorithm>
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace rapid {
namespace cg = cooperative_groups;

typedef __int128 i128;

// The TMA box starts HX = 4 blocks left of the tile: the inner coordinate of a tile load
// must be 16-B aligned (measured: x = -1 faults, x = -4 loads); width TX + 8 = 72 int32.
constexpr int HX = 4;
constexpr int BOXW = TX + 2 * HX;  // 72 int32 = 288 B
constexpr int BOXH = TY + 2;       // 18
constexpr int NSTAGE = 6;
constexpr unsigned TILE_BYTES = BOXH * BOXW * 4;
constexpr int STAGE_INTS = (BOXH * BOXW + 31) / 32 * 32;  // each TMA destination 128-B aligned
constexpr int NWARP = TY / 2;                             // consumer warps (one candidate row each)
constexpr int K4A_THREADS = (NWARP + 1) * 32;
constexpr int CHUNK = 64;                                 // candidate slots reserved per atomic
constexpr int K4B_THREADS = 256;

// candidate entry (32 B = 2 x uint4): {pos = gx | gy << 16, img, A, N}, {E, S, W, 0};
// A = -1 marks an unused reserved slot.

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

// Work count of a list-driven kernel, read once per CTA (thread 0) and broadcast through
// shared memory: 0 when the sweep is skipped (A25) or the list is empty, and also 0 for
// CTAs whose first element lies beyond the list.  Must be called by all threads.
// the phase's list length as seen by this CTA: 0 when the CTA has no entry (per_cta) — or only
// when the list is empty (grid-uniform, for kernels with a grid barrier)
__device__ __forceinline__ unsigned long long cta_count(const unsigned long long *prev,
                                                         const unsigned long long *count,
                                                         bool per_cta = true) {
  __shared__ unsigned long long s_n;
  if (threadIdx.x == 0) s_n = sweep_skipped(prev) ? 0ull : *count;
  __syncthreads();
  const unsigned long long n = s_n;
  return (!per_cta || (unsigned long long)blockIdx.x * blockDim.x < n) ? n : 0ull;
}


// ------------------------------------------------------------------ K4a: scan
template <bool USE_TMA>
__global__ void __launch_bounds__(K4A_THREADS) k_scan(const PhaseArgs a,
                                                      const __grid_constant__ CUtensorMap tmap) {
  if (sweep_skipped(a.prev)) return;
  __shared__ __align__(128) int32_t buf[NSTAGE][STAGE_INTS];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
  __shared__ int4 s_info[NSTAGE];  // gx0, gy0, img, border
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
  // LDG loader: private 3-row windows per warp, carved from the (then unused) TMA ring
  int32_t(*wrow)[3][BOXW] = reinterpret_cast<int32_t(*)[3][BOXW]>(&buf[0][0]);
  const int li = 2 * lane + a.cx;  // candidate column within the tile
  const int lr = 2 * warp + a.cy;  // candidate row within the tile
  unsigned c_cand = 0, c_topo = 0;
  unsigned long long cbase = 0;
  int cleft = 0;
  for (unsigned k = 0;; k++) {
    const unsigned w = blockIdx.x + k * gridDim.x;
    if (w >= ntiles) break;
    const int st = (int)(k % NSTAGE);
    int gx0, gy0, img;
    const int32_t(*T)[BOXW];
    if (USE_TMA) {
      mbar_wait(&full[st], (k / NSTAGE) & 1u);
      const int4 inf = s_info[st];
      gx0 = inf.x; gy0 = inf.y; img = inf.z;
      int32_t *rows = buf[st] + lr * BOXW;  // smem rows lr .. lr+2 = gy-1 .. gy+1
      if (inf.w) {  // TMA zero-fills outside the image; 0 is a label: mark "no block"
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
      constexpr int PER = (3 * BOXW + 31) / 32;
      int32_t v[PER];
#pragma unroll
      for (int u = 0; u < PER; u++) {
        const int idx = lane + 32 * u;
        const int rr = idx / BOXW, cc = idx - rr * BOXW;
        const int y = gy0 + lr - 1 + rr, x = gx0 + cc - HX;
        v[u] = (idx < 3 * BOXW && x >= 0 && x < nbx && y >= 0 && y < nby) ? map[(size_t)y * nbx + x] : -1;
      }
#pragma unroll
      for (int u = 0; u < PER; u++) {
        const int idx = lane + 32 * u;
        if (idx < 3 * BOXW) (&wrow[warp][0][0])[idx] = v[u];
      }
      __syncwarp();
      T = reinterpret_cast<const int32_t(*)[BOXW]>(&wrow[warp][0][0] + (HX - 1));
    }
    // boundary (Eq. 2) + simple point (E_topo) from shared memory; T[r][c] = (gx0+c-1, gy-1+r)
    const int gx = gx0 + li, gy = gy0 + lr;
    bool bnd = false, topo_ok = false;
    int A = -1, n0 = -1, n1 = -1, n2 = -1, n3 = -1;
    if (gx < nbx && gy < nby) {
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
    __syncwarp();
    if (USE_TMA && lane == 0) mbar_arrive(&empty[st]);  // tile slot free for the producer
    // gate (A22): CLASS/BSP -> active[A]; EQ7 -> a neighbour of another label and class
    bool cand = bnd;
    if (bnd && a.gating) {
      const int kb = img * a.M;
      if (a.gating == 1) {
        cand = a.sp.active[kb + A] != 0;
      } else {
        const int8_t yA = a.sp.y[kb + A];
        cand = (n0 >= 0 && n0 != A && a.sp.y[kb + n0] != yA) || (n1 >= 0 && n1 != A && a.sp.y[kb + n1] != yA) ||
               (n2 >= 0 && n2 != A && a.sp.y[kb + n2] != yA) || (n3 >= 0 && n3 != A && a.sp.y[kb + n3] != yA);
      }
    }
    const bool emit = cand && topo_ok;
    c_cand += __popc(__ballot_sync(FULL, cand));
    const unsigned em = __ballot_sync(FULL, emit);
    const int ne = __popc(em);
    c_topo += ne;
    if (ne) {
      if (ne > cleft) {  // retire the rest of the chunk, reserve a new one
        if (lane < cleft) a.cands[2 * (cbase + lane)] = make_uint4(0u, 0u, 0xffffffffu, 0u);
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(a.cand_count, (unsigned long long)CHUNK);
        cbase = __shfl_sync(FULL, nb, 0);
        cleft = CHUNK;
      }
      if (emit) {
        const unsigned long long slot = cbase + __popc(em & lanemask_lt());
        a.cands[2 * slot] = make_uint4((uint32_t)gx | ((uint32_t)gy << 16), (uint32_t)img, (uint32_t)A, (uint32_t)n0);
        a.cands[2 * slot + 1] = make_uint4((uint32_t)n1, (uint32_t)n2, (uint32_t)n3, 0u);
      }
      cbase += ne;
      cleft -= ne;
    }
  }
  if (lane < cleft) a.cands[2 * (cbase + lane)] = make_uint4(0u, 0u, 0xffffffffu, 0u);
  if (cleft > 32 && lane + 32 < cleft) a.cands[2 * (cbase + lane + 32)] = make_uint4(0u, 0u, 0xffffffffu, 0u);
  if (lane == 0) {
    if (c_cand) atomicAdd(&a.cnt[0], (unsigned long long)c_cand);
    if (c_topo) atomicAdd(&a.cnt[1], (unsigned long long)c_topo);
  }
}

// ------------------------------------------------------------------ K4b: evaluate
template <bool PIXEL, bool GATED>
#ifndef K4B_MIN_BLOCKS
#define K4B_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(K4B_THREADS, K4B_MIN_BLOCKS) k_eval(const PhaseArgs a) {
  const unsigned long long n = cta_count(a.prev, a.cand_count);
  if (n == 0) return;
  const int lane = lane_id();
  const int nbx = a.st.nbx, nby = a.st.nby;
  unsigned c_prop = 0, c_srej = 0, c_commit = 0;
  unsigned long long pbase = 0;  // this warp's reserved proposal slots
  int pleft = 0;
  for (unsigned long long base = blockIdx.x * (unsigned long long)K4B_THREADS; base < n;
       base += (unsigned long long)gridDim.x * K4B_THREADS) {  // warp-uniform trip count
    const unsigned long long i = base + threadIdx.x;
    bool prop = false, srej = false;
    int A = 0, Bm = 0, kb = 0, gx = 0, gy = 0, img = 0;
    uint32_t rgb = 0;
    long long d[6] = {0, 0, 0, 0, 0, 0};
    if (i < n) {
      const uint4 e0 = a.cands[2 * i];
      A = (int)e0.z;
      if (A >= 0) {
        const uint4 e1 = a.cands[2 * i + 1];
        const int nq[4] = {(int)e0.w, (int)e1.x, (int)e1.y, (int)e1.z};
        gx = (int)(e0.x & 0xffffu);
        gy = (int)(e0.x >> 16);
        img = (int)e0.y;
        kb = img * a.M;
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
        // distinct candidate labels (A8), all record loads in flight together
        int cb[4];
        int nb = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int B = nq[k];
          bool u = B >= 0 && B != A;
#pragma unroll
          for (int r = 0; r < k; r++) u &= (nq[r] != B);
          if (u) cb[nb++] = B;
        }
        const Rec recA = a.sp.rec[kb + A];
        int4 rn[4];  // first half of each record (means only): 16 B instead of 32
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (k < nb) rn[k] = __ldg(reinterpret_cast<const int4 *>(&a.sp.rec[kb + cb[k]]));
        const RecV ra = rec_vals(recA);
        bool have = false;
        i128 bestE = 0;
        int bestB = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if (k >= nb) break;
          const int B = cb[k];
          long long dB2 = 0;
#pragma unroll
          for (int r = 0; r < 4; r++)
            if (nq[r] >= 0) dB2 += ew[r] * ((long long)(nq[r] != B) - (long long)(nq[r] != A));
          RecV rb;
          rb.c0 = (unsigned)rn[k].z & 0xffffu;
          rb.c1 = (unsigned)rn[k].z >> 16;
          rb.c2 = (unsigned)rn[k].w & 0xffffu;
          rb.mx = rn[k].x;
          rb.my = rn[k].y;
          const i128 E = delta_e(ra, rb, d, 2 * dB2, a.lam_pos, a.lam_b);
          if (!have || E < bestE || (E == bestE && B < bestB)) {
            have = true;
            bestE = E;
            bestB = B;
          }
        }
        if (have && bestE < 0) {
          if (a.size_mode != 0 && ((long long)recA.n - d[0]) * a.l_den < a.l_num * (long long)recA.init) {
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
    c_srej += __popc(__ballot_sync(FULL, srej));
    const unsigned pm = __ballot_sync(FULL, prop);
    c_prop += __popc(pm);
    if (pm) {
      const size_t idx = ((size_t)img * nby + gy) * nbx + gx;
      if (!GATED) {  // size_mode NONE: no budget to check, commit in place
        if (prop) a.st.map[idx] = Bm;
        agg_sums(prop, kb + A, d, true, a.sp.sums, a.sp.dirty);
        agg_sums(prop, kb + Bm, d, false, a.sp.sums, a.sp.dirty);
        c_commit += __popc(pm);
      } else {  // outflow budget, as in k_sweep
        agg_add_i32(prop, kb + A, -(int)d[0], a.sp.out);
        const int np = __popc(pm);
        if (np > pleft) {  // retire the rest of the chunk (sentinels), reserve a new one
          if (lane < pleft) a.props[pbase + lane] = make_uint4(0u, 0xffffffffu, 0u, 0u);
          unsigned long long nb = 0;
          if (lane == 0) nb = atomicAdd(a.prop_count, (unsigned long long)CHUNK);
          pbase = __shfl_sync(FULL, nb, 0);
          pleft = CHUNK;
        }
        if (prop)
          a.props[pbase + __popc(pm & lanemask_lt())] = make_uint4((unsigned)idx, (unsigned)A, (unsigned)Bm, rgb);
        pbase += np;
        pleft -= np;
      }
    }
  }
  if (lane < pleft) a.props[pbase + lane] = make_uint4(0u, 0xffffffffu, 0u, 0u);
  if (lane + 32 < pleft) a.props[pbase + lane + 32] = make_uint4(0u, 0xffffffffu, 0u, 0u);
  if (lane == 0) {
    if (c_prop) atomicAdd(&a.cnt[2], (unsigned long long)c_prop);
    if (c_srej) atomicAdd(&a.cnt[3], (unsigned long long)c_srej);
    if (c_commit) atomicAdd(&a.cnt[4], (unsigned long long)c_commit);
  }
}

// ------------------------------------------------------------------ boundary sets
// bset word (t, c, pr), t = sweep tile (img, ty, tx) of TX x TY blocks, c = cx + 2 cy the phase
// colour, pr = plane row 0..TY/2-1: bit i <-> block (tx*TX + 2i + cx, ty*TY + 2pr + cy).
// Invariant before every phase: each block that is a boundary block (Eq. 2) whose label can
// pass the static gate (active[A] for CLASS/BSP, anything otherwise) has its bit set.  Set
// bits may be stale (the sweep re-tests everything and clears them).
static_assert(TX == 64 && TY == 16, "bset layout assumes 64 x 16 sweep tiles");
constexpr int BSET_WORDS_PER_TILE = 4 * (TY / 2);  // 32

__device__ __forceinline__ uint32_t bset_word(const StageDev &st, int img, int gx, int gy) {
  const uint32_t t = ((uint32_t)img * (uint32_t)st.tiles_y + (uint32_t)(gy >> 4)) * (uint32_t)st.tiles_x +
                     (uint32_t)(gx >> 6);
  return t * BSET_WORDS_PER_TILE + (uint32_t)(((gx & 1) | ((gy & 1) << 1)) * (TY / 2) + ((gy & 15) >> 1));
}
__device__ __forceinline__ void bset_set(uint32_t *bset, const StageDev &st, int img, int gx, int gy) {
  atomicOr(&bset[bset_word(st, img, gx, gy)], 1u << ((gx & 63) >> 1));
}
// the neighbours that a committed move p: A -> B turns into boundary blocks (4-bit mask over
// N, E, S, W): label != B, inside the image, and passing the static gate
__device__ __forceinline__ void bset_insert(uint32_t *bset, const StageDev &st, int img, int gx, int gy,
                                            unsigned ins) {
  if (ins & 1u) bset_set(bset, st, img, gx, gy - 1);
  if (ins & 2u) bset_set(bset, st, img, gx + 1, gy);
  if (ins & 4u) bset_set(bset, st, img, gx, gy + 1);
  if (ins & 8u) bset_set(bset, st, img, gx - 1, gy);
}


// K4 build (once per stage, after the transition): one CTA per sweep tile, thread (r, q) owns
// the 4 blocks gx0+4q .. gx0+4q+3 of row gy0+r; writes all 32 words of the tile.
__global__ void __launch_bounds__(256) k_bset_build(const PhaseArgs a) {
  const StageDev &st = a.st;
  const int nbx = st.nbx, nby = st.nby;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const int r = threadIdx.x >> 4, q = threadIdx.x & 15;
  for (unsigned w = blockIdx.x; w < ntiles; w += gridDim.x) {
    const uint32_t t = a.worklist ? (uint32_t)a.worklist[w] : w;
    const uint32_t rr = fdiv(t, st.fd_tx), img = fdiv(rr, st.fd_ty);
    const int gx0 = (int)(t - rr * (uint32_t)st.tiles_x) * TX, gy0 = (int)(rr - img * (uint32_t)st.tiles_y) * TY;
    const int32_t *map = st.map + (size_t)img * nby * nbx;
    const int gy = gy0 + r, x0 = gx0 + 4 * q;
    const bool row_in = gy < nby;
    int L[4], U[4], D[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int x = x0 + k;
      const bool in = row_in && x < nbx;
      const size_t o = (size_t)gy * nbx + x;
      L[k] = in ? map[o] : -1;
      U[k] = in && gy > 0 ? map[o - nbx] : -1;
      D[k] = in && gy + 1 < nby ? map[o + nbx] : -1;
    }
    int left = __shfl_up_sync(FULL, L[3], 1, 16), right = __shfl_down_sync(FULL, L[0], 1, 16);
    if (q == 0) left = (row_in && x0 > 0 && x0 - 1 < nbx) ? map[(size_t)gy * nbx + x0 - 1] : -1;
    if (q == 15) right = (row_in && x0 + 4 < nbx) ? map[(size_t)gy * nbx + x0 + 4] : -1;
    unsigned s = 0;
    int last = -1;
    bool last_act = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int A = L[k];
      const int Wn = k ? L[k - 1] : left, En = k < 3 ? L[k + 1] : right;
      bool b = A >= 0 && ((U[k] >= 0 && U[k] != A) | (D[k] >= 0 && D[k] != A) | (Wn >= 0 && Wn != A) |
                          (En >= 0 && En != A));
      if (b && a.gating == 1) {
        if (A != last) {
          last = A;
          last_act = a.sp.active[(size_t)img * a.M + A] != 0;
        }
        b = last_act;
      }
      s |= (unsigned)b << k;
    }
    // colour cx = 0: columns 4q, 4q+2 -> bits 2q, 2q+1; cx = 1: columns 4q+1, 4q+3
    unsigned w0 = ((s & 1u) | ((s >> 1) & 2u)) << (2 * q);
    unsigned w1 = (((s >> 1) & 1u) | ((s >> 2) & 2u)) << (2 * q);
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      w0 |= __shfl_xor_sync(FULL, w0, o);
      w1 |= __shfl_xor_sync(FULL, w1, o);
    }
    if (q == 0) {
      const int cy = r & 1;
      uint32_t *tw = a.bset + (size_t)t * BSET_WORDS_PER_TILE + (r >> 1);
      tw[(0 + 2 * cy) * (TY / 2)] = w0;
      tw[(1 + 2 * cy) * (TY / 2)] = w1;
    }
  }
}

// ------------------------------------------------------------------ TMA tile streamer
// Persistent warp-specialised CTAs over the sweep tiles (worklist or all): one producer lane
// streams (TY+2) x (TX+8) label boxes with TMA into an NSTAGE ring (full/empty mbarriers, as
// K4a); 8 consumer warps each take two tile rows, every lane two adjacent columns (one block
// of each column colour).  OP selects the per-stage pass:
//   TILE_BSET  boundary-set build: bit = boundary (Eq. 2) and static gate; a lane's two
//              columns have colours cx = 0, 1, so each row's two words are two ballots.
//   TILE_ADJ   merge adjacency (O7 step 1): boundary blocks of victims add their shared edge
//              lengths to the (victim, neighbour) hash.
constexpr int TILE_BSET = 0, TILE_ADJ = 1;

// The u8 flags of the labels of a lane's two columns (b0/b1: whether each is needed), looked up
// together — at most two independent loads — unless the lane's cached label (keyed by the global
// id: images share local ids) or the other column already has it; the cache keeps the last one.
__device__ __forceinline__ void flag_pair(const uint8_t *flags, bool b0, bool b1, int g0, int g1, int &last,
                                          bool &last_flag, bool &a0, bool &a1) {
  const bool m0 = b0 && g0 != last;
  const bool m1 = b1 && g1 != last && !(m0 && g1 == g0);
  const bool f0 = m0 && flags[g0] != 0, f1 = m1 && flags[g1] != 0;
  a0 = m0 ? f0 : last_flag;
  a1 = m1 ? f1 : ((m0 && g1 == g0) ? a0 : last_flag);
  if (b1) {
    last = g1;
    last_flag = a1;
  } else if (b0) {
    last = g0;
    last_flag = a0;
  }
}

template <int OP>
__global__ void __launch_bounds__(K4A_THREADS) k_tiles(const PhaseArgs a, const MergeArgs ma,
                                                       const __grid_constant__ CUtensorMap tmap) {
  __shared__ __align__(128) int32_t buf[NSTAGE][STAGE_INTS];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];
  __shared__ int4 s_info[NSTAGE];  // gx0, gy0, img, border
  if (OP == TILE_ADJ && *ma.victim_any == 0u) return;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const StageDev &st = a.st;
  const int nbx = st.nbx, nby = st.nby;
  const int tiles_x = st.tiles_x, tiles_y = st.tiles_y;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(tiles_x * tiles_y) * (unsigned)a.B;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; i++) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NWARP) {  // ---- producer
    for (unsigned kb = 0; blockIdx.x + kb * gridDim.x < ntiles; kb += 32) {
      const unsigned wl = blockIdx.x + (kb + lane) * gridDim.x;
      int4 inf = make_int4(0, 0, 0, 0);
      if (wl < ntiles) {
        const uint32_t t = a.worklist ? (uint32_t)a.worklist[wl] : wl;
        const uint32_t r = fdiv(t, st.fd_tx), img = fdiv(r, st.fd_ty);
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
          const int si = (int)(k % NSTAGE);
          if (k >= NSTAGE) mbar_wait(&empty[si], ((k / NSTAGE) - 1) & 1u);
          s_info[si] = v;
          fence_proxy_async();
          mbar_expect_tx(&full[si], TILE_BYTES);
          tma_load_3d(&buf[si][0], &tmap, v.x - HX, v.y - 1, v.z, &full[si]);
        }
        __syncwarp();
      }
    }
    return;
  }
  // ---- consumers: rows 2*warp, 2*warp+1 of the tile; columns 2*lane, 2*lane+1
  int last = -1;
  bool last_flag = false;
  for (unsigned k = 0;; k++) {
    const unsigned w = blockIdx.x + k * gridDim.x;
    if (w >= ntiles) break;
    const int si = (int)(k % NSTAGE);
    mbar_wait(&full[si], (k / NSTAGE) & 1u);
    const int4 inf = s_info[si];
    const int gx0 = inf.x, gy0 = inf.y, img = inf.z;
    int32_t *box = buf[si];
    if (inf.w) {  // TMA zero-fills outside the image; 0 is a label: mark "no block" (-1)
      for (int idx = lane; idx < 4 * BOXW; idx += 32) {
        const int r = idx / BOXW, cc = idx - r * BOXW;
        const int y = gy0 + 2 * warp - 1 + r, x = gx0 + cc - HX;
        if (x < 0 || x >= nbx || y < 0 || y >= nby) box[(2 * warp + r) * BOXW + cc] = -1;
      }
      __syncwarp();
    }
    const int kb = img * a.M;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int rr = 2 * warp + h;  // tile row
      const int32_t *up = box + rr * BOXW + HX, *mid = up + BOXW, *dn = mid + BOXW;
      const int2 U = *reinterpret_cast<const int2 *>(up + 2 * lane);
      const int2 Mv = *reinterpret_cast<const int2 *>(mid + 2 * lane);
      const int2 D = *reinterpret_cast<const int2 *>(dn + 2 * lane);
      const int Wn = mid[2 * lane - 1], En = mid[2 * lane + 2];
      const int L[2] = {Mv.x, Mv.y}, N[2] = {U.x, U.y}, S[2] = {D.x, D.y}, Wv[2] = {Wn, Mv.x}, Ev[2] = {Mv.y, En};
      bool bnd[2];
      if (!inf.w) {  // interior tile (warp-uniform): no "no block" marks in the box
#pragma unroll
        for (int c = 0; c < 2; c++)
          bnd[c] = (N[c] != L[c]) | (S[c] != L[c]) | (Wv[c] != L[c]) | (Ev[c] != L[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 2; c++)
          bnd[c] = L[c] >= 0 && ((N[c] >= 0 && N[c] != L[c]) | (S[c] >= 0 && S[c] != L[c]) |
                                 (Wv[c] >= 0 && Wv[c] != L[c]) | (Ev[c] >= 0 && Ev[c] != L[c]));
      }
      if (OP == TILE_BSET) {
        bool bit[2] = {bnd[0], bnd[1]};
        if (a.gating == 1) {  // static gate: the labels' active flags
          bool a0, a1;
          flag_pair(a.sp.active, bnd[0], bnd[1], kb + L[0], kb + L[1], last, last_flag, a0, a1);
          bit[0] = bnd[0] && a0;
          bit[1] = bnd[1] && a1;
        }
        const unsigned w0 = __ballot_sync(FULL, bit[0]), w1 = __ballot_sync(FULL, bit[1]);
        if (lane == 0) {
          const uint32_t tile = ((uint32_t)img * (uint32_t)tiles_y + (uint32_t)(gy0 / TY)) * (uint32_t)tiles_x +
                                (uint32_t)(gx0 / TX);
          uint32_t *tw = a.bset + (size_t)tile * BSET_WORDS_PER_TILE + (rr >> 1);
          tw[(0 + 2 * (rr & 1)) * (TY / 2)] = w0;
          tw[(1 + 2 * (rr & 1)) * (TY / 2)] = w1;
        }
      } else {  // TILE_ADJ
        const int gy = gy0 + rr;
        bool vic[2];  // the labels' victim flags
        flag_pair(ma.sp.victim, bnd[0], bnd[1], kb + L[0], kb + L[1], last, last_flag, vic[0], vic[1]);
#pragma unroll
        for (int c = 0; c < 2; c++) {
          if (!bnd[c] || !vic[c]) continue;
          const int gx = gx0 + 2 * lane + c;
          const unsigned ew = (unsigned)(st.xs[gx + 1] - st.xs[gx]), eh = (unsigned)(st.ys[gy + 1] - st.ys[gy]);
          const int nq[4] = {N[c], Ev[c], S[c], Wv[c]};
#pragma unroll
          for (int d = 0; d < 4; d++)
            if (nq[d] >= 0 && nq[d] != L[c]) hash_add(ma, kb + L[c], kb + nq[d], (d & 1) ? eh : ew);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[si]);
  }
}

// lam * v exactly, for 0 <= lam < 2^31 and any int64 v: two 32 x 32 -> 64 products
__device__ __forceinline__ i128 mul_u31_s64(long long lam, long long v) {
  const unsigned long long p0 = (unsigned long long)(uint32_t)lam * (uint32_t)v;  // IMAD.WIDE.U32
  const long long p1 = (long long)(int32_t)lam * (int32_t)(v >> 32);               // IMAD.WIDE
  return ((i128)p1 << 32) + (i128)p0;
}

// 2^(-16) x the oracle's weighted dE of relabelling the block (data d) from A to the label of
// record rb: E = X * 2^16 + lam_pos * dP with X = colour part + lam_b * dB2 (exact in int64)
// and dP the position part (exact in int64).  At the pixel stage (n = 1, values
// < 2^8, coordinates < 2^16) every factor fits 32 bits, so each product is one IMAD.WIDE.
template <bool PIXEL, bool SMALLB = false>
__device__ __forceinline__ i128 energy(const Rec &ra, const int4 rb, const int d[6], long long dB2,
                                       long long lam_pos, long long lam_b) {
  const int cA0 = (int)(ra.cq01 & 0xffffu), cA1 = (int)(ra.cq01 >> 16), cA2 = (int)(ra.cq2f & 0xffffu);
  const int cB0 = (int)((unsigned)rb.z & 0xffffu), cB1 = (int)((unsigned)rb.z >> 16);
  const int cB2 = (int)((unsigned)rb.w & 0xffffu);
  long long X, dP;
  if (PIXEL) {
    X = (long long)(cB0 - cA0) * (cB0 + cA0 - (d[1] << (FRAC + 1))) +
        (long long)(cB1 - cA1) * (cB1 + cA1 - (d[2] << (FRAC + 1))) +
        (long long)(cB2 - cA2) * (cB2 + cA2 - (d[3] << (FRAC + 1))) + (long long)(int)lam_b * (int)dB2;
    dP = (long long)(rb.x - ra.mux) * (rb.x + ra.mux - (d[4] << (FRAC + 1))) +
         (long long)(rb.y - ra.muy) * (rb.y + ra.muy - (d[5] << (FRAC + 1)));
  } else {
    // n <= 4096 and sums < 2^21 (b <= 64): the colour factors fit 32 bits, the position
    // factors need 64 (n * (mB + mA) < 2^37)
    const int n = d[0];
    X = (long long)(cB0 - cA0) * (n * (cB0 + cA0) - (d[1] << (FRAC + 1))) +
        (long long)(cB1 - cA1) * (n * (cB1 + cA1) - (d[2] << (FRAC + 1))) +
        (long long)(cB2 - cA2) * (n * (cB2 + cA2) - (d[3] << (FRAC + 1))) + lam_b * dB2;
    if (SMALLB) {
      // n * max coordinate < 2^22 (checked per stage on the host): |n (mB + mA) - 2^9 sum| < 2^31,
      // so each position product is one 32 x 32 -> 64 IMAD.WIDE as at the pixel stage
      dP = (long long)(rb.x - ra.mux) * (n * (rb.x + ra.mux) - (d[4] << (FRAC + 1))) +
           (long long)(rb.y - ra.muy) * (n * (rb.y + ra.muy) - (d[5] << (FRAC + 1)));
    } else {
      dP = (long long)(rb.x - ra.mux) * ((long long)n * ((long long)rb.x + ra.mux) - ((long long)d[4] << (FRAC + 1))) +
           (long long)(rb.y - ra.muy) * ((long long)n * ((long long)rb.y + ra.muy) - ((long long)d[5] << (FRAC + 1)));
    }
  }
  return ((i128)X << 16) + mul_u31_s64(lam_pos, dP);
}

// K4 sweep (fused scan + evaluate, one launch per phase): warps stride over groups of 4 sweep
// tiles; lane l loads bset word (tile l/8, colour c, plane row l%8), the set bits are
// distributed 32 at a time over the lanes, and every lane re-tests its block from the label
// map (boundary, static gate, simple point, Eq. 7), then evaluates Eqs. 1-3 as K4b does.
// UNI: the stage is uniform (every block b x b at (gx b, gy b)) at compile time — the block
// geometry folds into st.b and the table path is not compiled (fewer live registers)
template <bool PIXEL, bool GATED, int MINB, bool SMALLB = false, bool LIST = false, bool UNI = false>
__global__ void __launch_bounds__(K4B_THREADS, MINB) k_sweep(const PhaseArgs a) {
  pdl_wait_and_trigger();
  if (sweep_skipped(a.prev)) return;
  const int lane = lane_id();
  const StageDev &st = a.st;
  const int nbx = st.nbx, nby = st.nby;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  // words per warp iteration (4..32, power of 2): the largest giving every warp gpw groups of
  // the (device-side) worklist; larger groups fill the rounds better and take fewer of the
  // queue's same-address atomics (measured: gpw 2 best at config 4)
  unsigned G = 32;
  while (G > 4 && ntiles * (TY / 2) / G < (unsigned)a.gpw * nw) G >>= 1;
  // the last tail_pct % of the words go out in groups of G/4 (>= 4): a shorter tail when the
  // queue runs dry (the kernel ends with its slowest warp)
  const unsigned nwords = ntiles * (TY / 2);
  const unsigned Gt = G >= 16 ? G / 4 : 4;
  const unsigned nhead = (unsigned)(((unsigned long long)nwords * (100u - (unsigned)a.tail_pct) / 100u) / G);
  const unsigned head_words = nhead * G;
  const unsigned ngroups = nhead + (nwords - head_words + Gt - 1) / Gt;
  const int colour = a.cx | (a.cy << 1);
  __shared__ unsigned s_cnt[5];  // cand, topo, prop, srej, commit (per CTA; flushed at the end)
  __shared__ uint32_t s_simple[8];  // 256-bit truth table of simple_point (E_topo) by ring mask
  if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0u;
  {
    static_assert(K4B_THREADS == 256, "one thread per ring mask");
    const unsigned t = __ballot_sync(FULL, simple_point(threadIdx.x));
    if ((threadIdx.x & 31) == 0) s_simple[threadIdx.x >> 5] = t;
  }
  __syncthreads();
  unsigned long long pbase = 0;  // this warp's reserved proposal slots
  int pleft = 0;
  unsigned r_cand = 0, r_topo = 0, r_prop = 0, r_srej = 0, r_commit = 0;  // this warp's counters
  // one round: every lane tests (have) the block of bit r of word wj (bit 0 of a one-bit word in
  // LIST mode) at plane position pj = (x of bit 0) | (y << 16) and evaluates it (Eqs. 1-3)
  auto round = [&](const bool have, const int img, const uint32_t xj, const uint32_t wj, const unsigned r,
                   const uint32_t pj) {
      bool cand = false, emit = false, prop = false, srej = false;
      int A = 0, Bm = 0, kb = img * a.M, gx = 0, gy = 0;
      unsigned ins = 0;
      uint32_t rgb = 0;
      int d[6] = {0, 0, 0, 0, 0, 0};  // block data: n, colour sums, position sums (all < 2^31)
      if (have) {
        const unsigned bit = nth_set_bit(wj, r);
        gx = (int)(pj & 0xffffu) + 2 * (int)bit;
        gy = (int)(pj >> 16);
        // block data depends on the position only: issued together with the window loads
        // (kept raw until it is needed, so that no use of it waits before the window loads go out)
        uint32_t pk32 = 0;
        uint64_t pk64 = 0;
        int bx0 = 0, bw = 1, by0 = 0, bh = 1;
        if (PIXEL) {
          const uint8_t *p = a.image + (((size_t)img * a.H + gy) * a.W + gx) * 3;
#if RAPID_RGB2
          // the 3 bytes from the aligned word holding the first and, when they cross into it,
          // the next one (2 loads at most instead of 3; never a byte outside those words)
          const uint32_t *pw = reinterpret_cast<const uint32_t *>((uintptr_t)p & ~(uintptr_t)3);
          const unsigned sh = (unsigned)((uintptr_t)p & 3u) * 8u;
          const uint32_t w0 = ld_stream64(pw), w1 = sh > 8u ? ld_stream64(pw + 1) : 0u;
          rgb = __funnelshift_r(w0, w1, sh) & 0xffffffu;
#else
          rgb = ld_stream64(p) | (ld_stream64(p + 1) << 8) | (ld_stream64(p + 2) << 16);
#endif
        } else {
          const size_t bi = ((size_t)img * nby + gy) * nbx + gx;
          if (st.bsum32) pk32 = ld_stream64(reinterpret_cast<const uint32_t *>(st.bsum) + bi);
          else pk64 = ld_stream64(reinterpret_cast<const unsigned long long *>(st.bsum) + bi);
          if (UNI) {
            // geometry formed where it is used (below): nothing held across the loads
          } else if (st.uniform) {  // every block b x b at (gx b, gy b): no geometry-table loads
            bx0 = gx * st.b;
            by0 = gy * st.b;
            bw = bh = st.b;
          } else {
            bx0 = st.xs[gx]; bw = st.xs[gx + 1] - bx0;
            by0 = st.ys[gy]; bh = st.ys[gy + 1] - by0;
          }
        }
        const int32_t *m = st.map + (size_t)img * nby * nbx;
        const size_t o = (size_t)gy * nbx + gx;
        const bool hN = gy > 0, hS = gy + 1 < nby, hW = gx > 0, hE = gx + 1 < nbx;
        // streaming loads (evict-first, 64-B DRAM fill): keep L2 for the per-superpixel tables
#ifndef RAPID_RGB2
#define RAPID_RGB2 1  // measured: pixel-stage K4 3.61 -> 3.58 ms per step
#endif
#ifndef RAPID_WLD
#define RAPID_WLD ld_stream64
#endif
        A = RAPID_WLD(m + o);
        const int nq0 = hN ? RAPID_WLD(m + o - nbx) : -1, nq1 = hE ? RAPID_WLD(m + o + 1) : -1;
        const int nq2 = hS ? RAPID_WLD(m + o + nbx) : -1, nq3 = hW ? RAPID_WLD(m + o - 1) : -1;
        const int dNE = hN && hE ? RAPID_WLD(m + o - nbx + 1) : -1, dSE = hS && hE ? RAPID_WLD(m + o + nbx + 1) : -1;
        const int dSW = hS && hW ? RAPID_WLD(m + o + nbx - 1) : -1, dNW = hN && hW ? RAPID_WLD(m + o - nbx - 1) : -1;
        const int nq[4] = {nq0, nq1, nq2, nq3};
        // topology (E_topo) and the distinct candidate labels need only the window; the
        // records of A and of the candidates are then loaded together (one dependent L2
        // round trip instead of two)
        const unsigned m8 = (unsigned)(nq0 == A) | ((unsigned)(dNE == A) << 1) | ((unsigned)(nq1 == A) << 2) |
                            ((unsigned)(dSE == A) << 3) | ((unsigned)(nq2 == A) << 4) |
                            ((unsigned)(dSW == A) << 5) | ((unsigned)(nq3 == A) << 6) |
                            ((unsigned)(dNW == A) << 7);
        const bool topo_ok = (s_simple[m8 >> 5] >> (m8 & 31u)) & 1u;
        // distinct candidate labels (A8), compacted: cb[0..nb) with the slot mask cm of each;
        // maskA = slots labelled A.  (Compaction keeps the candidate loop below SIMD-coherent:
        // every lane's first candidate is evaluated in the same iteration.)
        const unsigned maskA = (m8 & 1u) | ((m8 >> 1) & 2u) | ((m8 >> 2) & 4u) | ((m8 >> 3) & 8u);
        const bool bnd = (nq0 >= 0 && nq0 != A) | (nq1 >= 0 && nq1 != A) | (nq2 >= 0 && nq2 != A) |
                         (nq3 >= 0 && nq3 != A);
        int cb[4] = {0, 0, 0, 0};
        unsigned cm[4] = {0u, 0u, 0u, 0u};
        int nb = 0;
#pragma unroll
        for (int s = 0; s < 4; s++) {
          const int L = nq[s];
          if (L < 0 || L == A) continue;
          bool found = false;
#pragma unroll
          for (int r = 0; r < s; r++)
            if (r < nb && cb[r] == L) {
              cm[r] |= 1u << s;
              found = true;
            }
          if (!found) {
#pragma unroll
            for (int r = 0; r <= s; r++)
              if (r == nb) {
                cb[r] = L;
                cm[r] = 1u << s;
              }
            nb++;
          }
        }
        Rec recA;
        int4 rn[4];
        const bool need_rn = bnd && (topo_ok || a.gating == 2);
        if (bnd) recA = ldnc64_rec(&a.sp.rec[kb + A]);
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++)
          rn[k2] = (need_rn && k2 < nb) ? ldnc64_v4(&a.sp.rec[kb + cb[k2]]) : make_int4(0, 0, 0, 0);
        bool keep = bnd;
        if (bnd && a.gating == 1) keep = ((recA.cq2f >> 16) & F_ACTIVE) != 0u;
        if (!keep) {
          atomicAnd(&a.bset[xj], ~(1u << bit));  // stale: no longer a gated boundary block
        } else {
          cand = true;
          if (a.gating == 2) {  // Eq. 7: a neighbour of another label and another class
            const unsigned yA = (recA.cq2f >> 18) & 3u;
            bool e7 = false;
#pragma unroll
            for (int k2 = 0; k2 < 4; k2++)
              if (k2 < nb) e7 |= ((((unsigned)rn[k2].w >> 18) & 3u) != yA);
            cand = e7;
          }
          emit = cand && topo_ok;
          if (emit) {
            if (PIXEL) {
              d[0] = 1; d[1] = rgb & 0xffu; d[2] = (rgb >> 8) & 0xffu; d[3] = rgb >> 16; d[4] = gx; d[5] = gy;
            } else {
              const uint64_t pk = st.bsum32 ? widen_bsum32(pk32) : pk64;
              if (UNI) { bx0 = gx * st.b; by0 = gy * st.b; bw = bh = st.b; }
              d[0] = bw * bh;
              d[1] = (int)(pk & 0x1FFFFFull);
              d[2] = (int)((pk >> 21) & 0x1FFFFFull);
              d[3] = (int)(pk >> 42);
              d[4] = bh * ((bw * (2 * bx0 + bw - 1)) / 2);
              d[5] = bw * ((bh * (2 * by0 + bh - 1)) / 2);
            }
            // E_b weight of the slots in a mask: N (1), S (4) edges have length bw; E (2), W (8) bh
            auto wsum = [&](unsigned msk) -> int {
              return PIXEL ? __popc(msk) : UNI ? st.b * __popc(msk) : bw * __popc(msk & 5u) + bh * __popc(msk & 10u);
            };
            const int wA = wsum(maskA);
            bool hv = false;
            i128 bestE = 0;
            int bestB = 0;
#pragma unroll
            for (int k2 = 0; k2 < 4; k2++) {
              if (k2 >= nb) break;
              const int B = cb[k2];
              const i128 E = energy<PIXEL, SMALLB>(recA, rn[k2], d, 2ll * (wA - wsum(cm[k2])), a.lam_pos, a.lam_b);
              if (!hv || E < bestE || (E == bestE && B < bestB)) {
                hv = true;
                bestE = E;
                bestB = B;
              }
            }
            if (hv && bestE < 0) {
              if (GATED && ((long long)recA.n - d[0]) * a.l_den < a.l_num * (long long)recA.init) {
                srej = true;  // A12: the desired move would leave A below l * InitSize
                if (a.size_mode == 2) a.sp.victim[kb + A] = 1;  // (victim_any: once per warp below)
              } else {
                prop = true;
                Bm = bestB;
                // neighbours whose boundary-set bit the move may have to set: only those labelled
                // A (they now touch B); a neighbour of another label C != B already touched p's
                // A, so it was a boundary block and its bit is set (invariant; A passed the gate
                // and C's bit is needed only if C does).  An A-neighbour q is skipped too when a
                // diagonal of p — q's other 4-neighbour across the row or column, a colour that
                // does not move in this phase — holds another label: q was already a boundary block.
                const bool oNE = dNE >= 0 && dNE != A, oSE = dSE >= 0 && dSE != A;
                const bool oSW = dSW >= 0 && dSW != A, oNW = dNW >= 0 && dNW != A;
                const unsigned known = ((unsigned)(oNW | oNE)) | ((unsigned)(oNE | oSE) << 1) |
                                       ((unsigned)(oSW | oSE) << 2) | ((unsigned)(oNW | oSW) << 3);
                ins = maskA & ~known;
              }
            }
          }
        }
      }
      r_cand += __popc(__ballot_sync(FULL, cand));  // warp-uniform running counts
      r_topo += __popc(__ballot_sync(FULL, emit));
      {
        const unsigned bs = __ballot_sync(FULL, srej);
        r_srej += __popc(bs);
        // one store per warp round to the stage's victim flag (a store by every rejecting lane
        // serialises on the one address)
        if (bs && a.size_mode == 2 && lane == 0) *a.victim_any = 1u;
      }
      const unsigned pm = __ballot_sync(FULL, prop);
      r_prop += __popc(pm);
      if (pm) {
        const size_t idx = ((size_t)img * nby + gy) * nbx + gx;
        if (!GATED) {  // size_mode NONE: no budget to check, commit in place
          if (prop) {
            st.map[idx] = Bm;
            bset_insert(a.bset, st, img, gx, gy, ins);
          }
          const long long dl[6] = {d[0], d[1], d[2], d[3], d[4], d[5]};
          if (PIXEL || st.b <= 4) {  // warp-uniform
            agg_sums_small(prop, kb + A, dl, true, a.sp.sums, a.sp.dirty);
            agg_sums_small(prop, kb + Bm, dl, false, a.sp.sums, a.sp.dirty);
          } else {
            agg_sums(prop, kb + A, dl, true, a.sp.sums, a.sp.dirty);
            agg_sums(prop, kb + Bm, dl, false, a.sp.sums, a.sp.dirty);
          }
          r_commit += __popc(pm);
        } else {
          // HARD / MERGE: A's outflow is subtracted from its budget rem[A]; K5 applies A's moves
          // iff rem[A] >= 0 afterwards (all-or-nothing, A19)
          agg_add_i32(prop, kb + A, -(int)d[0], a.sp.out);
          const int np = __popc(pm);
          if (np > pleft) {  // retire the rest of the chunk (sentinels), reserve a new one
            if (lane < pleft) a.props[pbase + lane] = make_uint4(0u, 0xffffffffu, 0u, 0u);
            unsigned long long nb = 0;
            if (lane == 0) nb = atomicAdd(a.prop_count, (unsigned long long)CHUNK);
            pbase = __shfl_sync(FULL, nb, 0);
            pleft = CHUNK;
          }
          if (prop)
            a.props[pbase + __popc(pm & lanemask_lt())] =
                make_uint4((unsigned)idx, (unsigned)A, (unsigned)Bm, rgb | (ins << 24));
          pbase += np;
          pleft -= np;
        }
      }
  };
  auto deal_groups = [&]() {
  // dynamic distribution of the word groups (one returned atomic per group and warp): the
  // per-group work varies with the boundary density, static striding left a 10 % tail
  for (unsigned g = 0;;) {
    if (lane == 0) g = atomicAdd(a.wq, 1u);
    g = __shfl_sync(FULL, g, 0);
    if (g >= ngroups) break;
    // ---- this lane's word
    const unsigned gsz = g < nhead ? G : Gt;
    const unsigned q = (g < nhead ? g * G : head_words + (g - nhead) * Gt) + (unsigned)lane, w = q >> 3;  // (tile slot, plane row q % 8)
    uint32_t word = 0, wpos = 0, widx = 0;
    int wimg = 0;
    if ((unsigned)lane < gsz && w < ntiles) {
      const uint32_t t = a.worklist ? (uint32_t)a.worklist[w] : w;
      const uint32_t rr = fdiv(t, st.fd_tx), img = fdiv(rr, st.fd_ty);
      const int gx0 = (int)(t - rr * (uint32_t)st.tiles_x) * TX, gy0 = (int)(rr - img * (uint32_t)st.tiles_y) * TY;
      widx = t * BSET_WORDS_PER_TILE + (uint32_t)(colour * (TY / 2) + (q & 7));
      word = ld64_u32(a.bset + widx);  // 64-B fill: the phase needs 32 B of the tile's 128
      wpos = (uint32_t)(gx0 + a.cx) | ((uint32_t)(gy0 + 2 * (q & 7) + a.cy) << 16);
      wimg = (int)img;
    }
    const unsigned cw = __popc(word);
    unsigned incl = cw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned total = __shfl_sync(FULL, incl, 31);
    for (unsigned rb = 0; rb < total; rb += 32) {
      const unsigned k = rb + lane;
      int j = 0;  // the lane whose word holds candidate k: #lanes with incl <= k
#pragma unroll
      for (int h = 16; h > 0; h >>= 1) {
        const unsigned v = __shfl_sync(FULL, incl, j + h - 1);
        if (v <= k) j += h;
      }
      const uint32_t wj = __shfl_sync(FULL, word, j);
      const unsigned ej = __shfl_sync(FULL, incl, j) - __popc(wj);
      const uint32_t pj = __shfl_sync(FULL, wpos, j);
      const uint32_t xj = __shfl_sync(FULL, widx, j);
      const int img = __shfl_sync(FULL, wimg, j);
      round(k < total, img, xj, wj, k - ej, pj);
    }
  }
  };
  if constexpr (LIST) {
    // the phase's set bits compacted into a.list by k_bset_list (one entry per bit: word index
    // << 5 | bit): every round is 32 candidates, no dealing; static striding (the rounds cost
    // about the same)
    const unsigned n = *a.list_count;
    for (unsigned base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; base < n; base += nw * 32u) {
      const unsigned i = base + (unsigned)lane;
      uint32_t e = 0, xj = 0, pj = 0;
      int img = 0;
      if (i < n) {
        e = a.list[i];
        xj = e >> 5;
        const uint32_t t = xj / BSET_WORDS_PER_TILE, q = xj & 7u;
        const uint32_t rr = fdiv(t, st.fd_tx), im = fdiv(rr, st.fd_ty);
        const int gx0 = (int)(t - rr * (uint32_t)st.tiles_x) * TX, gy0 = (int)(rr - im * (uint32_t)st.tiles_y) * TY;
        pj = (uint32_t)(gx0 + a.cx) | ((uint32_t)(gy0 + 2 * (int)q + a.cy) << 16);
        img = (int)im;
      }
      round(i < n, img, xj, 1u << (e & 31u), 0u, pj);
    }
  } else {
    deal_groups();
  }
  if (GATED) {
    if (lane < pleft) a.props[pbase + lane] = make_uint4(0u, 0xffffffffu, 0u, 0u);
    if (lane + 32 < pleft) a.props[pbase + lane + 32] = make_uint4(0u, 0xffffffffu, 0u, 0u);
  }
  if (lane == 0) {
    if (r_cand) atomicAdd(&s_cnt[0], r_cand);
    if (r_topo) atomicAdd(&s_cnt[1], r_topo);
    if (r_prop) atomicAdd(&s_cnt[2], r_prop);
    if (r_srej) atomicAdd(&s_cnt[3], r_srej);
    if (r_commit) atomicAdd(&s_cnt[4], r_commit);
  }
  __syncthreads();
  if (threadIdx.x < 5 && s_cnt[threadIdx.x]) atomicAdd(&a.cnt[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// Per-phase candidate list of a block stage (k_sweep's LIST mode): every set bit of the phase
// colour's boundary-set words of the worklist tiles as (word index << 5 | bit), compacted with
// one returned atomic per warp.  The order is irrelevant: K4's decisions, K5's all-or-nothing
// budgets and the integer atomics do not depend on it.
__global__ void __launch_bounds__(256) k_bset_list(const PhaseArgs a) {
  pdl_wait_and_trigger();
  if (sweep_skipped(a.prev)) return;
  const StageDev &st = a.st;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const unsigned nwords = ntiles * (TY / 2);
  const int colour = a.cx | (a.cy << 1);
  const int lane = lane_id();
  for (unsigned base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < nwords; base += gridDim.x * blockDim.x) {
    const unsigned q = base + (unsigned)lane;
    uint32_t word = 0, widx = 0;
    if (q < nwords) {
      const unsigned w = q >> 3;
      const uint32_t t = a.worklist ? (uint32_t)a.worklist[w] : w;
      widx = t * BSET_WORDS_PER_TILE + (uint32_t)(colour * (TY / 2) + (q & 7));
      word = a.bset[widx];
    }
    unsigned incl = __popc(word);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned total = __shfl_sync(FULL, incl, 31);
    if (total == 0u) continue;  // warp-uniform
    unsigned off = 0;
    if (lane == 31) off = atomicAdd(a.list_count, total);
    off = __shfl_sync(FULL, off, 31) + incl - __popc(word);
    while (word) {
      const uint32_t b = (uint32_t)__ffs(word) - 1u;
      word &= word - 1u;
      a.list[off++] = (widx << 5) | b;
    }
  }
}

// ------------------------------------------------------------------ K5: commit
// O6' (A19): the proposals of source A commit iff A's total outflow fits its budget, i.e. iff
// rem[A] >= 0 after K4 subtracted every proposal of A (all-or-nothing; one 4-B gather from the
// small budget table per proposal).  Accepted moves are applied here: label, boundary-set bits,
// warp-aggregated sums; a rejected source is marked dirty (its budget is restored next phase).
// SNAP (cooperative launch, every CTA resident): after a grid barrier the same CTAs refresh the
// records marked dirty in this phase (K3 of the next phase / of the stage end, without a launch)
template <bool PIXEL, bool SNAP>
__global__ void __launch_bounds__(256, 8) k_commit(const PhaseArgs a) {  // 8 CTAs/SM: the grid is one wave
  pdl_wait_and_trigger();
  const unsigned long long n = cta_count(a.prev, a.prop_count, !SNAP);
  if (n == 0) return;  // SNAP: grid-uniform (an empty list marks nothing to refresh)
  // packed deltas (3 REDs per aggregated run instead of 6) while every snapshot size is within
  // the stage's limit: then no field of a superpixel's phase total leaves int32
  unsigned long long *const ds = (a.sp.dsum != nullptr && *a.sp.big == 0u) ? a.sp.dsum : nullptr;
  unsigned c_commit = 0, c_rej = 0;
  for (unsigned long long base = blockIdx.x * 256ull; base < n; base += gridDim.x * 256ull) {
    const unsigned long long i = base + threadIdx.x;
    const bool valid = i < n;
    bool ok = false, rej = false;
    int A = 0, B = 0, kb = 0;
    long long d[6] = {0, 0, 0, 0, 0, 0};
    const uint4 pr = valid ? a.props[i] : make_uint4(0u, 0xffffffffu, 0u, 0u);
    if (pr.y != 0xffffffffu) {  // skip unused reserved slots
      A = (int)pr.y;
      B = (int)pr.z;
      const int img = (int)fdivu(pr.x, a.st.fd_nper);
      const uint32_t r = pr.x - (uint32_t)img * a.st.fd_nper.d;
      const int gy = (int)fdivu(r, a.st.fd_nbx), gx = (int)(r - (uint32_t)gy * (uint32_t)a.st.nbx);
      kb = img * a.M;
      // the block's data (loads at block stages) is issued with the budget load
      if (PIXEL) {
        d[0] = 1; d[1] = pr.w & 0xffu; d[2] = (pr.w >> 8) & 0xffu; d[3] = (pr.w >> 16) & 0xffu;
        d[4] = gx; d[5] = gy;
      } else {
        block_data_blk(a.st, img, gx, gy, d);
      }
      ok = (int)ldnc64_u32(&a.sp.out[kb + A]) >= 0;
      if (ok) {
        a.st.map[pr.x] = B;
        if (a.bset) bset_insert(a.bset, a.st, img, gx, gy, pr.w >> 24);
      } else {
        rej = true;
        for (int f = 0; f < 6; f++) d[f] = 0;
        mark_dirty(a.sp.dirty, kb + A);  // so that the next K3 restores rem[A] (and re-derives A's record)
        if (a.size_mode == 2) a.sp.victim[kb + A] = 1;
      }
    }
    if (a.size_mode == 2 && __ballot_sync(FULL, rej) && lane_id() == 0) *a.victim_any = 1u;  // once per warp
    if (PIXEL || a.st.b <= 4) {  // warp-uniform
      agg_sums_small(ok, kb + A, d, true, a.sp.sums, a.sp.dirty, ds);
      agg_sums_small(ok, kb + B, d, false, a.sp.sums, a.sp.dirty, ds);
    } else {
      agg_sums(ok, kb + A, d, true, a.sp.sums, a.sp.dirty, ds);
      agg_sums(ok, kb + B, d, false, a.sp.sums, a.sp.dirty, ds);
    }
    c_commit += __popc(__ballot_sync(FULL, ok));
    c_rej += __popc(__ballot_sync(FULL, rej));
  }
  if (lane_id() == 0) {
    if (c_commit) atomicAdd(&a.cnt[4], (unsigned long long)c_commit);
    if (c_rej) atomicAdd(&a.cnt[5], (unsigned long long)c_rej);
  }
  if (SNAP) {  // n is grid-uniform (cta_count per_cta = false): every CTA gets here or none did
    cg::this_grid().sync();
    const SnapArgs sa{a.sp, a.B * a.M, a.stamp, a.l_num, a.l_den};
    snapshot_warps(sa, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
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
  // L2 promotion: the 288-B box rows straddle 256-B granules, so 256-B promotion over-fetches
  // (RAPID_TMA_PROMO=0/64/128/256 for A/B; default 64)
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  if (const char *e = getenv("RAPID_TMA_PROMO")) {
    const int v = atoi(e);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
          : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)nbx, (cuuint64_t)nby, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)nbx * 4, (cuuint64_t)nbx * nby * 4};
  const cuuint32_t box[3] = {(cuuint32_t)BOXW, (cuuint32_t)BOXH, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode((CUtensorMap *)tmap64B, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, base, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


int scan_occupancy() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_scan<true>, K4A_THREADS, 0);
  return nb < 1 ? 1 : nb;
}

int eval_occupancy() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_eval<true, true>, K4B_THREADS, 0);
  return nb < 1 ? 1 : nb;
}

void launch_scan(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s) {
  static CUtensorMap dummy;
  if (tmap) k_scan<true><<<grid, K4A_THREADS, 0, s>>>(a, *(const CUtensorMap *)tmap);
  else k_scan<false><<<grid, K4A_THREADS, 0, s>>>(a, dummy);
}

void launch_eval(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s) {
  const bool gated = a.size_mode != 0;
  if (pixel && gated) k_eval<true, true><<<grid, K4B_THREADS, 0, s>>>(a);
  else if (pixel) k_eval<true, false><<<grid, K4B_THREADS, 0, s>>>(a);
  else if (gated) k_eval<false, true><<<grid, K4B_THREADS, 0, s>>>(a);
  else k_eval<false, false><<<grid, K4B_THREADS, 0, s>>>(a);
}

// Register budget per variant (measured): the pixel stage runs best at 4 CTAs/SM (64
// registers), the block stages at 3 (80; their 64-bit position sums spill at 64).
// RAPID_SWEEP_MINB=2..4 forces one budget for every stage (A/B testing).
static int g_sweep_minb = 0;
bool g_pdl = false;  // RAPID_PDL=1: programmatic dependent launch of the phase-loop kernels
int g_sweep_uni = 1;  // RAPID_SWEEP_UNI=0: uniform block stages take the runtime-geometry K4 variant
static int g_sweep_minb_small = 4;  // RAPID_SWEEP_MINB_SMALL: CTAs/SM of the small-block variant (4: 64 registers, a few bytes of spill, -0.1 ms)

template <int MB>
static int sweep_occ() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep<true, true, MB>, K4B_THREADS, 0);
  return nb < 1 ? 1 : nb;
}

int sweep_occupancy() {
  const char *e = getenv("RAPID_SWEEP_MINB");
  if (e && e[0] >= '2' && e[0] <= '4') g_sweep_minb = e[0] - '0';
  const char *es = getenv("RAPID_SWEEP_MINB_SMALL");
  if (es && es[0] >= '2' && es[0] <= '4') g_sweep_minb_small = es[0] - '0';
  return g_sweep_minb == 2 ? sweep_occ<2>() : g_sweep_minb == 3 ? sweep_occ<3>() : sweep_occ<4>();
}

void launch_bset_build(const PhaseArgs &a, const void *tmap, int grid, cudaStream_t s) {
  if (tmap) {
    MergeArgs none{};
    k_tiles<TILE_BSET><<<grid, K4A_THREADS, 0, s>>>(a, none, *(const CUtensorMap *)tmap);
  } else {
    k_bset_build<<<grid, 256, 0, s>>>(a);
  }
}

int tiles_occupancy() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tiles<TILE_ADJ>, K4A_THREADS, 0);
  return nb < 1 ? 1 : nb;
}

bool launch_merge_adjacency_tma(const MergeArgs &m, const void *tmap, int grid, cudaStream_t s) {
  if (!tmap) return false;
  PhaseArgs a{};
  a.st = m.st;
  a.sp = m.sp;
  a.B = m.B;
  a.M = m.M;
  a.worklist = m.worklist;
  a.nwork = m.nwork;
  k_tiles<TILE_ADJ><<<grid, K4A_THREADS, 0, s>>>(a, m, *(const CUtensorMap *)tmap);
  return true;
}

void launch_sweep(const PhaseArgs &a, bool pixel, bool smallb, bool list, int sm_count, cudaStream_t s) {
  const bool gated = a.size_mode != 0;
  static int occ[5] = {0, 0, 0, 0, 0};
  const int mb = g_sweep_minb ? g_sweep_minb : (pixel ? 4 : smallb ? g_sweep_minb_small : 3);
  if (!occ[mb]) occ[mb] = mb == 2 ? sweep_occ<2>() : mb == 3 ? sweep_occ<3>() : sweep_occ<4>();
  const int grid = sm_count * occ[mb];
  list = list && !pixel;
  const bool uni = g_sweep_uni && !pixel && a.st.uniform;  // compile-time uniform geometry (RAPID_SWEEP_UNI=0: runtime)
  if (list) launch_pdl(k_bset_list, dim3(sm_count * 8), dim3(256), s, a);
#define RAPID_SWEEP_LAUNCH(MB)                                                                     \
  if (pixel && gated) launch_pdl(k_sweep<true, true, MB>, dim3(grid), dim3(K4B_THREADS), s, a);        \
  else if (pixel) launch_pdl(k_sweep<true, false, MB>, dim3(grid), dim3(K4B_THREADS), s, a);           \
  else if (list && gated && smallb) launch_pdl(k_sweep<false, true, MB, true, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (list && smallb) launch_pdl(k_sweep<false, false, MB, true, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (list && gated) launch_pdl(k_sweep<false, true, MB, false, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (list) launch_pdl(k_sweep<false, false, MB, false, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (gated && smallb && uni) launch_pdl(k_sweep<false, true, MB, true, false, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (gated && smallb) launch_pdl(k_sweep<false, true, MB, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (smallb) launch_pdl(k_sweep<false, false, MB, true>, dim3(grid), dim3(K4B_THREADS), s, a);   \
  else if (gated && uni) launch_pdl(k_sweep<false, true, MB, false, false, true>, dim3(grid), dim3(K4B_THREADS), s, a); \
  else if (gated) launch_pdl(k_sweep<false, true, MB>, dim3(grid), dim3(K4B_THREADS), s, a);           \
  else launch_pdl(k_sweep<false, false, MB>, dim3(grid), dim3(K4B_THREADS), s, a);
  if (mb == 2) { RAPID_SWEEP_LAUNCH(2) }
  else if (mb == 4) { RAPID_SWEEP_LAUNCH(4) }
  else { RAPID_SWEEP_LAUNCH(3) }
#undef RAPID_SWEEP_LAUNCH
}

void launch_commit(const PhaseArgs &a, bool pixel, int grid, cudaStream_t s) {
  if (pixel) launch_pdl(k_commit<true, false>, dim3(grid), dim3(256), s, a);
  else launch_pdl(k_commit<false, false>, dim3(grid), dim3(256), s, a);
}

// K5 + the next K3 in one cooperative launch (grid = every CTA that fits at once)
cudaError_t launch_commit_snap(const PhaseArgs &a, bool pixel, int sm_count, cudaStream_t s) {
  const void *fn = pixel ? (const void *)k_commit<true, true> : (const void *)k_commit<false, true>;
  int nb = 0;  // per call: the current device / context decides what fits co-resident
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 256, 0);
  if (e != cudaSuccess) return e;
  PhaseArgs copy = a;
  void *args[] = {&copy};
  return cudaLaunchCooperativeKernel(fn, dim3(sm_count * std::max(nb, 1)), dim3(256), args, 0, s);
}

}  // namespace rapid
