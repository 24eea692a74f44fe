// kernels.cu — the RAPID / CTFTPS refinement hot path on sm_100a.
//
// Kernel map (SURVEY §2.4 / DESIGN.md §4):
//   K1 pyramid_leaf/pyramid_up  block-sum pyramid (Eq. 8 exact, A23)
//   K2 init_sp/init_map0/stats0 grid labels + S_1 (RAPID l.1, l.9-10)
//   K3 snapshot                 frozen per-phase fixed-point means (RAPID l.18; A4, A24)
//   K4 propose                  parity-phase boundary sweep: Eq. 1-3, E_topo, Eq. 7 gate, size gate
//   K5 commit                   all-or-nothing size budget + warp-aggregated stats deltas
//   K6 merge round              Eqs. 4-5, ordered resolution (A12-A16)
//   K7 predict                  Eq. 6 + boundary superpixels + active compaction
//   K8 transition               label mapping to the next stage + active-tile worklist
//   K9 final                    final grain upsample / pending remap (Table 1 grain)
#include <cstdio>

#include <algorithm>
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace rapid {

typedef __int128 i128;

// ------------------------------------------------------------------------------- helpers
// ------------------------------------------------------------------ K2: initial state
__global__ void k_init_sp(const InitArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x) {
    const int local = k % a.M;
    const int j = local / a.cols, i = local - j * a.cols;
    a.sp.init[k] = (a.X[i + 1] - a.X[i]) * (a.Y[j + 1] - a.Y[j]);  // InitSize = cell area
    a.sp.alive[k] = 1;
    a.sp.active[k] = 1;
    a.sp.y[k] = 0;
    a.sp.victim[k] = 0;
    a.sp.remap[k] = local;
#pragma unroll
    for (int f = 0; f < SUMW; f++) a.sp.sums[(size_t)k * SUMW + f] = 0ull;
  }
}

// K1: packed colour sums of the finest block stage, by direct summation over each block.
// f3 / A32 literal image pyramid: a block's colour data become area x the rounded (half up)
// mean of its exact (leaf) or level-synthesised (parent) sums, per packed channel
__device__ __forceinline__ uint64_t lit_round(uint64_t pk, uint64_t area) {
  uint64_t o = 0;
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    const uint64_t sc = (pk >> (21 * ch)) & 0x1FFFFFull;
    o |= (area * ((2 * sc + area) / (2 * area))) << (21 * ch);
  }
  return o;
}

__global__ void k_pyramid_leaf(const StageDev st, const uint8_t *__restrict__ image, int H, int W,
                               int B, uint64_t *__restrict__ bsum, bool literal) {
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
    const int x0 = st.xs[gx], x1 = st.xs[gx + 1], y0 = st.ys[gy], y1 = st.ys[gy + 1];
    uint32_t sr = 0, sg = 0, sb = 0;
    for (int y = y0; y < y1; y++) {
      const uint8_t *row = image + (((size_t)img * H + y) * W) * 3;
      for (int x = x0; x < x1; x++) {
        sr += row[3 * x];
        sg += row[3 * x + 1];
        sb += row[3 * x + 2];
      }
    }
    uint64_t pk = (uint64_t)sr | ((uint64_t)sg << 21) | ((uint64_t)sb << 42);
    if (literal) pk = lit_round(pk, (uint64_t)(x1 - x0) * (uint64_t)(y1 - y0));
    if (st.bsum32) reinterpret_cast<uint32_t *>(bsum)[t] = narrow_bsum32(pk);
    else bsum[t] = pk;
  }
}

// K1 fast path: uniform 2x2 leaf, W % 8 == 0.  A thread sums 4 consecutive blocks of one
// block row from two 24-B pixel segments (8-B vector loads) and writes 4 packed sums.
__device__ __forceinline__ uint32_t byte_of(const uint2 (&v)[3], int i) {
  const uint32_t w = (i < 8) ? ((i < 4) ? v[0].x : v[0].y) : (i < 16) ? ((i < 12) ? v[1].x : v[1].y)
                                                                      : ((i < 20) ? v[2].x : v[2].y);
  return (w >> (8 * (i & 3))) & 0xffu;
}
__global__ void k_pyramid_leaf2(const StageDev st, const uint8_t *__restrict__ image, int H, int W,
                                int B, uint64_t *__restrict__ bsum, bool literal) {
  const int q = st.nbx / 4;  // thread groups per block row
  const size_t n = (size_t)q * st.nby * B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t row = t / q;  // img * nby + gy
    const int gx = (int)(t - row * q) * 4;
    const int img = (int)(row / st.nby), gy = (int)(row - (size_t)img * st.nby);
    const uint8_t *p0 = image + (((size_t)img * H + 2 * gy) * W + 2 * gx) * 3;
    const uint2 *r0 = reinterpret_cast<const uint2 *>(p0);
    const uint2 *r1 = reinterpret_cast<const uint2 *>(p0 + (size_t)W * 3);
    const uint2 a[3] = {__ldg(r0), __ldg(r0 + 1), __ldg(r0 + 2)};
    const uint2 b[3] = {__ldg(r1), __ldg(r1 + 1), __ldg(r1 + 2)};
    uint64_t out[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t s[3];
#pragma unroll
      for (int ch = 0; ch < 3; ch++)
        s[ch] = byte_of(a, 6 * j + ch) + byte_of(a, 6 * j + 3 + ch) + byte_of(b, 6 * j + ch) +
                byte_of(b, 6 * j + 3 + ch);
      out[j] = (uint64_t)s[0] | ((uint64_t)s[1] << 21) | ((uint64_t)s[2] << 42);
      if (literal) out[j] = lit_round(out[j], 4);
    }
    // uniform b = 2: u32 storage (StageDev::bsum32)
    *reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(bsum) + row * st.nbx + gx) =
        make_uint4(narrow_bsum32(out[0]), narrow_bsum32(out[1]), narrow_bsum32(out[2]), narrow_bsum32(out[3]));
  }
}

// K1: coarser stage from its <= 2x2 children (packed fields never overflow: block <= 64^2).
// Fused leaf for dyadic pyramids (b = 2 leaf, b = 4 parent, both uniform): one thread reads a
// 8 x 4 pixel patch (four 2x2 blocks in each of two block rows) with 8-B loads and writes the
// eight b = 2 sums and the two b = 4 sums: the b = 4 level is not re-read from HBM.
template <bool literal>
__global__ void k_pyramid_leaf24(const StageDev st, const StageDev up, const uint8_t *__restrict__ image, int H,
                                 int W, int B, uint64_t *__restrict__ bsum, uint64_t *__restrict__ bsum_up) {
  const int q = st.nbx / 4;        // thread groups per block-row pair
  const int npair = st.nby / 2;    // block-row pairs per image
  const size_t n = (size_t)q * npair * B;
  const unsigned lane = threadIdx.x & 31u;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the stores below exchange data between lanes)
  for (size_t base = blockIdx.x * (size_t)blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
    const size_t t = base + lane;
    const bool valid = t < n;
    const size_t pr = valid ? t / q : 0;  // img * npair + pair
    const int gx = valid ? (int)(t - pr * q) * 4 : 0;
    const int img = (int)(pr / npair), gy = 2 * (int)(pr - (size_t)img * npair);
    uint64_t o2[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (!valid) continue;
      const uint8_t *p0 = image + (((size_t)img * H + 2 * (gy + h)) * W + 2 * gx) * 3;
      const uint2 *r0 = reinterpret_cast<const uint2 *>(p0);
      const uint2 *r1 = reinterpret_cast<const uint2 *>(p0 + (size_t)W * 3);
      const uint2 a[3] = {__ldcs(r0), __ldcs(r0 + 1), __ldcs(r0 + 2)};
      const uint2 b[3] = {__ldcs(r1), __ldcs(r1 + 1), __ldcs(r1 + 2)};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        uint32_t sc[3];
#pragma unroll
        for (int ch = 0; ch < 3; ch++)
          sc[ch] = byte_of(a, 6 * j + ch) + byte_of(a, 6 * j + 3 + ch) + byte_of(b, 6 * j + ch) +
                   byte_of(b, 6 * j + 3 + ch);
        o2[h][j] = (uint64_t)sc[0] | ((uint64_t)sc[1] << 21) | ((uint64_t)sc[2] << 42);
        if (literal) o2[h][j] = lit_round(o2[h][j], 4);
      }
    }
    // b = 2 sums in u32 storage (StageDev::bsum32): a thread's four blocks are 16 contiguous
    // bytes, so the lanes of a warp on one block row write whole 32-B sectors
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (valid)
        *reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(bsum) + ((size_t)img * st.nby + gy + h) * st.nbx + gx) =
            make_uint4(narrow_bsum32(o2[h][0]), narrow_bsum32(o2[h][1]), narrow_bsum32(o2[h][2]), narrow_bsum32(o2[h][3]));
    if (valid) {  // packed fields never carry: each stays < 2^21 up to b = 90
      uint64_t u0 = o2[0][0] + o2[0][1] + o2[1][0] + o2[1][1], u1 = o2[0][2] + o2[0][3] + o2[1][2] + o2[1][3];
      if (literal) {
        u0 = lit_round(u0, 16);
        u1 = lit_round(u1, 16);
      }
      uint64_t *dup = bsum_up + ((size_t)img * up.nby + (gy >> 1)) * up.nbx + (gx >> 1);
      *reinterpret_cast<ulonglong2 *>(dup) = make_ulonglong2(u0, u1);
    }
  }
}

__global__ void k_pyramid_up(const StageDev st, const StageDev ch, int B, uint64_t *__restrict__ bsum,
                             bool literal) {
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
    uint64_t acc = 0;
    for (int cy = st.cys[gy]; cy < st.cys[gy + 1]; cy++)
      for (int cx = st.cxs[gx]; cx < st.cxs[gx + 1]; cx++)
        acc += bsum_at(ch, ((size_t)img * ch.nby + cy) * ch.nbx + cx);
    if (literal)
      acc = lit_round(acc, (uint64_t)(st.xs[gx + 1] - st.xs[gx]) * (uint64_t)(st.ys[gy + 1] - st.ys[gy]));
    bsum[t] = acc;
  }
}

__global__ void k_init_map0(const InitArgs a) {
  const StageDev &st = a.st0;
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * a.B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t r = t % nper;
    const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
    st.map[t] = a.celly[gy] * a.cols + a.cellx[gx];  // label j*c + i (RAPID l.1)
  }
}

// S_1: per-superpixel int64 sums from the stage-0 blocks (warp-aggregated atomics).
template <bool PIXEL>
__global__ void k_stats0(const InitArgs a) {
  const StageDev &st = a.st0;
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * a.B;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = blockIdx.x * (size_t)blockDim.x; base < n; base += stride) {
    const size_t t = base + threadIdx.x;
    const bool valid = t < n;
    long long d[6] = {0, 0, 0, 0, 0, 0};
    int key = 0;
    if (valid) {
      const int img = (int)(t / nper);
      const size_t r = t - (size_t)img * nper;
      const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
      if (PIXEL) block_data_pix(a.image, a.H, a.W, img, gx, gy, d);
      else block_data_blk(st, img, gx, gy, d);
      key = img * a.M + st.map[t];
    }
    agg_sums(valid, key, d, false, a.sp.sums, nullptr);
  }
}

// ------------------------------------------------------------------ K3: snapshot
__global__ void __launch_bounds__(256, 8) k_snapshot(const SnapArgs a) {  // one wave at K = 2^20
  pdl_wait_and_trigger();
  snapshot_warps(a, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
}


// ------------------------------------------------------- ordered compaction of u8 flags
// chunk = 1024 flags per CTA of 256 threads (4 consecutive flags per thread)
constexpr int CHUNK = 1024;

__global__ void k_flag_count(const uint8_t *__restrict__ flags, int n, unsigned *chunk,
                             const uint32_t *gate) {
  if (gate && *gate == 0u) return;
  __shared__ unsigned s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const int b0 = blockIdx.x * CHUNK + threadIdx.x * 4;
  unsigned c = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (b0 + k < n) c += flags[b0 + k] != 0;
  c = __reduce_add_sync(FULL, c);
  if (lane_id() == 0) atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0) chunk[blockIdx.x] = s;
}

// single-CTA exclusive scan in place; *total = sum
__global__ void k_scan_chunks(unsigned *chunk, int nchunks, unsigned *total, const uint32_t *gate) {
  if (gate && *gate == 0u) return;
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nchunks; base += blockDim.x) {
    const int i = base + threadIdx.x;
    unsigned v = i < nchunks ? chunk[i] : 0u;
    // inclusive warp scan
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(FULL, x, o);
      if (lane_id() >= o) x += y;
    }
    if (lane_id() == 31) warp_tot[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = blockDim.x >> 5;
      unsigned t = threadIdx.x < nw ? warp_tot[threadIdx.x] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(FULL, t, o);
        if (lane_id() >= o) t += y;
      }
      warp_tot[threadIdx.x] = t;  // inclusive
    }
    __syncthreads();
    const unsigned woff = (threadIdx.x >> 5) ? warp_tot[(threadIdx.x >> 5) - 1] : 0u;
    if (i < nchunks) chunk[i] = carry + woff + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_flag_scatter(const uint8_t *__restrict__ flags, int n, const unsigned *chunk,
                               int32_t *list, const uint32_t *gate) {
  if (gate && *gate == 0u) return;
  __shared__ unsigned warp_tot[8];
  const int b0 = blockIdx.x * CHUNK + threadIdx.x * 4;
  unsigned c = 0;
  uint8_t f[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    f[k] = (b0 + k < n) ? flags[b0 + k] : 0;
    c += f[k] != 0;
  }
  unsigned x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(FULL, x, o);
    if (lane_id() >= o) x += y;
  }
  if (lane_id() == 31) warp_tot[threadIdx.x >> 5] = x;
  __syncthreads();
  unsigned woff = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); w++) woff += warp_tot[w];
  unsigned pos = chunk[blockIdx.x] + woff + x - c;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (f[k]) list[pos++] = b0 + k;
}

// ------------------------------------------------------------------ K6: merge round
// victims: head[V] = -1
__global__ void k_merge_heads(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.npairs = 0u;  // this round's pair counter
  const unsigned nv = *a.total;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x)
    a.head[a.vlist[i]] = -1;
}

// O7 step 1: (victim, neighbour) -> shared edge length.  Counted from the victim's side: each
// block p of a victim V adds, for every 4-neighbour q with L_q != V, the shared edge length
// to len[V][L_q] — the same totals as summing over unordered adjacent pairs.  At gated
// stages only worklist tiles can hold victim blocks (victims are active superpixels, and
// active superpixels' blocks never leave the worklist tiles), so only those are scanned.
// One CTA per sweep tile; thread (r, q) owns blocks gx0+4q .. +3 of row gy0+r.  With boundary
// sets (a.bset), only blocks whose bit is set are examined: a victim is an active superpixel
// (it passed the static gate) and the sets hold every gated boundary block (sweep.cu).
__global__ void __launch_bounds__(256) k_merge_adjacency(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const StageDev &st = a.st;
  const int nbx = st.nbx, nby = st.nby;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const int r = threadIdx.x >> 4, q = threadIdx.x & 15;
  for (unsigned w = blockIdx.x; w < ntiles; w += gridDim.x) {
    const uint32_t tile = a.worklist ? (uint32_t)a.worklist[w] : w;
    const uint32_t rr = fdiv(tile, st.fd_tx), img = fdiv(rr, st.fd_ty);
    const int gx0 = (int)(tile - rr * (uint32_t)st.tiles_x) * TX, gy0 = (int)(rr - img * (uint32_t)st.tiles_y) * TY;
    const int gy = gy0 + r;
    if (gy >= nby) continue;
    unsigned m4 = 0xfu;  // blocks of this thread to examine
    if (a.bset) {
      const uint32_t *tw = a.bset + (size_t)tile * 32 + (r >> 1);
      const uint32_t w0 = tw[(0 + 2 * (r & 1)) * (TY / 2)], w1 = tw[(1 + 2 * (r & 1)) * (TY / 2)];
      m4 = ((w0 >> (2 * q)) & 1u) | (((w1 >> (2 * q)) & 1u) << 1) | (((w0 >> (2 * q + 1)) & 1u) << 2) |
           (((w1 >> (2 * q + 1)) & 1u) << 3);
    }
    if (!m4) continue;
    const int32_t *map = st.map + (size_t)img * nby * nbx;
    const int kb = (int)img * a.M;
    const unsigned eh = (unsigned)(st.ys[gy + 1] - st.ys[gy]);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int gx = gx0 + 4 * q + k;
      if (!((m4 >> k) & 1u) || gx >= nbx) continue;
      const size_t p = (size_t)gy * nbx + gx;
      const int la = map[p];
      if (!a.sp.victim[kb + la]) continue;  // victims are rare: their neighbours only are loaded
      const int nq[4] = {gy > 0 ? map[p - nbx] : la, gx + 1 < nbx ? map[p + 1] : la,
                         gy + 1 < nby ? map[p + nbx] : la, gx > 0 ? map[p - 1] : la};
      if (nq[0] == la && nq[1] == la && nq[2] == la && nq[3] == la) continue;
      const unsigned ew = (unsigned)(st.xs[gx + 1] - st.xs[gx]);
#pragma unroll
      for (int d = 0; d < 4; d++)
        if (nq[d] != la) hash_add(a, kb + la, kb + nq[d], (d & 1) ? eh : ew);
    }
  }
}

// Victim adjacency from the boundary sets, one warp per worklist tile: the tile's 32 bitset words
// (4 colours x 8 plane rows) hold every gated boundary block at the stage end, a superset of the
// victims' boundary blocks (a victim passed the static gate); their set bits are dealt 32 at a
// time to the lanes, each lane loads its block's label and victim flag and, for a victim block
// only, its four neighbours, adding the shared edge lengths to the (victim, neighbour) hash.
// Two dependent loads per set bit instead of a full pass over the stage map.  U rounds of 32
// set bits are dealt at once and their label loads (then their victim-flag loads) issued
// together: one dependent round trip per U rounds (the pass is latency-bound; the hash totals
// and everything after them do not depend on the insertion order).
template <int U, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_merge_adj_bset(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const StageDev &st = a.st;
  const int nbx = st.nbx, nby = st.nby;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const int lane = lane_id();
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ntiles; w += nw) {
    const uint32_t tile = a.worklist ? (uint32_t)a.worklist[w] : w;
    const uint32_t rr = fdiv(tile, st.fd_tx), img = fdiv(rr, st.fd_ty);
    const int gx0 = (int)(tile - rr * (uint32_t)st.tiles_x) * TX, gy0 = (int)(rr - img * (uint32_t)st.tiles_y) * TY;
    const uint32_t word = a.bset[(size_t)tile * 32 + lane];  // colour lane >> 3, plane row lane & 7
    const unsigned cw = __popc(word);
    unsigned incl = cw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned total = __shfl_sync(FULL, incl, 31);
    const int32_t *map = st.map + (size_t)img * nby * nbx;
    const int kb = (int)img * a.M;
    for (unsigned rb = 0; rb < total; rb += 32 * U) {
      int gx[U], gy[U], la[U];
      bool in[U], vic[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const unsigned k = rb + 32 * u + lane;
        int j = 0;  // the lane whose word holds set bit k: #lanes with incl <= k
#pragma unroll
        for (int h = 16; h > 0; h >>= 1) {
          const unsigned v = __shfl_sync(FULL, incl, j + h - 1);
          if (v <= k) j += h;
        }
        const uint32_t wj = __shfl_sync(FULL, word, j);
        const unsigned ej = __shfl_sync(FULL, incl, j) - __popc(wj);
        gx[u] = 0;
        gy[u] = 0;
        in[u] = false;
        if (k < total) {
          const unsigned bit = nth_set_bit(wj, k - ej);
          gx[u] = gx0 + 2 * (int)bit + ((j >> 3) & 1);
          gy[u] = gy0 + 2 * (j & 7) + (j >> 4);
          in[u] = gx[u] < nbx && gy[u] < nby;
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) la[u] = in[u] ? map[(size_t)gy[u] * nbx + gx[u]] : -1;
#pragma unroll
      for (int u = 0; u < U; u++) vic[u] = in[u] && a.sp.victim[kb + la[u]] != 0;  // victims are rare
#pragma unroll
      for (int u = 0; u < U; u++) {
        const unsigned vm = __ballot_sync(FULL, vic[u]);
        if (vm == 0u) continue;  // warp-uniform
        if (a.vtile && lane == __ffs(vm) - 1) a.vtile[tile] = a.vstamp;  // (the final remap visits marked tiles only)
        if (!vic[u]) continue;
        const size_t p = (size_t)gy[u] * nbx + gx[u];
        const int l = la[u];
        const int nq[4] = {gy[u] > 0 ? map[p - nbx] : l, gx[u] + 1 < nbx ? map[p + 1] : l,
                           gy[u] + 1 < nby ? map[p + nbx] : l, gx[u] > 0 ? map[p - 1] : l};
        const unsigned ew = (unsigned)(st.xs[gx[u] + 1] - st.xs[gx[u]]), eh = (unsigned)(st.ys[gy[u] + 1] - st.ys[gy[u]]);
#pragma unroll
        for (int d = 0; d < 4; d++)
          if (nq[d] != l) hash_add(a, kb + l, kb + nq[d], (d & 1) ? eh : ew);
      }
    }
  }
}

__global__ void k_merge_degree(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const unsigned nv = *a.total;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    unsigned c = 0;
    for (int h = a.head[a.vlist[i]]; h >= 0; h = a.hnext[h]) c++;
    a.deg[i] = c;
  }
}

// exclusive scan of deg[0..nv) by a single CTA (victims per stage are few): warp w owns the
// contiguous segment w of 32; pass 1 sums each segment with coalesced loads, the 32 segment
// sums are scanned, pass 2 rescans each segment from its offset and writes it
__global__ void __launch_bounds__(1024) k_merge_scan_deg(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  __shared__ unsigned seg_tot[32];
  const int nv = (int)*a.total;
  const int warp = threadIdx.x >> 5, lane = lane_id(), nwarps = blockDim.x >> 5;
  const int per = ((nv + nwarps - 1) / nwarps + 31) & ~31;
  const int b0 = min(nv, warp * per), b1 = min(nv, b0 + per);
  unsigned sum = 0;
  for (int i = b0 + lane; i < b1; i += 32) sum += a.deg[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
  if (lane == 0) seg_tot[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    unsigned t = lane < nwarps ? seg_tot[lane] : 0u;
    const unsigned own = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nwarps) seg_tot[lane] = t - own;  // exclusive segment offsets
    if (lane == 31) {
      a.deg[nv] = t;
      *a.deg_total = t;
    }
  }
  __syncthreads();
  unsigned carry = seg_tot[warp];
  for (int base = b0; base < b1; base += 32) {
    const int i = base + lane;
    const unsigned v = i < b1 ? a.deg[i] : 0u;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (i < b1) a.deg[i] = carry + x - v;
    carry += __shfl_sync(FULL, x, 31);
  }
}

__device__ __forceinline__ i128 merge_energy(const MergeArgs &a, int A, int T, long long len) {
  // ΔE_m of relabelling all of A to T (A14): A's whole sums as the pixel set
  const unsigned long long *s = a.sp.sums + (size_t)A * SUMW;
  const RecV ra = rec_vals(a.sp.rec[A]), rt = rec_vals(a.sp.rec[T]);
  const i128 n = (i128)(long long)s[0];
  const long long cA[3] = {ra.c0, ra.c1, ra.c2}, cT[3] = {rt.c0, rt.c1, rt.c2};
  i128 dC = 0, dP = 0;
#pragma unroll
  for (int ch = 0; ch < 3; ch++)
    dC += (i128)(cT[ch] - cA[ch]) * (n * (i128)(cT[ch] + cA[ch]) - ((i128)(long long)s[1 + ch] << (FRAC + 1)));
  dP += (i128)(rt.mx - ra.mx) * (n * (i128)(rt.mx + ra.mx) - ((i128)(long long)s[4] << (FRAC + 1)));
  dP += (i128)(rt.my - ra.my) * (n * (i128)(rt.my + ra.my) - ((i128)(long long)s[5] << (FRAC + 1)));
  return (dC << 16) + (i128)a.lam_pos * dP - ((i128)a.lam_b * (i128)(2 * len) << 16);
}

// candidates of every victim: Eq. 5-feasible neighbours sorted by (ΔE_m, T)
__global__ void k_merge_fill(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const unsigned nv = *a.total;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const int A = a.vlist[i];
    const unsigned off = a.deg[i];
    unsigned c = 0;
    const long long nA = (long long)a.sp.sums[(size_t)A * SUMW];
    for (int h = a.head[A]; h >= 0; h = a.hnext[h]) {
      const int T = (int)(a.hkeys[h] & 0xffffffffull);
      const long long nT = (long long)a.sp.sums[(size_t)T * SUMW];
      // Eq. 5: Size(T) + Size(A) <= u * InitSize(T)
      const bool feas = (nT + nA) * a.u_den <= a.u_num * (long long)a.sp.init[T];
      const i128 E = merge_energy(a, A, T, (long long)a.hvals[h]);
      // insertion into the sorted segment [off, off+c)
      unsigned k = c;
      while (k > 0) {
        const unsigned p = off + k - 1;
        const int Tp = a.candT[p];
        const i128 Ep = (i128)((unsigned __int128)a.candE[2 * p] << 64 | a.candE[2 * p + 1]);
        const bool later = feas ? (Tp < 0 || E < Ep || (E == Ep && T < Tp)) : false;
        if (!later) break;
        a.candT[p + 1] = Tp;
        a.candE[2 * (p + 1)] = a.candE[2 * p];
        a.candE[2 * (p + 1) + 1] = a.candE[2 * p + 1];
        k--;
      }
      a.candT[off + k] = feas ? T : -1;
      a.candE[2 * (off + k)] = (unsigned long long)((unsigned __int128)E >> 64);
      a.candE[2 * (off + k) + 1] = (unsigned long long)E;
      c++;
    }
    for (unsigned k = 0; k < c; k++) a.candV[off + k] = A;
  }
}

// O7 steps 3-4.  The sequential rule — victims in ascending id; an unlocked victim takes its
// first unlocked candidate (sorted by (dE_m, T)); both get locked — is exactly the greedy
// maximal matching over the edges (A, T) taken in CSR order (victims ascending, candidates
// sorted).  It is computed with deterministic reservations: every pending edge whose ends
// are both free reserves both ends with atomicMin(edge id); an edge holding both of its
// reservations is the earliest pending edge at both ends, so the sequential order would
// take it too.  Rounds repeat until no edge is pending; the result is order-independent.
// mlock[] (per superpixel) and res[] (reservations) are zero / ~0 outside this kernel.
// Cooperative (grid-synchronised) version: every round is three grid-wide passes over the
// edges; a.flag[2] = "some edge still pending" per round parity, a.npairs the pair counter.
__global__ void __launch_bounds__(256) k_merge_match(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  cg::grid_group grid = cg::this_grid();
  const unsigned ne = a.deg[*a.total];
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (unsigned round = 0;; round++) {
    int any = 0;
    for (unsigned p = tid; p < ne; p += nth) {
      const int T = a.candT[p];
      if (T < 0) continue;
      const int V = a.candV[p];
      if (a.mlock[V] || a.mlock[T]) {
        a.candT[p] = -1;  // an end is taken: dropped for good
        continue;
      }
      atomicMin(&a.res[V], p);
      atomicMin(&a.res[T], p);
      any = 1;
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(&a.flag[round & 1], 1u);
    grid.sync();
    const bool more = *reinterpret_cast<volatile unsigned *>(&a.flag[round & 1]) != 0u;
    if (!more) break;
    if (tid == 0) a.flag[(round + 1) & 1] = 0u;  // next round's flag (nobody sets it before the next sync)
    for (unsigned p = tid; p < ne; p += nth) {
      const int T = a.candT[p];
      if (T < 0) continue;
      const int V = a.candV[p];
      if (a.res[V] == p && a.res[T] == p) {
        a.mlock[V] = 1u;
        a.mlock[T] = 1u;
        const unsigned qq = atomicAdd(a.npairs, 1u);
        a.pairs[2 * qq] = V;
        a.pairs[2 * qq + 1] = T;
        a.candT[p] = -1;
      }
    }
    grid.sync();
    for (unsigned p = tid; p < ne; p += nth) {  // release reservations
      const int T = a.candT[p];
      const int V = a.candV[p];
      a.res[V] = 0xffffffffu;
      if (T >= 0) a.res[T] = 0xffffffffu;
    }
    grid.sync();
  }
  if (tid == 0) {
    const unsigned np = *a.npairs;
    a.stage_info[0] += *a.total;
    a.stage_info[1] += np;
    if (np) *a.remap_pending = 1u;
    a.flag[0] = a.flag[1] = 0u;
  }
}

__global__ void k_merge_apply(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const unsigned np = *a.npairs;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) {
    const int A = a.pairs[2 * i], T = a.pairs[2 * i + 1];
#pragma unroll
    for (int f = 0; f < 6; f++) {
      a.sp.sums[(size_t)T * SUMW + f] += a.sp.sums[(size_t)A * SUMW + f];
      a.sp.sums[(size_t)A * SUMW + f] = 0ull;
    }
    a.sp.alive[A] = 0;
    a.sp.active[A] = 0;
    a.sp.y[A] = 0;
    a.sp.remap[A] = T % a.M;  // local id of the target
    mark_dirty(a.sp.dirty, A);  // (the next stage's first snapshot refreshes only these)
    mark_dirty(a.sp.dirty, T);
    a.mlock[A] = 0u;
    a.mlock[T] = 0u;
  }
}

__global__ void k_merge_cleanup(const MergeArgs a) {
  if (*a.victim_any == 0u) return;
  const unsigned nv = *a.total;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const int A = a.vlist[i];
    a.sp.victim[A] = 0;
    for (int h = a.head[A]; h >= 0; h = a.hnext[h]) {
      a.hkeys[h] = HEMPTY;
      a.hvals[h] = 0u;
    }
  }
}

__global__ void k_merge_done(const MergeArgs a) { *a.victim_any = 0u; }

// ------------------------------------------------------------------ K7: prediction
__global__ void k_predict_y(const PredictArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x) {
    if (!a.sp.alive[k]) {
      a.sp.y[k] = 0;
      a.sp.active[k] = 0;
      continue;
    }
    const Rec r = a.sp.rec[k];
    const long long c[3] = {(long long)(r.cq01 & 0xffffu), (long long)(r.cq01 >> 16),
                            (long long)(r.cq2f & 0xffffu)};
    long long dmin = -1;
    for (int t = 0; t < a.n_proto; t++) {
      long long dd = 0;
#pragma unroll
      for (int ch = 0; ch < 3; ch++) {
        const long long e = c[ch] - ((long long)a.proto[t][ch] << FRAC);
        dd += e * e;
      }
      if (dmin < 0 || dd < dmin) dmin = dd;
    }
    const int8_t y = ((a.tau2 << (2 * FRAC)) - dmin >= 0) ? 1 : -1;  // Eq. 6
    a.sp.y[k] = y;
    a.sp.active[k] = (a.mask_rule == 1) ? (y == 1) : 0;
  }
}


// boundary superpixels: a 4-adjacent superpixel of the other class
__device__ __forceinline__ int resolve(const SpDev &sp, int kb, int l, bool remap) {
  if (remap && !sp.alive[kb + l]) return sp.remap[kb + l];
  return l;
}

// ---------------------------------------------------- f2: feature model of the prediction
// A31 (oracle.h / oracle.c predict_features): brightness (r+g+b)/3; per superpixel n,
// S = sum(r+g+b), Q = sum((r+g+b)^2) over its pixels at stage 0 (after the stage-0 merges).
// scratch[k*SUMW + 0] = Q, + 1 = S (from the pixels: with the literal pyramid the superpixel
// sums are approximations, A33), + 2 = f1, + 3 = sum |f1 - f1_q|, + 4 = distinct neighbours, + 5 = f3;
// image totals S, N at scratch[img*M*SUMW + 6 / 7].  Everything exact (integers, round half up).
__device__ __forceinline__ long long rhu128(__int128 num, __int128 den) {
  return (long long)((2 * num + den) / (2 * den));
}

__global__ void k_feat_q(const PredictArgs a) {  // S, Q per superpixel from the pixels
  const bool rm = *a.remap_pending != 0u;
  const StageDev &st = a.st;
  const size_t nper = (size_t)a.H * a.W, n = nper * a.B;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = blockIdx.x * (size_t)blockDim.x; base < n; base += stride) {  // warp-uniform
    const size_t t = base + threadIdx.x;
    const bool valid = t < n;
    int key = 0;
    unsigned long long v = 0, w = 0;
    if (valid) {
      const int img = (int)(t / nper);
      const size_t r = t - (size_t)img * nper;
      const int y = (int)(r / a.W), x = (int)(r - (size_t)y * a.W);
      const int kb = img * a.M;
      const int l = resolve(a.sp, kb, st.map[((size_t)img * st.nby + a.b0y[y]) * st.nbx + a.b0x[x]], rm);
      key = kb + l;
      const uint8_t *p = a.image + t * 3;
      const unsigned long long s = (unsigned long long)p[0] + p[1] + p[2];
      v = s * s;
      w = s;
    }
    const WarpRun run = warp_runs(valid, key);
    const int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(FULL, v, o), uw = __shfl_up_sync(FULL, w, o);
      if (lane - o >= run.start) {
        v += u;
        w += uw;
      }
    }
    if (valid && run.end) {
      atomicAdd(&a.scratch[(size_t)key * SUMW + 0], v);
      atomicAdd(&a.scratch[(size_t)key * SUMW + 1], w);
    }
  }
}

// Q on uniform stage-0 grids (square b0 x b0 blocks, b0 in {8, 16, 32, 64}, W % 8 == 0): a CTA
// takes a band of b0 rows x 256 columns; a thread reads 8 pixels of a row with 8-B loads
// (they lie in one block), warps reduce each block's row sums with shuffles and add them in
// shared memory; one atomic per block and band.
template <int b0>
__global__ void __launch_bounds__(256) k_feat_q_band(const PredictArgs a) {
  __shared__ unsigned long long s_q[32], s_s[32];  // blocks of the band (256 / b0 <= 32)
  const bool rm = *a.remap_pending != 0u;
  const StageDev &st = a.st;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int gcols = (a.W + 255) / 256, bands_y = a.H / b0;
  const unsigned nbands = (unsigned)a.B * bands_y * gcols;
  const int per = b0 / 8;                // lanes per block in a warp row
  const int nblk = 256 / b0;             // blocks per band
  for (unsigned band = blockIdx.x; band < nbands; band += gridDim.x) {
    const unsigned gx = band % gcols, r2 = band / gcols;
    const int by = (int)(r2 % bands_y), img = (int)(r2 / bands_y);
    if (threadIdx.x < 32) s_q[threadIdx.x] = s_s[threadIdx.x] = 0ull;
    __syncthreads();
    const int x0 = (int)gx * 256 + 8 * lane;
#pragma unroll
    for (int row = warp; row < b0; row += 8) {  // b0 / 8 independent rows per warp
      const int y = by * b0 + row;
      unsigned long long q = 0, sv = 0;
      if (x0 < a.W) {
        const uint2 *p = reinterpret_cast<const uint2 *>(a.image + (((size_t)img * a.H + y) * a.W + x0) * 3);
        const uint2 v[3] = {__ldcs(p), __ldcs(p + 1), __ldcs(p + 2)};
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const unsigned long long t = (unsigned long long)byte_of(v, 3 * j) + byte_of(v, 3 * j + 1) + byte_of(v, 3 * j + 2);
          q += t * t;
          sv += t;
        }
      }
      for (int o = 1; o < per; o <<= 1) {
        q += __shfl_xor_sync(FULL, q, o);
        sv += __shfl_xor_sync(FULL, sv, o);
      }
      if ((lane % per) == 0 && x0 < a.W) {
        atomicAdd(&s_q[lane / per], q);
        atomicAdd(&s_s[lane / per], sv);
      }
    }
    __syncthreads();
    if (threadIdx.x < nblk) {
      const int bx = (int)gx * nblk + (int)threadIdx.x;
      if (bx < st.nbx) {
        const int kb = img * a.M;
        const int l = resolve(a.sp, kb, st.map[((size_t)img * st.nby + by) * st.nbx + bx], rm);
        atomicAdd(&a.scratch[(size_t)(kb + l) * SUMW + 0], s_q[threadIdx.x]);
        atomicAdd(&a.scratch[(size_t)(kb + l) * SUMW + 1], s_s[threadIdx.x]);
      }
    }
    __syncthreads();
  }
}

__global__ void k_feat_f1(const PredictArgs a) {  // f1, f3 per superpixel; image totals
  // warp-uniform trip count: the image totals are warp-aggregated (one atomic per image run)
  for (int base = blockIdx.x * blockDim.x; base < a.K; base += gridDim.x * blockDim.x) {
    const int k = base + (int)threadIdx.x;
    const bool valid = k < a.K && a.sp.alive[k];
    long long n = 0, S = 0;
    if (valid) {
      const unsigned long long *sm = a.sp.sums + (size_t)k * SUMW;
      n = (long long)sm[0];
      S = (long long)a.scratch[(size_t)k * SUMW + 1];
      const unsigned long long Q = a.scratch[(size_t)k * SUMW + 0];
      // f1: S 2^16 < 2^58 and 765 n < 2^42 fit 64 bits
      const long long f1 = (long long)((2ull * ((unsigned long long)S << 16) + 765ull * n) / (2ull * 765ull * n));
      long long f3;
      if (n < (1ll << 20)) {  // n Q and S^2 < 2^60: 64-bit products
        const unsigned long long var = (unsigned long long)n * Q - (unsigned long long)S * S;
        const unsigned long long den = 585225ull * n * n;  // < 2^60
        if (var >> 45) f3 = rhu128((__int128)var << 16, (__int128)den);  // keep 2 var 2^16 + den < 2^64
        else f3 = (long long)((2 * (var << 16) + den) / (2 * den));
      } else {
        f3 = rhu128(((__int128)n * Q - (__int128)S * S) << 16, (__int128)585225 * n * n);
      }
      a.scratch[(size_t)k * SUMW + 2] = (unsigned long long)f1;
      a.scratch[(size_t)k * SUMW + 5] = (unsigned long long)f3;
    }
    const int img = valid ? k / a.M : -1;
    const long long d[6] = {n, S, 0, 0, 0, 0};
    // run-aggregate over lanes of the same image (fields 0, 1 -> totals N, S)
    if (__ballot_sync(FULL, valid)) {
      const WarpRun run = warp_runs(valid, img);
      const int lane = lane_id();
      long long vn = d[0], vs = d[1];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long tn = __shfl_up_sync(FULL, vn, o), ts = __shfl_up_sync(FULL, vs, o);
        if (lane - o >= run.start) {
          vn += tn;
          vs += ts;
        }
      }
      if (valid && run.end) {
        atomicAdd(&a.scratch[(size_t)img * a.M * SUMW + 6], (unsigned long long)vs);
        atomicAdd(&a.scratch[(size_t)img * a.M * SUMW + 7], (unsigned long long)vn);
      }
    }
  }
}

// distinct 4-adjacent superpixel pairs of the stage-0 map: a directed pair (u, v) counts for u
// once (set insert into the merge hash); f4's sum and degree are accumulated at insertion
__global__ void k_feat_adj(const PredictArgs a) {
  const StageDev &st = a.st;
  const bool rm = *a.remap_pending != 0u;
  const size_t nper = (size_t)st.nbx * st.nby, n = nper * a.B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
    const int kb = img * a.M;
    const int la = kb + resolve(a.sp, kb, st.map[t], rm);
#pragma unroll
    for (int dir = 0; dir < 2; dir++) {
      if (dir == 0 ? gx + 1 >= st.nbx : gy + 1 >= st.nby) continue;
      const int lb = kb + resolve(a.sp, kb, st.map[t + (dir == 0 ? 1 : st.nbx)], rm);
      if (lb == la) continue;
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int u = e ? lb : la, v = e ? la : lb;
        const unsigned long long key = ((unsigned long long)(unsigned)u << 32) | (unsigned)v;
        unsigned long long h = hmix(key) & a.hmask;
        while (true) {
          const unsigned long long seen = *reinterpret_cast<volatile unsigned long long *>(&a.hkeys[h]);
          if (seen == key) break;  // already counted
          if (seen == HEMPTY) {
            const unsigned long long old = atomicCAS(&a.hkeys[h], HEMPTY, key);
            if (old == HEMPTY) {  // first sighting of the pair: count it for u
              const long long fu = (long long)a.scratch[(size_t)u * SUMW + 2];
              const long long fv = (long long)a.scratch[(size_t)v * SUMW + 2];
              atomicAdd(&a.scratch[(size_t)u * SUMW + 3], (unsigned long long)(fu > fv ? fu - fv : fv - fu));
              atomicAdd(&a.scratch[(size_t)u * SUMW + 4], 1ull);
              break;
            }
            if (old == key) break;
          }
          h = (h + 1) & a.hmask;
        }
      }
    }
  }
}

__global__ void k_feat_classify(const PredictArgs a) {  // Eq. 6 on the features
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x) {
    if (!a.sp.alive[k]) {
      a.sp.y[k] = 0;
      a.sp.active[k] = 0;
      continue;
    }
    const int img = k / a.M;
    const unsigned long long *ims = a.scratch + (size_t)img * a.M * SUMW;
    const long long fimg = rhu128((__int128)(long long)ims[6] << 16, (__int128)765 * (long long)ims[7]);
    const unsigned long long *f = a.scratch + (size_t)k * SUMW;
    const long long f1 = (long long)f[2], f2 = f1 - fimg, f3 = (long long)f[5];
    const long long deg = (long long)f[4];
    const long long f4 = deg ? rhu128((long long)f[3], deg) : 0;
    const __int128 h = ((__int128)a.feat_w[0] << 16) + (__int128)a.feat_w[1] * f1 + (__int128)a.feat_w[2] * f2 +
                       (__int128)a.feat_w[3] * f3 + (__int128)a.feat_w[4] * f4;
    const int8_t y = h >= 0 ? 1 : -1;
    a.sp.y[k] = y;
    a.sp.active[k] = (a.mask_rule == 1) ? (y == 1) : 0;
  }
}

__global__ void k_predict_bsp(const PredictArgs a) {
  const StageDev &st = a.st;
  const bool rm = *a.remap_pending != 0u;
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * a.B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
    const int kb = img * a.M;
    const int la = resolve(a.sp, kb, st.map[t], rm);
    if (gx + 1 < st.nbx) {
      const int lb = resolve(a.sp, kb, st.map[t + 1], rm);
      if (la != lb && a.sp.y[kb + la] != a.sp.y[kb + lb]) {
        a.sp.active[kb + la] = 1;
        a.sp.active[kb + lb] = 1;
      }
    }
    if (gy + 1 < st.nby) {
      const int lb = resolve(a.sp, kb, st.map[t + st.nbx], rm);
      if (la != lb && a.sp.y[kb + la] != a.sp.y[kb + lb]) {
        a.sp.active[kb + la] = 1;
        a.sp.active[kb + lb] = 1;
      }
    }
  }
}

// ------------------------------------------------------------------ K8: transition
__global__ void __launch_bounds__(256) k_transition(const TransArgs a) {
  const StageDev &pv = a.prev, &nx = a.next;
  const unsigned t = blockIdx.x;
  const int tx = (int)(t % (unsigned)nx.tiles_x);
  const unsigned rr = t / (unsigned)nx.tiles_x;
  const int ty = (int)(rr % (unsigned)nx.tiles_y);
  const int img = (int)(rr / (unsigned)nx.tiles_y);
  const int kb = img * a.M;
  const bool rm = *a.remap_pending != 0u;
  const int32_t *pmap = pv.map + (size_t)img * pv.nby * pv.nbx;
  int32_t *nmap = nx.map + (size_t)img * nx.nby * nx.nbx;
  // each thread: 4 consecutive children of one row (16 threads per 64-wide tile row)
  int act = 0;
  const int gx = tx * TX + 4 * (threadIdx.x & 15), gy = ty * TY + (threadIdx.x >> 4);
  if (gy < nx.nby && gx < nx.nbx) {
    const int32_t *prow = pmap + (size_t)nx.py[gy] * pv.nbx;
    const int4 pc = *reinterpret_cast<const int4 *>(nx.px + gx);  // tables are 16-B padded
    int l[4] = {prow[pc.x], -1, -1, -1};
#pragma unroll
    for (int u = 1; u < 4; u++)
      if (gx + u < nx.nbx) l[u] = prow[(&pc.x)[u]];
    int last = -1, res = -1;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      if (l[u] < 0) continue;
      if (l[u] != last) {  // remap / activity once per distinct parent label
        last = l[u];
        res = (rm && !a.sp.alive[kb + last]) ? a.sp.remap[kb + last] : last;
        if (a.gate) act |= a.sp.active[kb + res];
      }
      l[u] = res;
    }
    int32_t *dst = nmap + (size_t)gy * nx.nbx + gx;
    if (gx + 3 < nx.nbx && (nx.nbx & 3) == 0) {
      *reinterpret_cast<int4 *>(dst) = make_int4(l[0], l[1], l[2], l[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (gx + u < nx.nbx) dst[u] = l[u];
    }
  }
  if (a.gate) {
    act = __syncthreads_or(act);
    if (threadIdx.x == 0 && act) {
      const unsigned p = atomicAdd(a.nwork, 1u);
      a.worklist[p] = (int)t;
    }
  }
}

// Dyadic fast path (both stages uniform, b_prev = 2 b_next, so nx.nbx = 2 pv.nbx): the parent
// of child (x, y) is (x >> 1, y >> 1), so a parent row yields two identical child rows.
// Persistent CTAs of 128 threads, one 64 x 16-child tile (32 x 8 parents) per iteration; thread
// (r, q) = (u >> 4, u & 15) writes children 4q..4q+3 of rows 2r, 2r+1 from parents 2q, 2q+1 of
// parent row r.  The next tile's parents are loaded while this one is written (two loads in
// flight per thread).  BSET: the boundary sets of the next stage come from the parents too (a
// child's outer neighbours are its parent's neighbours, its siblings share its label): the
// remapped parents plus a one-parent halo go through shared memory, each thread forms its 8
// children's bits (boundary and static gate) and half-warps OR them into the tile's 32 words —
// the next stage's bset build pass (a full read of the new map) is not needed.
template <bool BSET>
__global__ void __launch_bounds__(128) k_transition_dyadic(const TransArgs a) {
  __shared__ int32_t s_lab[10][34];  // parent rows -1..8, columns -1..32 of the tile (remapped)
  const StageDev &pv = a.prev, &nx = a.next;
  const unsigned ntiles = (unsigned)(nx.tiles_x * nx.tiles_y) * (unsigned)a.B;
  const bool rm = *a.remap_pending != 0u;
  const bool vec = (pv.nbx & 1) == 0;
  const int u = threadIdx.x, q = u & 15, r = u >> 4;
  auto load_par = [&](unsigned t, int &p0, int &p1) {
    p0 = p1 = -1;
    if (t >= ntiles) return;
    const uint32_t rr = fdiv(t, nx.fd_tx), img = fdiv(rr, nx.fd_ty);
    const int px = (int)(t - rr * (uint32_t)nx.tiles_x) * (TX / 2) + 2 * q;
    const int py = (int)(rr - img * (uint32_t)nx.tiles_y) * (TY / 2) + r;
    if (py >= pv.nby || px >= pv.nbx) return;
    const int32_t *prow = pv.map + ((size_t)img * pv.nby + py) * pv.nbx;
    if (vec) {
      const int2 pp = *reinterpret_cast<const int2 *>(prow + px);
      p0 = pp.x;
      p1 = pp.y;
    } else {
      p0 = prow[px];
      if (px + 1 < pv.nbx) p1 = prow[px + 1];
    }
  };
  int n0, n1;
  load_par(blockIdx.x, n0, n1);
  for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int p0 = n0, p1 = n1;
    load_par(t + gridDim.x, n0, n1);  // prefetch
    const uint32_t rr = fdiv(t, nx.fd_tx), img = fdiv(rr, nx.fd_ty);
    const int tpx = (int)(t - rr * (uint32_t)nx.tiles_x) * (TX / 2), tpy = (int)(rr - img * (uint32_t)nx.tiles_y) * (TY / 2);
    const int kb = (int)img * a.M;
    // flag / remap gathers with a 64-B L2 fill (scattered: a plain load fills 128 B)
    auto res = [&](int p) {
      return (p >= 0 && rm && !ld64_u8(a.sp.alive + kb + p)) ? (int)ld64_u32(a.sp.remap + kb + p) : p;
    };
    p0 = res(p0);
    p1 = res(p1);
    const bool need_act = a.gate || (BSET && a.gating == 1);
    const int a0 = (p0 >= 0 && need_act) ? (int)ld64_u8(a.sp.active + kb + p0) : 0;
    const int a1 = (p1 >= 0 && need_act) ? (int)ld64_u8(a.sp.active + kb + p1) : 0;
    if (BSET) {  // remapped parents and halo into shared memory
      s_lab[r + 1][1 + 2 * q] = p0;
      s_lab[r + 1][2 + 2 * q] = p1;
      if (u < 80) {
        int hy, hx;
        if (u < 32) { hy = -1; hx = u; }
        else if (u < 64) { hy = 8; hx = u - 32; }
        else if (u < 72) { hy = u - 64; hx = -1; }
        else { hy = u - 72; hx = 32; }
        const int y = tpy + hy, x = tpx + hx;
        int v = -1;
        if (y >= 0 && y < pv.nby && x >= 0 && x < pv.nbx)
          v = res((int)ld64_u32(pv.map + ((size_t)img * pv.nby + y) * pv.nbx + x));
        s_lab[hy + 1][hx + 1] = v;
      }
    }
    const int py = tpy + r, px = tpx + 2 * q;
    if (py < pv.nby && px < pv.nbx) {
      int32_t *dst = nx.map + ((size_t)img * nx.nby + 2 * py) * nx.nbx + 2 * px;
      if (vec) {
        const int4 v = make_int4(p0, p0, p1, p1);
        *reinterpret_cast<int4 *>(dst) = v;
        *reinterpret_cast<int4 *>(dst + nx.nbx) = v;
      } else {
        const int l[4] = {p0, p0, p1, p1};
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (2 * px + k < nx.nbx) {
            dst[k] = l[k];
            dst[nx.nbx + k] = l[k];
          }
      }
    }
    if (BSET) {
      __syncthreads();
      // child (i, j) of this thread: parent column pc = 2q + (i >> 1); horizontal outer
      // neighbour on side i & 1, vertical on side j; word (colour (i & 1) + 2 j, plane row r),
      // bit 2q + (i >> 1)
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int pc = 2 * q + h, L = h ? p1 : p0;
        const bool gate = a.gating != 1 || (h ? a1 : a0);
        if (L < 0 || !gate) continue;
        const int lw = s_lab[r + 1][pc], le = s_lab[r + 1][pc + 2];
        const int lu = s_lab[r][pc + 1], ld = s_lab[r + 2][pc + 1];
        const bool bw = lw >= 0 && lw != L, be = le >= 0 && le != L;
        const bool bu = lu >= 0 && lu != L, bd = ld >= 0 && ld != L;
        const uint32_t bit = 1u << (2 * q + h);
        if (bw | bu) w[0] |= bit;  // (i even, j = 0): colour 0
        if (be | bu) w[1] |= bit;  // (i odd, j = 0): colour 1
        if (bw | bd) w[2] |= bit;  // (i even, j = 1): colour 2
        if (be | bd) w[3] |= bit;  // (i odd, j = 1): colour 3
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1)
#pragma unroll
        for (int c = 0; c < 4; c++) w[c] |= __shfl_xor_sync(0xffffffffu, w[c], o);
      if (q == 0) {
        uint32_t *tw = a.bset + (size_t)t * 32 + r;
#pragma unroll
        for (int c = 0; c < 4; c++) tw[c * (TY / 2)] = w[c];
      }
    }
    const int act = __syncthreads_or(a.gate ? (a0 | a1) : 0);
    if (a.gate && threadIdx.x == 0 && act) {
      const unsigned p = atomicAdd(a.nwork, 1u);
      a.worklist[p] = (int)t;
    }
  }
}

// Boundary sets of a dyadic stage from its parents (both stages uniform, b_prev = 2 b_next):
// a child's 4-neighbours are its sibling pair (same parent, same label) and the children of
// its parent's W/E and N/S neighbours on its side, so child (2px + cx, 2py + cy) is a boundary
// block iff its parent's label differs from the parent neighbour on side cx horizontally or
// cy vertically (labels after the pending remap, exactly the child map's values).  One CTA per
// worklist tile of the child stage, warp w = plane row w, lane i = parent column tx*32 + i:
// the four colour words of the row are four ballots.  Reads a quarter of the bytes of the
// child-map tile pass (k_tiles<BSET>) with a fraction of its instructions.
__global__ void __launch_bounds__(256) k_bset_dyadic(const TransArgs a) {
  const StageDev &pv = a.prev, &nx = a.next;
  const unsigned ntiles = a.gate ? *a.nwork : (unsigned)(nx.tiles_x * nx.tiles_y) * (unsigned)a.B;
  const bool rm = *a.remap_pending != 0u;
  const int lane = lane_id(), pr = threadIdx.x >> 5;
  for (unsigned w = blockIdx.x; w < ntiles; w += gridDim.x) {
    const uint32_t t = a.gate ? (uint32_t)a.worklist[w] : w;
    const uint32_t rr = fdiv(t, nx.fd_tx), img = fdiv(rr, nx.fd_ty);
    const int px = (int)(t - rr * (uint32_t)nx.tiles_x) * (TX / 2) + lane;
    const int py = (int)(rr - img * (uint32_t)nx.tiles_y) * (TY / 2) + pr;
    const int kb = (int)img * a.M;
    const int32_t *pm = pv.map + (size_t)img * pv.nby * pv.nbx;
    const bool in = px < pv.nbx && py < pv.nby;
    auto res = [&](int p) {
      return (p >= 0 && rm && !ld64_u8(a.sp.alive + kb + p)) ? (int)ld64_u32(a.sp.remap + kb + p) : p;
    };
    const size_t o = (size_t)py * pv.nbx + px;
    int L = in ? pm[o] : -1;
    int Nl = in && py > 0 ? pm[o - pv.nbx] : -1;
    int Sl = in && py + 1 < pv.nby ? pm[o + pv.nbx] : -1;
    int Wh = (lane == 0 && in && px > 0) ? pm[o - 1] : -1;          // halo (lane 0)
    int Eh = (lane == 31 && in && px + 1 < pv.nbx) ? pm[o + 1] : -1;  // halo (lane 31)
    L = res(L);
    Nl = res(Nl);
    Sl = res(Sl);
    Wh = res(Wh);
    Eh = res(Eh);
    int Wl = __shfl_up_sync(FULL, L, 1), El = __shfl_down_sync(FULL, L, 1);
    if (lane == 0) Wl = Wh;
    if (lane == 31) El = Eh;
    bool gate = L >= 0;
    if (gate && a.gating == 1) gate = ld64_u8(a.sp.active + kb + L) != 0;
    const bool dW = Wl >= 0 && Wl != L, dE = El >= 0 && El != L;
    const bool dN = Nl >= 0 && Nl != L, dS = Sl >= 0 && Sl != L;
    const unsigned w0 = __ballot_sync(FULL, gate && (dW || dN));  // (cx, cy) = (0, 0)
    const unsigned w1 = __ballot_sync(FULL, gate && (dE || dN));  // (1, 0)
    const unsigned w2 = __ballot_sync(FULL, gate && (dW || dS));  // (0, 1)
    const unsigned w3 = __ballot_sync(FULL, gate && (dE || dS));  // (1, 1)
    if (lane == 0) {
      uint32_t *tw = a.bset + (size_t)t * 32 + pr;
      tw[0 * (TY / 2)] = w0;
      tw[1 * (TY / 2)] = w1;
      tw[2 * (TY / 2)] = w2;
      tw[3 * (TY / 2)] = w3;
    }
  }
}

// The same boundary sets with one warp per child tile: the warp walks the tile's 8 parent rows
// top to bottom keeping the resolved rows above and below in registers, so every parent row of
// the tile (plus one halo row above and below) is loaded, remap-resolved and flag-checked once
// instead of by three warps; the next row's loads are issued before the current row's words are
// formed.
__global__ void __launch_bounds__(256) k_bset_dyadic_rows(const TransArgs a) {
  const StageDev &pv = a.prev, &nx = a.next;
  const unsigned ntiles = a.gate ? *a.nwork : (unsigned)(nx.tiles_x * nx.tiles_y) * (unsigned)a.B;
  const bool rm = *a.remap_pending != 0u;
  const int lane = lane_id();
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ntiles; w += nw) {
    const uint32_t t = a.gate ? (uint32_t)a.worklist[w] : w;
    const uint32_t rr = fdiv(t, nx.fd_tx), img = fdiv(rr, nx.fd_ty);
    const int px = (int)(t - rr * (uint32_t)nx.tiles_x) * (TX / 2) + lane;
    const int tpy = (int)(rr - img * (uint32_t)nx.tiles_y) * (TY / 2);
    const int kb = (int)img * a.M;
    const int32_t *pm = pv.map + (size_t)img * pv.nby * pv.nbx;
    const bool inx = px < pv.nbx;
    auto res = [&](int p) {
      return (p >= 0 && rm && !ld64_u8(a.sp.alive + kb + p)) ? (int)ld64_u32(a.sp.remap + kb + p) : p;
    };
    // raw labels of parent row py: this lane's column and (lanes 0 / 31) the W / E halo
    auto load_row = [&](int py, int &L, int &Wh, int &Eh) {
      const bool iny = py >= 0 && py < pv.nby;
      const int32_t *row = pm + (size_t)py * pv.nbx;
      L = (inx && iny) ? row[px] : -1;
      Wh = (lane == 0 && iny && inx && px > 0) ? row[px - 1] : -1;
      Eh = (lane == 31 && iny && inx && px + 1 < pv.nbx) ? row[px + 1] : -1;
    };
    int Lp, Lc, Wc, Ec, t0, t1;
    load_row(tpy - 1, Lp, t0, t1);
    load_row(tpy, Lc, Wc, Ec);
    Lp = res(Lp);
    Lc = res(Lc);
    Wc = res(Wc);
    Ec = res(Ec);
    uint32_t *tw = a.bset + (size_t)t * 32;
#pragma unroll 1
    for (int r = 0; r < TY / 2; r++) {
      int Ln, Wn, En;
      load_row(tpy + r + 1, Ln, Wn, En);  // the next row's loads go out first
      bool gate = Lc >= 0;
      if (gate && a.gating == 1) gate = ld64_u8(a.sp.active + kb + Lc) != 0;
      int Wl = __shfl_up_sync(FULL, Lc, 1), El = __shfl_down_sync(FULL, Lc, 1);
      if (lane == 0) Wl = Wc;
      if (lane == 31) El = Ec;
      const bool dW = Wl >= 0 && Wl != Lc, dE = El >= 0 && El != Lc;
      const bool dN = Lp >= 0 && Lp != Lc;
      Ln = res(Ln);
      const bool dS = Ln >= 0 && Ln != Lc;
      const unsigned w0 = __ballot_sync(FULL, gate && (dW || dN));  // (cx, cy) = (0, 0)
      const unsigned w1 = __ballot_sync(FULL, gate && (dE || dN));  // (1, 0)
      const unsigned w2 = __ballot_sync(FULL, gate && (dW || dS));  // (0, 1)
      const unsigned w3 = __ballot_sync(FULL, gate && (dE || dS));  // (1, 1)
      if (lane == 0) {
        tw[0 * (TY / 2) + r] = w0;
        tw[1 * (TY / 2) + r] = w1;
        tw[2 * (TY / 2) + r] = w2;
        tw[3 * (TY / 2) + r] = w3;
      }
      Lp = Lc;
      Lc = Ln;
      Wc = res(Wn);
      Ec = res(En);
    }
  }
}

bool launch_bset_dyadic(const TransArgs &a, int sms, cudaStream_t s) {
  if (!(a.prev.uniform && a.next.uniform && a.prev.b == 2 * a.next.b && a.bset)) return false;
  const unsigned ntiles = (unsigned)(a.next.tiles_x * a.next.tiles_y) * (unsigned)a.B;
  // (small stages: too few tiles for a warp each, measured; RAPID_BSET_ROWS=2 forces it for tests)
  if ((g_bset_rows && ntiles >= 32768u) || g_bset_rows == 2)
    k_bset_dyadic_rows<<<std::min<unsigned>((ntiles + 7) / 8, (unsigned)sms * 8), 256, 0, s>>>(a);
  else
    k_bset_dyadic<<<std::min<unsigned>(ntiles, (unsigned)sms * 8), 256, 0, s>>>(a);
  return true;
}

// ------------------------------------------------------------------ RECOUNT
template <bool PIXEL>
__global__ void k_recount(const RecountArgs a) {
  const StageDev &st = a.st;
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * a.B;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = blockIdx.x * (size_t)blockDim.x; base < n; base += stride) {
    const size_t t = base + threadIdx.x;
    const bool valid = t < n;
    long long d[6] = {0, 0, 0, 0, 0, 0};
    int key = 0;
    if (valid) {
      const int img = (int)(t / nper);
      const size_t r = t - (size_t)img * nper;
      const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
      if (PIXEL) block_data_pix(a.image, a.H, a.W, img, gx, gy, d);
      else block_data_blk(st, img, gx, gy, d);
      key = img * a.M + st.map[t];
    }
    agg_sums(valid, key, d, false, a.rc, nullptr);
  }
}

__global__ void k_recount_check(const RecountArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += gridDim.x * blockDim.x) {
#pragma unroll
    for (int f = 0; f < 6; f++) {
      if (a.rc[(size_t)k * SUMW + f] != a.sp.sums[(size_t)k * SUMW + f]) *a.err = 1u;
      a.rc[(size_t)k * SUMW + f] = 0ull;
    }
  }
}

// ------------------------------------------------------------------ K9: final
__global__ void k_final_upsample(const FinalArgs a) {
  const bool rm = *a.remap_pending != 0u;
  const size_t nper = (size_t)a.H * a.W;
  const size_t n = nper * a.B;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
       t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int y = (int)(r / a.W), x = (int)(r - (size_t)y * a.W);
    int l = a.last.map[((size_t)img * a.last.nby + a.byp[y]) * a.last.nbx + a.bxp[x]];
    if (rm && !a.sp.alive[img * a.M + l]) l = a.sp.remap[img * a.M + l];
    a.labels[t] = l;
  }
}

__global__ void __launch_bounds__(128) k_final_remap(const FinalArgs a) {
  // in place on the map of `last` (== labels); merged-away labels only occur in worklist
  // tiles at gated stages (victims are active superpixels).  Persistent CTAs; chunks of 128
  // worklist tiles: with the adjacency pass's marks (vtile) every thread first decides one tile —
  // no merged-away superpixel has a boundary block there, so either none has a block there at
  // all or one covers the whole tile (a tile holding blocks of two labels has a boundary block
  // of each): its first block decides — and the CTA then rewrites the tiles that need it, one
  // per iteration: a thread reads 4 consecutive labels of 2 rows (16-B loads when rows allow)
  // and writes back only labels whose superpixel was merged away.
  if (*a.remap_pending == 0u) return;
  __shared__ uint32_t s_need[128];
  __shared__ unsigned s_n;
  const StageDev &st = a.last;
  const unsigned ntiles = a.worklist ? *a.nwork : (unsigned)(st.tiles_x * st.tiles_y) * (unsigned)a.B;
  const bool vec = (st.nbx & 3) == 0;
  const int u = threadIdx.x;
  // tiles decided per CTA iteration: up to 128 with marks (about ntiles / grid, so that every CTA
  // has work), one without (every tile is needed)
  const unsigned chunk = a.vtile ? max(1u, min(128u, ntiles / gridDim.x)) : 1u;
  for (unsigned c0 = blockIdx.x * chunk; c0 < ntiles; c0 += gridDim.x * chunk) {
    if (u == 0) s_n = 0;
    __syncthreads();
    if ((unsigned)u < chunk) {
      const unsigned w = c0 + u;
      if (w < ntiles) {
        const uint32_t tile = a.worklist ? (uint32_t)a.worklist[w] : w;
        bool need = true;
        if (a.vtile && a.vtile[tile] != a.vstamp) {
          const uint32_t r = fdiv(tile, st.fd_tx), img = fdiv(r, st.fd_ty);
          const int tx0 = (int)(tile - r * (uint32_t)st.tiles_x) * TX, ty0 = (int)(r - img * (uint32_t)st.tiles_y) * TY;
          const int l0 = a.labels[((size_t)img * st.nby + ty0) * st.nbx + tx0];
          need = !a.sp.alive[(int)img * a.M + l0];
        }
        if (need) s_need[atomicAdd(&s_n, 1u)] = tile;
      }
    }
    __syncthreads();
    // the needed tiles, a warp each (4 at a time per CTA): lane l takes 4 consecutive labels of
    // row (l >> 4) + 2 h of the tile, h = 0..7
    const unsigned nneed = s_n;
    // a single needed tile: all 4 warps on it (rows 2 g + (lane >> 4) + 8 h); several: a warp each
    const bool one = nneed == 1u;
    const int lane = u & 31, g = u >> 5;
    for (unsigned k = one ? 0u : (unsigned)g; k < nneed; k += one ? 1u : 4u) {
      const uint32_t tile = s_need[k];
      const uint32_t r = fdiv(tile, st.fd_tx), img = fdiv(r, st.fd_ty);
      const int gx = (int)(tile - r * (uint32_t)st.tiles_x) * TX + 4 * (lane & 15);
      const int gy0 = (int)(r - img * (uint32_t)st.tiles_y) * TY + (lane >> 4) + (one ? 2 * g : 0);
      const int kb = (int)img * a.M;
      const int nh = one ? 2 : TY / 2, step = one ? 8 : 2;
#pragma unroll 2
      for (int h = 0; h < nh; h++) {
        const int gy = gy0 + step * h;
        if (gy >= st.nby || gx >= st.nbx) continue;
        int32_t *p = a.labels + ((size_t)img * st.nby + gy) * st.nbx + gx;
        int l[4];
        if (vec) {
          const int4 v = *reinterpret_cast<const int4 *>(p);
          l[0] = v.x; l[1] = v.y; l[2] = v.z; l[3] = v.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++) l[q] = gx + q < st.nbx ? p[q] : -1;
        }
        bool dirty = false;
        int last = -1, res = -1;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (l[q] < 0) continue;
          if (l[q] != last) {
            last = l[q];
            res = a.sp.alive[kb + last] ? last : a.sp.remap[kb + last];
          }
          dirty |= res != l[q];
          l[q] = res;
        }
        if (!dirty) continue;
        if (vec) {
          *reinterpret_cast<int4 *>(p) = make_int4(l[0], l[1], l[2], l[3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++)
            if (gx + q < st.nbx) p[q] = l[q];
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------- profiling: algorithmic window blocks
// blocks within Chebyshev distance 1 of a block whose label can pass the active gate
__global__ void k_count_window(const StageDev st, const SpDev sp, int B, int M,
                               unsigned long long *out) {
  const size_t nper = (size_t)st.nbx * st.nby;
  const size_t n = nper * B;
  unsigned c = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = blockIdx.x * (size_t)blockDim.x; base < n; base += stride) {
    const size_t t = base + threadIdx.x;
    bool hit = false;
    if (t < n) {
      const int img = (int)(t / nper);
      const size_t r = t - (size_t)img * nper;
      const int gy = (int)(r / st.nbx), gx = (int)(r - (size_t)gy * st.nbx);
      const int32_t *map = st.map + (size_t)img * nper;
      for (int dy = -1; dy <= 1 && !hit; dy++)
        for (int dx = -1; dx <= 1 && !hit; dx++) {
          const int x = gx + dx, y = gy + dy;
          if (x < 0 || y < 0 || x >= st.nbx || y >= st.nby) continue;
          hit = sp.active[img * M + map[(size_t)y * st.nbx + x]] != 0;
        }
    }
    c += __popc(__ballot_sync(FULL, hit));
  }
  if (lane_id() == 0 && c) atomicAdd(out, (unsigned long long)c);
}

void launch_count_window(const StageDev &st, const SpDev &sp, int B, int M, unsigned long long *out,
                         cudaStream_t s);

// =================================================================== launch wrappers
static int grid_for(size_t n, int threads, int cap = 148 * 16) {
  size_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > (size_t)cap) g = cap;
  return (int)g;
}

void launch_init_sp(const InitArgs &a, cudaStream_t s) {
  k_init_sp<<<grid_for(a.K, 256), 256, 0, s>>>(a);
}

bool launch_pyramid_leaf24(const StageDev &st, const StageDev &up, const uint8_t *image, int H, int W, int B,
                           uint64_t *bsum, uint64_t *bsum_up, bool literal, cudaStream_t s) {
  if (!(st.uniform && up.uniform && st.b == 2 && up.b == 4 && W % 8 == 0 && H % 4 == 0 &&
        ((uintptr_t)image & 7u) == 0))
    return false;
  const size_t n = (size_t)(st.nbx / 4) * (st.nby / 2) * B;
  if (literal) k_pyramid_leaf24<true><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(st, up, image, H, W, B, bsum, bsum_up);
  else k_pyramid_leaf24<false><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(st, up, image, H, W, B, bsum, bsum_up);
  return true;
}

void launch_pyramid_leaf(const StageDev &st, const uint8_t *image, int H, int W, int B,
                         uint64_t *bsum, bool literal, cudaStream_t s) {
  const size_t n = (size_t)st.nbx * st.nby * B;
  if (st.uniform && st.b == 2 && W % 8 == 0 && ((uintptr_t)image & 7u) == 0)
    k_pyramid_leaf2<<<grid_for(n / 4, 256, 148 * 32), 256, 0, s>>>(st, image, H, W, B, bsum, literal);
  else
    k_pyramid_leaf<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(st, image, H, W, B, bsum, literal);
}

// Dyadic parent level (both uniform, b_parent = 2 b_child, child sums in u64 storage): a thread
// forms two adjacent parents of one row from two 32-B child runs (two child rows x four
// children), with 16-B loads and one 16-B store.
template <bool literal>
__global__ void k_pyramid_up2(const StageDev st, const StageDev ch, int B, uint64_t *__restrict__ bsum) {
  const int q = st.nbx / 2;  // parent pairs per row
  const size_t n = (size_t)q * st.nby * B;
  const uint64_t area = (uint64_t)st.b * (uint64_t)st.b;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const size_t row = t / q;  // img * nby + gy
    const int gx = 2 * (int)(t - row * q);
    const int img = (int)(row / st.nby), gy = (int)(row - (size_t)img * st.nby);
    const uint64_t *c0 = ch.bsum + ((size_t)img * ch.nby + 2 * gy) * ch.nbx + 2 * gx;
    const uint64_t *c1 = c0 + ch.nbx;
    const ulonglong2 a0 = __ldcs(reinterpret_cast<const ulonglong2 *>(c0)), a1 = __ldcs(reinterpret_cast<const ulonglong2 *>(c0) + 1);
    const ulonglong2 b0 = __ldcs(reinterpret_cast<const ulonglong2 *>(c1)), b1 = __ldcs(reinterpret_cast<const ulonglong2 *>(c1) + 1);
    uint64_t u0 = a0.x + a0.y + b0.x + b0.y, u1 = a1.x + a1.y + b1.x + b1.y;  // fields never carry
    if (literal) {
      u0 = lit_round(u0, area);
      u1 = lit_round(u1, area);
    }
    *reinterpret_cast<ulonglong2 *>(bsum + row * st.nbx + gx) = make_ulonglong2(u0, u1);
  }
}

void launch_pyramid_up(const StageDev &parent, const StageDev &child, int B, uint64_t *bsum, bool literal,
                       cudaStream_t s) {
  const size_t n = (size_t)parent.nbx * parent.nby * B;
  if (parent.uniform && child.uniform && parent.b == 2 * child.b && !child.bsum32 && parent.nbx % 2 == 0 &&
      child.nbx == 2 * parent.nbx && child.nby == 2 * parent.nby) {
    if (literal) k_pyramid_up2<true><<<grid_for(n / 2, 256, 148 * 16), 256, 0, s>>>(parent, child, B, bsum);
    else k_pyramid_up2<false><<<grid_for(n / 2, 256, 148 * 16), 256, 0, s>>>(parent, child, B, bsum);
    return;
  }
  k_pyramid_up<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(parent, child, B, bsum, literal);
}

void launch_init_map0(const InitArgs &a, cudaStream_t s) {
  const size_t n = (size_t)a.st0.nbx * a.st0.nby * a.B;
  k_init_map0<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
}

void launch_stats0(const InitArgs &a, cudaStream_t s) {
  const size_t n = (size_t)a.st0.nbx * a.st0.nby * a.B;
  if (a.st0.b == 1) k_stats0<true><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
  else k_stats0<false><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
}

void launch_snapshot(const SnapArgs &a, int grid, cudaStream_t s) {
  // one pass: every warp checks 128 superpixels' dirty bytes once (grid capped at `grid` x 2)
  const int g = grid_for(((size_t)a.K + 127) / 128 * 32, 256, 2 * grid);
  launch_pdl(k_snapshot, dim3(g), dim3(256), s, a);
}

int g_bset_rows = 1;  // RAPID_BSET_ROWS=0: the warp-per-parent-row boundary-set pass (k_bset_dyadic); 2: rows everywhere
int g_adj_minb8 = 1;  // k_merge_adj_bset at 32 registers, 8 CTAs per SM (RAPID_ADJ_MINB8=0: 39 registers, 6)
int g_adj_ilp = 1;  // RAPID_ADJ_ILP=1/2/4: rounds of set bits whose label loads k_merge_adj_bset issues together
int g_adj_tma = 0;  // RAPID_ADJ=tma: the victim adjacency from the TMA tile stream instead of the boundary sets

cudaError_t launch_merge_round(const MergeArgs &a, const void *tmap, int tgrid, int grid, cudaStream_t s,
                        int *nlaunch) {
  const int nchunks = (a.K + CHUNK - 1) / CHUNK;
  k_flag_count<<<nchunks, 256, 0, s>>>(a.sp.victim, a.K, a.chunk, a.victim_any);
  k_scan_chunks<<<1, 1024, 0, s>>>(a.chunk, nchunks, a.total, a.victim_any);
  k_flag_scatter<<<nchunks, 256, 0, s>>>(a.sp.victim, a.K, a.chunk, a.vlist, a.victim_any);
  k_merge_heads<<<grid, 256, 0, s>>>(a);
  const size_t nb = (size_t)a.st.nbx * a.st.nby * a.B;
  (void)nb;
  if (a.bset && a.worklist && g_adj_tma == 0) {  // (ungated stages: dense sets, the tile stream is faster)
    // one wave of resident CTAs (the loop strides over the worklist tiles)
    const void *fn = g_adj_ilp >= 4 ? (const void *)k_merge_adj_bset<4>
                   : g_adj_ilp >= 2 ? (const void *)k_merge_adj_bset<2>
                   : g_adj_minb8 ? (const void *)k_merge_adj_bset<1, 8> : (const void *)k_merge_adj_bset<1>;
    int nbk = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbk, fn, 256, 0);
    MergeArgs aa = a;
    void *args[] = {&aa};
    const cudaError_t e = cudaLaunchKernel(fn, dim3(sms * std::max(1, std::min(nbk, 8))), dim3(256), args, 0, s);
    if (e != cudaSuccess) return e;
  }
  else if (!launch_merge_adjacency_tma(a, tmap, tgrid, s)) k_merge_adjacency<<<148 * 8, 256, 0, s>>>(a);
  k_merge_degree<<<grid, 256, 0, s>>>(a);
  k_merge_scan_deg<<<1, 1024, 0, s>>>(a);
  k_merge_fill<<<grid, 256, 0, s>>>(a);
  {
    // co-resident grid computed per call (device / context of this launch), launch checked
    int nbk = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbk, k_merge_match, 256, 0);
    if (e != cudaSuccess) return e;
    const int coop_grid = sms * std::max(1, std::min(nbk, 4));
    MergeArgs aa = a;
    void *args[] = {&aa};
    e = cudaLaunchCooperativeKernel((const void *)k_merge_match, coop_grid, 256, args, 0, s);
    if (e != cudaSuccess) return e;
  }
  k_merge_apply<<<grid, 256, 0, s>>>(a);
  k_merge_cleanup<<<grid, 256, 0, s>>>(a);
  k_merge_done<<<1, 1, 0, s>>>(a);
  *nlaunch += 12;
  return cudaSuccess;
}

void launch_predict(const PredictArgs &a, int grid, cudaStream_t s, int *nlaunch) {
  if (a.y_model == 1) {  // f2: linear model on the superpixel features
    const size_t npx = (size_t)a.B * a.H * a.W, nb = (size_t)a.st.nbx * a.st.nby * a.B;
    const int b0 = a.st.b;
    if (a.st.uniform && (b0 == 8 || b0 == 16 || b0 == 32 || b0 == 64) && a.W % 8 == 0 && a.H % b0 == 0 &&
        a.W % b0 == 0 && ((uintptr_t)a.image & 7u) == 0) {
      const size_t nbands = (size_t)a.B * (a.H / b0) * ((a.W + 255) / 256);
      const int g = (int)std::min<size_t>(nbands, 148 * 8);
      if (b0 == 8) k_feat_q_band<8><<<g, 256, 0, s>>>(a);
      else if (b0 == 16) k_feat_q_band<16><<<g, 256, 0, s>>>(a);
      else if (b0 == 32) k_feat_q_band<32><<<g, 256, 0, s>>>(a);
      else k_feat_q_band<64><<<g, 256, 0, s>>>(a);
    } else {
      k_feat_q<<<grid_for(npx, 256, 148 * 16), 256, 0, s>>>(a);
    }
    k_feat_f1<<<grid_for(a.K, 256), 256, 0, s>>>(a);
    k_feat_adj<<<grid_for(nb, 256, 148 * 16), 256, 0, s>>>(a);
    k_feat_classify<<<grid_for(a.K, 256), 256, 0, s>>>(a);
    // restore the invariants of the borrowed buffers: RECOUNT scratch zero, merge hash empty
    cudaMemsetAsync(a.scratch, 0, sizeof(unsigned long long) * SUMW * (size_t)a.K, s);
    cudaMemsetAsync(a.hkeys, 0xff, sizeof(unsigned long long) * (a.hmask + 1), s);
    *nlaunch += 4;
  } else {
    k_predict_y<<<grid_for(a.K, 256), 256, 0, s>>>(a);
    *nlaunch += 1;
  }
  if (a.mask_rule != 1) {
    const size_t nb = (size_t)a.st.nbx * a.st.nby * a.B;
    k_predict_bsp<<<grid_for(nb, 256, 148 * 32), 256, 0, s>>>(a);
    *nlaunch += 1;
  }
  const int nchunks = (a.K + CHUNK - 1) / CHUNK;
  k_flag_count<<<nchunks, 256, 0, s>>>(a.sp.active, a.K, a.chunk, nullptr);
  k_scan_chunks<<<1, 1024, 0, s>>>(a.chunk, nchunks, a.total, nullptr);
  k_flag_scatter<<<nchunks, 256, 0, s>>>(a.sp.active, a.K, a.chunk, a.alist, nullptr);
  *nlaunch += 3;
}

bool launch_transition(const TransArgs &a, cudaStream_t s) {
  const unsigned ntiles = (unsigned)(a.next.tiles_x * a.next.tiles_y) * (unsigned)a.B;
  if (a.prev.uniform && a.next.uniform && a.prev.b == 2 * a.next.b) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = std::min<unsigned>(ntiles, (unsigned)sms * 16);
    if (a.bset) k_transition_dyadic<true><<<grid, 128, 0, s>>>(a);
    else k_transition_dyadic<false><<<grid, 128, 0, s>>>(a);
    return a.bset != nullptr;
  }
  k_transition<<<ntiles, 256, 0, s>>>(a);
  return false;
}

void launch_recount(const RecountArgs &a, bool pixel, int grid, cudaStream_t s, int *nlaunch) {
  const size_t n = (size_t)a.st.nbx * a.st.nby * a.B;
  if (pixel) k_recount<true><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
  else k_recount<false><<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
  k_recount_check<<<grid_for(a.K, 256), 256, 0, s>>>(a);
  *nlaunch += 2;
  (void)grid;
}

void launch_count_window(const StageDev &st, const SpDev &sp, int B, int M, unsigned long long *out,
                         cudaStream_t s) {
  const size_t n = (size_t)st.nbx * st.nby * B;
  k_count_window<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(st, sp, B, M, out);
}

void launch_final(const FinalArgs &a, bool upsample, cudaStream_t s) {
  const size_t n = (size_t)a.H * a.W * a.B;
  if (upsample) k_final_upsample<<<grid_for(n, 256, 148 * 32), 256, 0, s>>>(a);
  else k_final_remap<<<148 * 16, 128, 0, s>>>(a);
}

}  // namespace rapid
