// quality.cu — SURVEY §8(f) f4: segmentation quality of a label map against a ground-truth
// segment map on the GPU (under-segmentation error UE and boundary recall BR, the
// metrics of the paper's §4.2; definitions in include/rapid.h).
//
//   Q1 k_q_pairs    one pass over the pixels: warp runs of equal (superpixel, segment) pairs
//                   add their length to an open-addressing pair histogram, runs of equal
//                   superpixels to the superpixel sizes; the superpixel-boundary flag of every
//                   pixel (a 4-neighbour with another label) is written as a byte.
//   Q2 k_q_leak     over the histogram: leak += min(|sp n S|, |sp| - |sp n S|).
//   Q3 k_q_recall   GT boundary pixels, and those with a superpixel-boundary pixel within
//                   Chebyshev distance eps.
// Product code: never includes or links anything under oracle/.
#include <algorithm>

#include "kernels.cuh"

namespace rapid {

constexpr unsigned long long QEMPTY = ~0ull;

__device__ __forceinline__ unsigned long long qmix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  return k;
}

__device__ void q_add(const QualityArgs &a, unsigned long long key, uint32_t c) {
  unsigned long long h = qmix(key) & a.cmask;
  for (unsigned long long probes = 0; probes <= a.cmask; probes++) {
    const unsigned long long seen = *reinterpret_cast<volatile unsigned long long *>(&a.keys[h]);
    if (seen == key) {
      atomicAdd(&a.cnt[h], c);
      return;
    }
    if (seen == QEMPTY) {
      const unsigned long long old = atomicCAS(&a.keys[h], QEMPTY, key);
      if (old == QEMPTY) {
        atomicAdd(&a.acc[3], 1ull);
        atomicAdd(&a.cnt[h], c);
        return;
      }
      if (old == key) {
        atomicAdd(&a.cnt[h], c);
        return;
      }
    }
    h = (h + 1) & a.cmask;
  }
  atomicOr(&a.acc[4], 1ull);  // histogram full
}

__global__ void __launch_bounds__(256) k_q_pairs(const QualityArgs a) {
  const size_t nper = (size_t)a.H * a.W, n = nper * a.B;
  const int lane = lane_id();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = blockIdx.x * (size_t)blockDim.x; base < n; base += stride) {  // warp-uniform
    const size_t t = base + threadIdx.x;
    const bool valid = t < n;
    int sp = 0, g = 0, img = 0;
    if (valid) {
      img = (int)(t / nper);
      const size_t r = t - (size_t)img * nper;
      const int y = (int)(r / a.W), x = (int)(r - (size_t)y * a.W);
      sp = a.labels[t];
      g = a.gt[t];
      if (sp < 0 || sp >= a.M || g < 0) atomicOr(&a.acc[4], 2ull);  // out-of-range id
      sp = min(max(sp, 0), a.M - 1);
      const int32_t *L = a.labels + (size_t)img * nper;
      const size_t o = (size_t)y * a.W + x;
      const int v = L[o];
      const bool b = (x > 0 && L[o - 1] != v) || (x + 1 < a.W && L[o + 1] != v) || (y > 0 && L[o - a.W] != v) ||
                     (y + 1 < a.H && L[o + a.W] != v);
      a.spb[t] = b ? 1 : 0;
    }
    const int key_sp = img * a.M + sp;
    // runs of adjacent lanes with equal pairs / equal superpixels (consecutive pixels)
    const unsigned long long pk = valid ? ((unsigned long long)(unsigned)key_sp << 32) | (unsigned)g : QEMPTY;
    const unsigned long long pkp = __shfl_up_sync(FULL, pk, 1);
    const unsigned long long pkn = __shfl_down_sync(FULL, pk, 1);
    const bool pstart = lane == 0 || pkp != pk, pend = lane == 31 || pkn != pk;
    const unsigned sm = __ballot_sync(FULL, pstart);
    const int pfirst = 31 - __clz(sm & ((2u << lane) - 1u));
    if (valid && pend) q_add(a, pk, (uint32_t)(lane - pfirst + 1));
    const int sk = valid ? key_sp : -1 - lane;
    const int skp = __shfl_up_sync(FULL, sk, 1), skn = __shfl_down_sync(FULL, sk, 1);
    const bool sstart = lane == 0 || skp != sk, send = lane == 31 || skn != sk;
    const unsigned ss = __ballot_sync(FULL, sstart);
    const int sfirst = 31 - __clz(ss & ((2u << lane) - 1u));
    if (valid && send) atomicAdd(&a.size[key_sp], (uint32_t)(lane - sfirst + 1));
  }
}

__global__ void __launch_bounds__(256) k_q_leak(const QualityArgs a) {
  unsigned long long leak = 0;
  for (unsigned long long h = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; h <= a.cmask;
       h += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k = a.keys[h];
    if (k == QEMPTY) continue;
    const uint32_t c = a.cnt[h], s = a.size[k >> 32];
    leak += c < s - c ? c : s - c;
  }
  leak = warp_sum_ll((long long)leak);
  if (lane_id() == 0 && leak) atomicAdd(&a.acc[0], leak);
}

__global__ void __launch_bounds__(256) k_q_recall(const QualityArgs a) {
  const size_t nper = (size_t)a.H * a.W, n = nper * a.B;
  unsigned long long gtb = 0, cov = 0;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const int img = (int)(t / nper);
    const size_t r = t - (size_t)img * nper;
    const int y = (int)(r / a.W), x = (int)(r - (size_t)y * a.W);
    const int32_t *G = a.gt + (size_t)img * nper;
    const size_t o = (size_t)y * a.W + x;
    const int v = G[o];
    const bool b = (x > 0 && G[o - 1] != v) || (x + 1 < a.W && G[o + 1] != v) || (y > 0 && G[o - a.W] != v) ||
                   (y + 1 < a.H && G[o + a.W] != v);
    if (!b) continue;
    gtb++;
    const uint8_t *S = a.spb + (size_t)img * nper;
    bool hit = false;
    for (int yy = max(0, y - a.eps); yy <= min(a.H - 1, y + a.eps) && !hit; yy++)
      for (int xx = max(0, x - a.eps); xx <= min(a.W - 1, x + a.eps) && !hit; xx++)
        hit = S[(size_t)yy * a.W + xx] != 0;
    cov += hit;
  }
  gtb = warp_sum_ll((long long)gtb);
  cov = warp_sum_ll((long long)cov);
  if (lane_id() == 0) {
    if (gtb) atomicAdd(&a.acc[1], gtb);
    if (cov) atomicAdd(&a.acc[2], cov);
  }
}

void launch_quality(const QualityArgs &a, int sms, cudaStream_t s) {
  const size_t n = (size_t)a.B * a.H * a.W;
  const int g = (int)std::min<size_t>((n + 255) / 256, (size_t)sms * 16);
  k_q_pairs<<<g, 256, 0, s>>>(a);
  k_q_leak<<<sms * 8, 256, 0, s>>>(a);
  k_q_recall<<<g, 256, 0, s>>>(a);
}

}  // namespace rapid
