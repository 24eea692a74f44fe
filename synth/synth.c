/*
 * synth.c — seeded, integer-only generator of synthetic H&E-like RGB u8 images.
 *
 * This is INPUT GENERATION ONLY. It holds none of the RAPID method's arithmetic
 * (no energy, no grid, no means): it is the one module both the CPU oracle's
 * tests and the CUDA path's tests/bench draw their inputs from (task rule ③).
 *
 * Recipe (SURVEY.md §8(d) "Synthetic inputs"; DESIGN.md §3 restates it):
 *   - PRNG: splitmix64 keyed by (seed, stream, index).
 *   - Tissue regions: R Voronoi seeds, uniform integer positions; nearest seed by
 *     exact expanding-ring search over a bucket grid of side ceil(sqrt(H*W/R));
 *     squared Euclidean distance, ties -> lower seed index.
 *   - Region class from the hash: pink (230,170,200) p=0.3, purple (120,70,150)
 *     p=0.2, white (240,235,240) p=0.5; flat colour per region.
 *   - Background: a coarse 64-seed Voronoi; exactly round(f*64) of its cells
 *     (chosen by a seeded Fisher-Yates permutation) are white background.
 *   - Nuclei: centres uniform, skipped when the centre lies in background;
 *     integer semi-axes in [3,8]; one of 8 orientations (Q12 cos/sin table);
 *     dark purple (70,35,100); painted in index order.
 *   - Noise: per channel, Irwin-Hall(12) of 16-bit uniforms scaled to sigma,
 *     rounded, added, clamped to [0,255].
 * Output: u8 [H][W][3], row-major, channel-last.
 *
 * Deterministic for a given parameter set, independent of the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  uint64_t seed;
  int32_t H, W;
  int32_t n_regions;    /* Voronoi tissue regions (>= 1) */
  int32_t n_nuclei;     /* elliptical blobs */
  int32_t bg_permille;  /* background fraction f in 1/1000 */
  int32_t noise_sigma;  /* Gaussian-like noise sigma (intensity units) */
} synth_params;

static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t index) {
  return splitmix64(splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull)) + index);
}

/* ---------- exact nearest-seed search over a bucket grid ---------- */
typedef struct {
  int n, G, nbx, nby;
  const int32_t *sx, *sy;
  int32_t *start; /* nbx*nby+1 */
  int32_t *ids;   /* seed ids, bucket-major, ascending within a bucket */
} vgrid;

static int isqrt_ceil(uint64_t v) {
  uint64_t r = (uint64_t)sqrt((double)v);
  while (r * r < v) r++;
  while (r > 0 && (r - 1) * (r - 1) >= v) r--;
  return (int)r;
}

static int vgrid_build(vgrid *g, int n, const int32_t *sx, const int32_t *sy, int H, int W) {
  g->n = n; g->sx = sx; g->sy = sy;
  uint64_t area = (uint64_t)H * (uint64_t)W;
  int G = isqrt_ceil((area + (uint64_t)n - 1) / (uint64_t)n);
  if (G < 1) G = 1;
  g->G = G;
  g->nbx = (W + G - 1) / G;
  g->nby = (H + G - 1) / G;
  size_t nb = (size_t)g->nbx * g->nby;
  g->start = (int32_t *)calloc(nb + 1, sizeof(int32_t));
  g->ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  if (!g->start || !g->ids) return -1;
  for (int k = 0; k < n; k++) g->start[(size_t)(sy[k] / G) * g->nbx + sx[k] / G + 1]++;
  for (size_t b = 0; b < nb; b++) g->start[b + 1] += g->start[b];
  int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * nb);
  if (!fill) return -1;
  memcpy(fill, g->start, sizeof(int32_t) * nb);
  for (int k = 0; k < n; k++) g->ids[fill[(size_t)(sy[k] / G) * g->nbx + sx[k] / G]++] = k;
  free(fill);
  return 0;
}

static void vgrid_free(vgrid *g) { free(g->start); free(g->ids); }

static inline void scan_bucket(const vgrid *g, int bx, int by, int x, int y,
                               int64_t *best_d, int *best) {
  if (bx < 0 || by < 0 || bx >= g->nbx || by >= g->nby) return;
  size_t b = (size_t)by * g->nbx + bx;
  for (int t = g->start[b]; t < g->start[b + 1]; t++) {
    int k = g->ids[t];
    int64_t dx = (int64_t)g->sx[k] - x, dy = (int64_t)g->sy[k] - y;
    int64_t d = dx * dx + dy * dy;
    if (d < *best_d || (d == *best_d && k < *best)) { *best_d = d; *best = k; }
  }
}

/* nearest seed to integer pixel (x,y): exact, ties to the lower seed index */
static int vgrid_nearest(const vgrid *g, int x, int y) {
  int bx = x / g->G, by = y / g->G;
  int64_t best_d = INT64_MAX;
  int best = -1;
  int rmax = g->nbx > g->nby ? g->nbx : g->nby;
  for (int r = 0; r <= rmax; r++) {
    if (r == 0) {
      scan_bucket(g, bx, by, x, y, &best_d, &best);
    } else {
      for (int i = -r; i <= r; i++) {
        scan_bucket(g, bx + i, by - r, x, y, &best_d, &best);
        scan_bucket(g, bx + i, by + r, x, y, &best_d, &best);
      }
      for (int j = -r + 1; j <= r - 1; j++) {
        scan_bucket(g, bx - r, by + j, x, y, &best_d, &best);
        scan_bucket(g, bx + r, by + j, x, y, &best_d, &best);
      }
    }
    /* every seed outside rings 0..r is at least r*G+1 away along one axis */
    int64_t lim = (int64_t)r * g->G + 1;
    if (best >= 0 && best_d < lim * lim) break;
  }
  return best;
}

/* Q12 cos/sin for angles k*pi/8, k = 0..7 */
static const int32_t COSQ12[8] = {4096, 3784, 2896, 1567, 0, -1567, -2896, -3784};
static const int32_t SINQ12[8] = {0, 1567, 2896, 3784, 4096, 3784, 2896, 1567};

static const uint8_t COL_PINK[3] = {230, 170, 200};
static const uint8_t COL_PURPLE[3] = {120, 70, 150};
static const uint8_t COL_WHITE[3] = {240, 235, 240};
static const uint8_t COL_NUC[3] = {70, 35, 100};

enum { ST_REG = 1, ST_CLASS = 2, ST_BG = 3, ST_BGPERM = 4, ST_NUC = 5, ST_NOISE = 6 };

/* One generator for both outputs: the RGB image (out, may be NULL) and the ground-truth
 * segment map (seg, may be NULL): segment id = tissue region k (0..R-1), background cell
 * R + j (j < 64), or nucleus R + 64 + k for the blob painted last at the pixel. */
static int synth_generate(const synth_params *p, uint8_t *out, int32_t *seg, int nthreads) {
  const int H = p->H, W = p->W;
  if (H < 1 || W < 1 || p->n_regions < 1 || p->n_nuclei < 0) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const uint64_t seed = p->seed;
  /* tissue regions */
  int R = p->n_regions;
  int32_t *rx = (int32_t *)malloc(sizeof(int32_t) * R), *ry = (int32_t *)malloc(sizeof(int32_t) * R);
  uint8_t *rcls = (uint8_t *)malloc(R);
  for (int k = 0; k < R; k++) {
    rx[k] = (int32_t)(rnd(seed, ST_REG, 2 * (uint64_t)k) % (uint64_t)W);
    ry[k] = (int32_t)(rnd(seed, ST_REG, 2 * (uint64_t)k + 1) % (uint64_t)H);
    uint64_t u = rnd(seed, ST_CLASS, (uint64_t)k) % 1000u;
    rcls[k] = u < 300 ? 0 : (u < 500 ? 1 : 2);
  }
  /* background cells */
  const int NB = 64;
  int32_t bx[64], by[64];
  uint8_t isbg[64];
  int perm[64];
  for (int k = 0; k < NB; k++) {
    bx[k] = (int32_t)(rnd(seed, ST_BG, 2 * (uint64_t)k) % (uint64_t)W);
    by[k] = (int32_t)(rnd(seed, ST_BG, 2 * (uint64_t)k + 1) % (uint64_t)H);
    perm[k] = k;
  }
  for (int k = NB - 1; k > 0; k--) {
    int j = (int)(rnd(seed, ST_BGPERM, (uint64_t)k) % (uint64_t)(k + 1));
    int t = perm[k]; perm[k] = perm[j]; perm[j] = t;
  }
  int nbg = (p->bg_permille * NB + 500) / 1000;
  memset(isbg, 0, sizeof isbg);
  for (int k = 0; k < nbg; k++) isbg[perm[k]] = 1;

  vgrid vr, vb;
  if (vgrid_build(&vr, R, rx, ry, H, W) || vgrid_build(&vb, NB, bx, by, H, W)) return -2;

  /* base colours */
#pragma omp parallel for schedule(dynamic, 4)
  for (int y = 0; y < H; y++) {
    uint8_t *row = out ? out + (size_t)y * W * 3 : NULL;
    for (int x = 0; x < W; x++) {
      const uint8_t *c;
      const int jb = nbg > 0 ? vgrid_nearest(&vb, x, y) : 0;
      int sid;
      if (nbg > 0 && isbg[jb]) {
        c = COL_WHITE;
        sid = R + jb;
      } else {
        int k = vgrid_nearest(&vr, x, y);
        c = rcls[k] == 0 ? COL_PINK : (rcls[k] == 1 ? COL_PURPLE : COL_WHITE);
        sid = k;
      }
      if (row) { row[3 * x] = c[0]; row[3 * x + 1] = c[1]; row[3 * x + 2] = c[2]; }
      if (seg) seg[(size_t)y * W + x] = sid;
    }
  }
  /* nuclei, painted in index order (sequential: later blobs overwrite earlier) */
  for (int64_t k = 0; k < p->n_nuclei; k++) {
    int cx = (int)(rnd(seed, ST_NUC, 4 * (uint64_t)k) % (uint64_t)W);
    int cy = (int)(rnd(seed, ST_NUC, 4 * (uint64_t)k + 1) % (uint64_t)H);
    if (nbg > 0 && isbg[vgrid_nearest(&vb, cx, cy)]) continue;
    uint64_t h = rnd(seed, ST_NUC, 4 * (uint64_t)k + 2);
    int64_t a = 3 + (int64_t)(h % 6u), b = 3 + (int64_t)((h >> 8) % 6u);
    int o = (int)((h >> 16) & 7u);
    int64_t cs = COSQ12[o], sn = SINQ12[o];
    int64_t a2b2 = a * a * b * b * (int64_t)(1 << 24);
    for (int y = cy - 8; y <= cy + 8; y++) {
      if (y < 0 || y >= H) continue;
      for (int x = cx - 8; x <= cx + 8; x++) {
        if (x < 0 || x >= W) continue;
        int64_t dx = x - cx, dy = y - cy;
        int64_t u = dx * cs + dy * sn, v = -dx * sn + dy * cs; /* Q12 */
        if (u * u * b * b + v * v * a * a <= a2b2) {
          if (out) {
            uint8_t *px = out + ((size_t)y * W + x) * 3;
            px[0] = COL_NUC[0]; px[1] = COL_NUC[1]; px[2] = COL_NUC[2];
          }
          if (seg) seg[(size_t)y * W + x] = (int32_t)(R + NB + k);
        }
      }
    }
  }
  /* noise: Irwin-Hall(12) of 16-bit uniforms; sum has mean 12*65535/2, sd 65536*1 (approx) */
  const int64_t sig = p->noise_sigma;
  if (out && sig > 0) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; y++) {
      for (int x = 0; x < W; x++) {
        uint64_t pix = (uint64_t)y * (uint64_t)W + (uint64_t)x;
        uint8_t *px = out + pix * 3;
        for (int ch = 0; ch < 3; ch++) {
          int64_t s = 0;
          for (int t = 0; t < 3; t++) {
            uint64_t h = rnd(seed, ST_NOISE, pix * 9 + (uint64_t)ch * 3 + (uint64_t)t);
            s += (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) +
                 (int64_t)((h >> 32) & 0xFFFF) + (int64_t)(h >> 48);
          }
          /* (2s - 12*65535) / 2 is centred; / 65536 gives unit variance; x sigma; round */
          int64_t num = (2 * s - 12 * 65535) * sig;
          int64_t nz = num >= 0 ? (num + 65536) >> 17 : -((-num + 65536) >> 17);
          int64_t v = (int64_t)px[ch] + nz;
          px[ch] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
        }
      }
    }
  }
  vgrid_free(&vr); vgrid_free(&vb);
  free(rx); free(ry); free(rcls);
  return 0;
}

int synth_image(const synth_params *p, uint8_t *out, int nthreads) { return synth_generate(p, out, NULL, nthreads); }

/* ground-truth segment map of the same parameters (int32 [H][W]) */
int synth_segments(const synth_params *p, int32_t *seg, int nthreads) { return synth_generate(p, NULL, seg, nthreads); }

/* hash helper exposed for configs that derive per-tile parameters (config 5) */
uint64_t synth_hash(uint64_t seed, uint64_t stream, uint64_t index) { return rnd(seed, stream, index); }
