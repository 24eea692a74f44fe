/*
 * oracle.c — plain, slow, single-threaded CPU oracle of the RAPID / CTFTPS
 * refinement hot path (arXiv 1704.02083).  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * It follows the paper's algorithm in the paper's order, with the readings of
 * SURVEY.md §8(c) (restated in DESIGN.md §2) wherever the paper is silent:
 *
 *   O1 grid init ............ RAPID l.1, "initializing superpixels with grids"
 *   O2 stage geometry ....... RAPID l.6 "Initialize each block with smaller regular grid"
 *   O3 block sums ........... P:90 (§2.2), P:205-213 (Eq. 8, A23: exact full-resolution sums)
 *   O4 S_1 .................. RAPID l.9-10
 *   O5 snapshot means ....... RAPID l.18, A4 (frozen per phase), A24 (rounding)
 *   O6 propose .............. Eq. 1, Eq. 2, Eq. 3, E_topo,
 *                             RAPID l.14-22, Eq. 7 gate
 *   O6' commit .............. RAPID l.25-26, A19 all-or-nothing budget
 *   O7 merge round .......... §3.1 Eqs. 4-5, A12-A16
 *   O8 prediction ........... RAPID l.3-4, Eq. 6, A20-A22
 *   O9 transition/final ..... RAPID l.7-8, §2.2, Table 1 grain
 *
 * Arithmetic: integers only; energy differences in __int128 (exact).  The
 * parity-coloured schedule (A5/A6) replaces the paper's queue order.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

#define FRAC 8 /* F: fractional bits of the snapshot means (A24) */

/* ------------------------------------------------------------------ O1 -- */
/* r*c = M with the squarest cells: minimise max(W r, H c)/min(W r, H c);
 * among equal ratios keep fewer rows; only factorisations that fit (c<=W, r<=H). */
int orc_grid(int H, int W, int M, int *rows, int *cols) {
  if (H < 1 || W < 1 || M < 1) return ORC_E_ARG;
  int best_r = 0, best_c = 0;
  i128 bmx = 0, bmn = 1;
  for (int r = 1; r <= M; r++) {
    if (M % r != 0) continue;
    int c = M / r;
    if (c > W || r > H) continue;
    i128 a = (i128)W * r, b = (i128)H * c;
    i128 mx = a > b ? a : b, mn = a > b ? b : a;
    if (best_r == 0 || mx * bmn < bmx * mn) {
      best_r = r; best_c = c; bmx = mx; bmn = mn;
    }
  }
  if (best_r == 0) return ORC_E_ARG;
  *rows = best_r;
  *cols = best_c;
  return ORC_OK;
}

/* ------------------------------------------------------------------ O2 -- */
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* sorted unique({k*b : k*b < len} U cuts U {len}); returns the count, or -1 */
int orc_stage_axis(int len, int b, const int32_t *cuts, int ncuts, int32_t *out, int cap) {
  int n = 0;
  int need = len / b + 2 + ncuts;
  int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)need);
  if (!tmp) return -1;
  for (int k = 0; (int64_t)k * b < len; k++) tmp[n++] = k * b;
  for (int k = 0; k < ncuts; k++) tmp[n++] = cuts[k];
  tmp[n++] = len;
  qsort(tmp, (size_t)n, sizeof(int32_t), cmp_i32);
  int m = 0;
  for (int k = 0; k < n; k++)
    if (m == 0 || tmp[k] != tmp[m - 1]) tmp[m++] = tmp[k];
  if (m > cap) { free(tmp); return -1; }
  memcpy(out, tmp, sizeof(int32_t) * (size_t)m);
  free(tmp);
  return m;
}

/* ------------------------------------------------------------------ A9 -- */
/* Yokoi 4-connectivity number of the 8-ring x_0..x_7 = N,NE,E,SE,S,SW,W,NW:
 * C4 = sum_{k in N,E,S,W} (x_k - x_k x_{k+1} x_{k+2}); simple point iff C4 == 1. */
int orc_yokoi_c4(int m) {
  int x[8];
  for (int k = 0; k < 8; k++) x[k] = (m >> k) & 1;
  int c = 0;
  for (int k = 0; k < 8; k += 2) c += x[k] - x[k] * x[(k + 1) % 8] * x[(k + 2) % 8];
  return c;
}

/* ------------------------------------------------------------------ O5 -- */
/* q = round-half-up(2^F * S / n) = floor((2^(F+1) S + n) / (2n)), S >= 0, n > 0 */
/* A33 (f3): a colour channel's snapshot mean is O5's rounding of S / n clamped to the
 * intensity range [0, 255] — a sum outside [0, 255 n] arises only from the literal pyramid's
 * synthesised block data, where blocks leave a superpixel with finer data than they entered
 * with; otherwise this is orc_round_mean. */
void orc_colour_mean(int64_t S, int64_t n, int64_t *q) {
  if (S < 0) *q = 0;
  else if (S > 255 * n) *q = (int64_t)255 << FRAC;
  else orc_round_mean(S, n, q);
}

void orc_round_mean(int64_t S, int64_t n, int64_t *q) {
  i128 num = ((i128)S << (FRAC + 1)) + n;
  *q = (int64_t)(num / (2 * (i128)n));
}

/* ------------------------------------------------------------ helpers ---- */
static const int RING_DX[8] = {0, 1, 1, 1, 0, -1, -1, -1}; /* N NE E SE S SW W NW */
static const int RING_DY[8] = {-1, -1, 0, 1, 1, 1, 0, -1};
static const int N4_DX[4] = {0, 1, 0, -1}; /* N E S W */
static const int N4_DY[4] = {-1, 0, 1, 0};

typedef struct {
  int nbx, nby;
  int32_t *xs, *ys; /* nbx+1, nby+1 boundaries */
  int64_t *bd;      /* per block: n, sum_r, sum_g, sum_b, sum_x, sum_y (NULL at b=1) */
} stage_t;

typedef struct {
  /* inputs */
  const uint8_t *I;
  int H, W, M, img;
  const orc_params *p;
  orc_debug *dbg;
  /* grid */
  int rows, cols;
  int32_t *X, *Y;
  /* per superpixel */
  int64_t *S;      /* [M][6]: n, r, g, b, x, y */
  int32_t *init;
  uint8_t *alive, *active, *victim, *locked;
  int8_t *y;
  int64_t *cq;     /* [M][3] snapshot colour means, 2^F units */
  int64_t *mq;     /* [M][2] snapshot position means, 2^F units */
  int64_t *nsnap;  /* [M] snapshot size */
  int64_t *out;    /* [M] proposed outflow this phase */
  int32_t *remap;
  /* stages */
  stage_t st[ORC_MAX_STAGES];
  int32_t *L;      /* current stage map */
  int cur;         /* current stage */
} seg_t;

static int64_t *cnt_ptr(seg_t *g, int s, int t, int ph) {
  if (!g->dbg || !g->dbg->phase_counters) return NULL;
  return g->dbg->phase_counters + (((size_t)s * ORC_MAX_SWEEPS + (size_t)t) * 4 + (size_t)ph) * ORC_NCNT;
}

static int32_t lab(const seg_t *g, int i, int j) {
  const stage_t *st = &g->st[g->cur];
  if (i < 0 || j < 0 || i >= st->nbx || j >= st->nby) return -1; /* A26: no neighbour */
  return g->L[(size_t)j * st->nbx + i];
}

/* O3: block data by direct summation over the block's pixels */
static void block_direct(const seg_t *g, int x0, int x1, int y0, int y1, int64_t d[6]) {
  memset(d, 0, sizeof(int64_t) * 6);
  for (int y = y0; y < y1; y++)
    for (int x = x0; x < x1; x++) {
      const uint8_t *px = g->I + ((size_t)y * g->W + x) * 3;
      d[0] += 1;
      d[1] += px[0]; d[2] += px[1]; d[3] += px[2];
      d[4] += x; d[5] += y;
    }
}

static void block_data(const seg_t *g, int s, int i, int j, int64_t d[6]) {
  const stage_t *st = &g->st[s];
  if (st->bd) {
    memcpy(d, st->bd + ((size_t)j * st->nbx + i) * 6, sizeof(int64_t) * 6);
  } else {
    block_direct(g, st->xs[i], st->xs[i + 1], st->ys[j], st->ys[j + 1], d);
  }
}

static void snapshot(seg_t *g) { /* O5 */
  for (int k = 0; k < g->M; k++) {
    const int64_t *s = g->S + (size_t)k * 6;
    g->nsnap[k] = s[0];
    if (!g->alive[k] || s[0] <= 0) continue;
    for (int ch = 0; ch < 3; ch++) orc_colour_mean(s[1 + ch], s[0], &g->cq[(size_t)k * 3 + ch]);
    for (int d = 0; d < 2; d++) orc_round_mean(s[4 + d], s[0], &g->mq[(size_t)k * 2 + d]);
  }
}

/* Weighted energy in units of 2^(16+4F) of the real energy (A1, O6 step 5) */
static i128 weigh(const orc_params *p, i128 dC, i128 dP, i128 dB2) {
  i128 Wc = (i128)1 << (2 * FRAC + 16);
  i128 Wp = (i128)p->lambda_pos_q16 << (2 * FRAC);
  i128 Wb = (i128)p->lambda_b_q16 << (4 * FRAC);
  return Wc * dC + Wp * dP + Wb * dB2;
}

/* colour and position parts of relabelling a pixel set with data d from A to B
 * under the frozen means (Eq. 1's E_col and E_pos): 2^(2F) x the real change. */
static void delta_cp(const seg_t *g, int A, int B, const int64_t d[6], i128 *dC, i128 *dP) {
  i128 c = 0, q = 0;
  for (int ch = 0; ch < 3; ch++) {
    i128 a = g->cq[(size_t)A * 3 + ch], b = g->cq[(size_t)B * 3 + ch];
    c += (i128)d[0] * (b * b - a * a) - ((i128)d[1 + ch] << (FRAC + 1)) * (b - a);
  }
  for (int k = 0; k < 2; k++) {
    i128 a = g->mq[(size_t)A * 2 + k], b = g->mq[(size_t)B * 2 + k];
    q += (i128)d[0] * (b * b - a * a) - ((i128)d[4 + k] << (FRAC + 1)) * (b - a);
  }
  *dC = c;
  *dP = q;
}

/* O6 steps 4-6 for one block with label A, 4-neighbour labels nq (N,E,S,W; -1 = none),
 * shared edge lengths eq and block data d: candidates are the distinct neighbour labels
 * other than A (A8); dE (Eq. 1 with Eq. 2, frozen quantised means from `means`) per
 * candidate; argmin with ties to the smallest label (A7).  Returns 0 if no candidate. */
typedef void (*means_fn)(const void *ctx, int32_t label, int64_t m[5]);

static int argmin_move(const orc_params *p, int32_t A, const int32_t nq[4], const int64_t eq[4],
                       const int64_t d[6], means_fn means, const void *ctx, int32_t *B_out, i128 *E_out) {
  int64_t mA[5];
  means(ctx, A, mA);
  int have = 0;
  int32_t bestB = -1;
  i128 bestE = 0;
  for (int q = 0; q < 4; q++) {
    int32_t B = nq[q];
    if (B < 0 || B == A) continue;
    int dup = 0;
    for (int r = 0; r < q; r++)
      if (nq[r] == B) dup = 1;
    if (dup) continue;
    int64_t mB[5];
    means(ctx, B, mB);
    i128 dC = 0, dP = 0, dB2 = 0;
    for (int ch = 0; ch < 3; ch++) /* E_col: n(cB^2 - cA^2) - 2^(F+1) S (cB - cA) */
      dC += (i128)d[0] * ((i128)mB[ch] * mB[ch] - (i128)mA[ch] * mA[ch]) -
            ((i128)d[1 + ch] << (FRAC + 1)) * ((i128)mB[ch] - mA[ch]);
    for (int k = 0; k < 2; k++) /* E_pos, same form with the position means */
      dP += (i128)d[0] * ((i128)mB[3 + k] * mB[3 + k] - (i128)mA[3 + k] * mA[3 + k]) -
            ((i128)d[4 + k] << (FRAC + 1)) * ((i128)mB[3 + k] - mA[3 + k]);
    for (int r = 0; r < 4; r++)
      if (nq[r] >= 0) dB2 += (i128)eq[r] * ((nq[r] != B) - (nq[r] != A));
    dB2 *= 2; /* ordered pairs (A3) */
    i128 E = weigh(p, dC, dP, dB2);
    if (!have || E < bestE || (E == bestE && B < bestB)) {
      have = 1; bestE = E; bestB = B;
    }
  }
  *B_out = bestB;
  *E_out = bestE;
  return have;
}

static void seg_means(const void *ctx, int32_t l, int64_t m[5]) {
  const seg_t *g = (const seg_t *)ctx;
  for (int ch = 0; ch < 3; ch++) m[ch] = g->cq[(size_t)l * 3 + ch];
  for (int k = 0; k < 2; k++) m[3 + k] = g->mq[(size_t)l * 2 + k];
}

typedef struct { const int32_t *labels; const int64_t *means; } win_means_t;
static void win_means(const void *ctx, int32_t l, int64_t m[5]) {
  const win_means_t *w = (const win_means_t *)ctx;
  for (int c = 0; c < 9; c++)
    if (w->labels[c] == l) {
      memcpy(m, w->means + 5 * c, 5 * sizeof(int64_t));
      return;
    }
  memset(m, 0, 5 * sizeof(int64_t));
}

/* One block's O6 decision in isolation (sampled parity checks at sizes the whole oracle cannot
 * run): win = 3x3 labels row-major (-1 = outside), means of each window cell's label
 * (cq_r, cq_g, cq_b, mq_x, mq_y in 2^F units), block data d, edge lengths e (N, E, S, W).
 * Returns 0 not a boundary block, 1 not a simple point, 2 no move (min dE >= 0), 3 move to
 * *B_out with *dE (hi/lo of the int128).  No mask gate, no size gate. */
int orc_block_move(const int32_t *win, const int64_t *means, const int64_t *d, const int64_t *e,
                   const orc_params *p, int32_t *B_out, int64_t *dE_hi, uint64_t *dE_lo) {
  const int32_t A = win[4];
  const int32_t nq[4] = {win[1], win[5], win[7], win[3]}; /* N, E, S, W */
  int bnd = 0;
  for (int q = 0; q < 4; q++)
    if (nq[q] >= 0 && nq[q] != A) bnd = 1;
  if (!bnd) return 0;
  static const int RING[8] = {1, 2, 5, 8, 7, 6, 3, 0}; /* N NE E SE S SW W NW in the 3x3 */
  int mask = 0;
  for (int k = 0; k < 8; k++)
    if (win[RING[k]] >= 0 && win[RING[k]] == A) mask |= 1 << k;
  if (orc_yokoi_c4(mask) != 1) return 1;
  win_means_t wm = {win, means};
  int32_t B;
  i128 E;
  if (!argmin_move(p, A, nq, e, d, win_means, &wm, &B, &E) || !(E < 0)) return 2;
  *B_out = B;
  *dE_hi = (int64_t)(E >> 64);
  *dE_lo = (uint64_t)E;
  return 3;
}

static void dump_state(seg_t *g) {
  orc_debug *dbg = g->dbg;
  const stage_t *st = &g->st[g->cur];
  size_t per = (size_t)st->nbx * st->nby;
  dbg->map_nbx = st->nbx;
  dbg->map_nby = st->nby;
  if (dbg->map_out && (int64_t)((g->img + 1) * per) <= dbg->map_cap)
    memcpy(dbg->map_out + (size_t)g->img * per, g->L, per * sizeof(int32_t));
  if (dbg->victim_out) memcpy(dbg->victim_out + (size_t)g->img * g->M, g->victim, (size_t)g->M);
  dbg->stopped = 1;
}

/* ----------------------------------------------------------- O6 / O6' -- */
typedef struct { int32_t i, j, A, B; i128 dE; } prop_t;

static int run_phase(seg_t *g, int s, int t, int ph, prop_t *props) {
  const orc_params *p = g->p;
  const stage_t *st = &g->st[s];
  const int cx = ph & 1, cy = ph >> 1; /* colours (0,0),(1,0),(0,1),(1,1) (A5) */
  const int gating = (s > 0 && p->mask_rule != ORC_MASK_OFF); /* A20: stage 0 ungated */
  int64_t *cnt = cnt_ptr(g, s, t, ph);
  int64_t c_cand = 0, c_topo = 0, c_prop = 0, c_sizerej = 0, c_commit = 0, c_commrej = 0;
  int np = 0;

  snapshot(g); /* O5: frozen means for the whole phase (A4) */
  for (int k = 0; k < g->M; k++) g->out[k] = 0;

  for (int j = cy; j < st->nby; j += 2) {
    for (int i = cx; i < st->nbx; i += 2) {
      const int32_t A = lab(g, i, j);
      const int64_t bw = st->xs[i + 1] - st->xs[i], bh = st->ys[j + 1] - st->ys[j];
      int32_t nq[4];
      int64_t eq[4];
      for (int q = 0; q < 4; q++) {
        nq[q] = lab(g, i + N4_DX[q], j + N4_DY[q]);
        eq[q] = (q == 0 || q == 2) ? bw : bh; /* shared edge length in pixels */
      }
      /* 1. mask gate (A22) */
      if (gating) {
        if (p->mask_rule == ORC_MASK_CLASS || p->mask_rule == ORC_MASK_BSP) {
          if (!g->active[A]) continue;
        } else { /* EQ7: a neighbour with another label AND another class (Eq. 7) */
          int ok = 0;
          for (int q = 0; q < 4; q++)
            if (nq[q] >= 0 && nq[q] != A && g->y[nq[q]] != g->y[A]) ok = 1;
          if (!ok) continue;
        }
      }
      /* 2. boundary block (Eq. 2) */
      int bnd = 0;
      for (int q = 0; q < 4; q++)
        if (nq[q] >= 0 && nq[q] != A) bnd = 1;
      if (!bnd) continue;
      c_cand++;
      /* 3. topology: E_topo finite iff p is a simple point of A (A9) */
      int mask = 0;
      for (int k = 0; k < 8; k++) {
        int32_t l = lab(g, i + RING_DX[k], j + RING_DY[k]);
        if (l >= 0 && l == A) mask |= 1 << k;
      }
      if (orc_yokoi_c4(mask) != 1) continue;
      c_topo++;
      /* 4./5./6. candidates = distinct 4-neighbour labels (A8); Eq. 3 argmin (A7) */
      int64_t d[6];
      block_data(g, s, i, j, d);
      int32_t bestB = -1;
      i128 bestE = 0;
      if (!argmin_move(p, A, nq, eq, d, seg_means, g, &bestB, &bestE) || !(bestE < 0)) continue;
      /* 7. size gate for the desired move (A12) */
      if (p->size_mode != ORC_SIZE_NONE) {
        if ((i128)(g->nsnap[A] - d[0]) * p->l_den < (i128)p->l_num * g->init[A]) {
          c_sizerej++;
          if (p->size_mode == ORC_SIZE_MERGE) g->victim[A] = 1;
          continue;
        }
      }
      props[np].i = i; props[np].j = j; props[np].A = A; props[np].B = bestB; props[np].dE = bestE;
      np++;
      g->out[A] += d[0];
      c_prop++;
    }
  }
  /* O6' commit: all-or-nothing budget per source superpixel (A19) */
  for (int k = 0; k < np; k++) {
    const prop_t *pr = &props[k];
    if (p->size_mode != ORC_SIZE_NONE &&
        (i128)(g->nsnap[pr->A] - g->out[pr->A]) * p->l_den < (i128)p->l_num * g->init[pr->A]) {
      c_commrej++;
      if (p->size_mode == ORC_SIZE_MERGE) g->victim[pr->A] = 1;
      continue;
    }
    int64_t d[6];
    block_data(g, s, pr->i, pr->j, d);
    g->L[(size_t)pr->j * st->nbx + pr->i] = pr->B;
    for (int f = 0; f < 6; f++) {
      g->S[(size_t)pr->A * 6 + f] -= d[f];
      g->S[(size_t)pr->B * 6 + f] += d[f];
    }
    c_commit++;
    orc_debug *dbg = g->dbg;
    if (dbg && dbg->moves && dbg->n_moves < dbg->moves_cap) {
      orc_move *m = &dbg->moves[dbg->n_moves++];
      m->stage = s; m->sweep = t; m->phase = ph; m->img = g->img;
      m->bi = pr->i; m->bj = pr->j; m->A = pr->A; m->B = pr->B;
      m->dE_hi = (int64_t)(pr->dE >> 64);
      m->dE_lo = (uint64_t)pr->dE;
    }
  }
  if (cnt) {
    cnt[ORC_C_CAND] += c_cand; cnt[ORC_C_TOPO] += c_topo; cnt[ORC_C_PROP] += c_prop;
    cnt[ORC_C_SIZEREJ] += c_sizerej; cnt[ORC_C_COMMIT] += c_commit; cnt[ORC_C_COMMREJ] += c_commrej;
  }
  return 0;
}

/* ------------------------------------------------------------------ O7 -- */
typedef struct { int32_t V, T; int64_t e; } adj_t;

static int cmp_adj(const void *a, const void *b) {
  const adj_t *x = (const adj_t *)a, *y = (const adj_t *)b;
  if (x->V != y->V) return (x->V > y->V) - (x->V < y->V);
  return (x->T > y->T) - (x->T < y->T);
}

static int merge_round(seg_t *g, int s) {
  const orc_params *p = g->p;
  const stage_t *st = &g->st[s];
  int64_t nvict = 0;
  for (int k = 0; k < g->M; k++) nvict += g->victim[k];
  if (g->dbg) g->dbg->stage_victims[s] += nvict;
  if (nvict == 0) return 0;
  /* 1. adjacency (victim, neighbour) -> shared edge length, over unordered 4-adjacent pairs */
  size_t cap = 1024, n = 0;
  adj_t *adj = (adj_t *)malloc(sizeof(adj_t) * cap);
  if (!adj) return ORC_E_OOM;
  for (int j = 0; j < st->nby; j++) {
    for (int i = 0; i < st->nbx; i++) {
      int32_t a = lab(g, i, j);
      for (int dir = 0; dir < 2; dir++) { /* right, down */
        int ii = i + (dir == 0), jj = j + (dir == 1);
        int32_t b = lab(g, ii, jj);
        if (b < 0 || b == a) continue;
        int64_t e = dir == 0 ? (st->ys[j + 1] - st->ys[j]) : (st->xs[i + 1] - st->xs[i]);
        for (int side = 0; side < 2; side++) {
          int32_t V = side == 0 ? a : b, T = side == 0 ? b : a;
          if (!g->victim[V]) continue;
          if (n == cap) {
            cap *= 2;
            adj_t *nadj = (adj_t *)realloc(adj, sizeof(adj_t) * cap);
            if (!nadj) { free(adj); return ORC_E_OOM; }
            adj = nadj;
          }
          adj[n].V = V; adj[n].T = T; adj[n].e = e; n++;
        }
      }
    }
  }
  qsort(adj, n, sizeof(adj_t), cmp_adj);
  /* 2. snapshot (O5) */
  snapshot(g);
  for (int k = 0; k < g->M; k++) { g->locked[k] = 0; g->remap[k] = k; }
  /* 3./4. victims in ascending id; Eq. 4 argmin over contiguous superpixels, Eq. 5 bound */
  int64_t merges = 0;
  size_t a0 = 0;
  while (a0 < n) {
    int32_t A = adj[a0].V;
    size_t a1 = a0;
    while (a1 < n && adj[a1].V == A) a1++;
    if (!g->locked[A]) {
      int have = 0;
      int32_t bestT = -1;
      i128 bestE = 0;
      int64_t bestLen = 0;
      size_t k = a0;
      while (k < a1) {
        int32_t T = adj[k].T;
        int64_t len = 0;
        while (k < a1 && adj[k].T == T) { len += adj[k].e; k++; }
        if (!g->alive[T] || g->locked[T]) continue;
        int64_t nA = g->S[(size_t)A * 6], nT = g->S[(size_t)T * 6];
        if ((i128)(nT + nA) * p->u_den > (i128)p->u_num * g->init[T]) continue; /* Eq. 5 */
        i128 dC, dP;
        delta_cp(g, A, T, g->S + (size_t)A * 6, &dC, &dP); /* A's whole sums (A14) */
        i128 E = weigh(p, dC, dP, -2 * (i128)len);
        if (!have || E < bestE || (E == bestE && T < bestT)) {
          have = 1; bestE = E; bestT = T; bestLen = len;
        }
      }
      if (have) { /* A15: pure argmin, no dE<0 requirement; A16: none feasible -> no merge */
        for (int f = 0; f < 6; f++) {
          g->S[(size_t)bestT * 6 + f] += g->S[(size_t)A * 6 + f];
          g->S[(size_t)A * 6 + f] = 0;
        }
        g->alive[A] = 0;
        g->active[A] = 0;
        g->y[A] = 0;
        g->remap[A] = bestT;
        g->locked[A] = 1;
        g->locked[bestT] = 1;
        merges++;
        orc_debug *dbg = g->dbg;
        if (dbg && dbg->merges && dbg->n_merges < dbg->merges_cap) {
          orc_merge *m = &dbg->merges[dbg->n_merges++];
          m->stage = s; m->img = g->img; m->A = A; m->T = bestT; m->len = bestLen;
          m->dE_hi = (int64_t)(bestE >> 64);
          m->dE_lo = (uint64_t)bestE;
        }
      }
    }
    a0 = a1;
  }
  free(adj);
  /* 5. clear victims, apply the remap to L_s (InitSize of targets unchanged) */
  for (int k = 0; k < g->M; k++) g->victim[k] = 0;
  size_t nb = (size_t)st->nbx * st->nby;
  for (size_t b = 0; b < nb; b++) g->L[b] = g->remap[g->L[b]];
  if (g->dbg) g->dbg->stage_merges[s] += merges;
  return 0;
}

/* ------------------------------------------------------------------ O8 -- */
static int cmp_u64_orc(const void *a, const void *b) {
  const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* round-half-up(num / den) for num >= 0, den > 0 */
static int64_t rhu(i128 num, i128 den) { return (int64_t)((2 * num + den) / (2 * den)); }

/* y from a linear model on the 4 features of P:271 (Q16 fixed point).
 * Brightness of a pixel = (r+g+b)/3; per superpixel n, S = sum(r+g+b), Q = sum((r+g+b)^2):
 *   f1 = rhu(2^16 S / (765 n))                     absolute brightness / 255
 *   f2 = f1 - rhu(2^16 S_img / (765 N_img))         comparative brightness
 *   f3 = rhu(2^16 (n Q - S^2) / (585225 n^2))       intra-region dissimilarity (variance / 255^2)
 *   f4 = rhu(sum_q |f1 - f1_q| / deg)               extra-region dissimilarity over the distinct
 *                                                    4-adjacent superpixels q of the stage map
 *   y = +1 iff w0 2^16 + sum_i w_i f_i >= 0        (Eq. 6) */
static void predict_features(seg_t *g) {
  const orc_params *p = g->p;
  const stage_t *st = &g->st[g->cur];
  const int M = g->M;
  i128 *Q = (i128 *)calloc((size_t)M, sizeof(i128));
  int64_t *f1 = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  int64_t *dsum = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  int64_t *deg = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  const size_t nb = (size_t)st->nbx * st->nby;
  uint64_t *pairs = (uint64_t *)malloc(sizeof(uint64_t) * (4 * nb + 1));  /* directed adjacent pairs */
  size_t np = 0;
  /* S and Q by the pixels of every block of the current map (the features read the image:
   * with the literal pyramid, f3, the superpixel sums are approximations) */
  int64_t *Sp = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  for (int j = 0; j < st->nby; j++)
    for (int i = 0; i < st->nbx; i++) {
      const int32_t a = lab(g, i, j);
      for (int y = st->ys[j]; y < st->ys[j + 1]; y++)
        for (int x = st->xs[i]; x < st->xs[i + 1]; x++) {
          const uint8_t *px = g->I + ((size_t)y * g->W + x) * 3;
          const int64_t s = (int64_t)px[0] + px[1] + px[2];
          Sp[a] += s;
          Q[a] += (i128)(s * s);
        }
    }
  i128 Simg = 0, Nimg = 0;
  for (int k = 0; k < M; k++)
    if (g->alive[k]) {
      Simg += (i128)Sp[k];
      Nimg += (i128)g->S[(size_t)k * 6];
    }
  const int64_t fimg = rhu(Simg << 16, 765 * Nimg);
  for (int k = 0; k < M; k++)
    if (g->alive[k]) f1[k] = rhu((i128)Sp[k] << 16, 765 * (i128)g->S[(size_t)k * 6]);
  for (int j = 0; j < st->nby; j++)
    for (int i = 0; i < st->nbx; i++) {
      const int32_t a = lab(g, i, j);
      for (int dir = 0; dir < 2; dir++) {
        const int32_t b = lab(g, i + (dir == 0), j + (dir == 1));
        if (b < 0 || b == a) continue;
        pairs[np++] = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
        pairs[np++] = ((uint64_t)(uint32_t)b << 32) | (uint32_t)a;
      }
    }
  qsort(pairs, np, sizeof(uint64_t), cmp_u64_orc);
  for (size_t t = 0; t < np; t++) {
    if (t > 0 && pairs[t] == pairs[t - 1]) continue;  /* each distinct neighbour once */
    const int32_t u = (int32_t)(pairs[t] >> 32), v = (int32_t)(pairs[t] & 0xffffffffu);
    deg[u]++;
    dsum[u] += f1[u] > f1[v] ? f1[u] - f1[v] : f1[v] - f1[u];
  }
  for (int k = 0; k < M; k++) {
    if (!g->alive[k]) { g->y[k] = 0; continue; }
    const i128 n = g->S[(size_t)k * 6], S = Sp[k];
    const int64_t f2 = f1[k] - fimg;
    const int64_t f3 = rhu((n * Q[k] - S * S) << 16, 585225 * n * n);
    const int64_t f4 = deg[k] ? rhu(dsum[k], deg[k]) : 0;
    const i128 h = ((i128)p->feat_w_q16[0] << 16) + (i128)p->feat_w_q16[1] * f1[k] + (i128)p->feat_w_q16[2] * f2 +
                   (i128)p->feat_w_q16[3] * f3 + (i128)p->feat_w_q16[4] * f4;
    g->y[k] = h >= 0 ? 1 : -1;
  }
  free(Q); free(f1); free(dsum); free(deg); free(pairs); free(Sp);
}

static void predict(seg_t *g) {
  const orc_params *p = g->p;
  const stage_t *st = &g->st[g->cur];
  snapshot(g);
  if (p->y_model == 1) predict_features(g);
  for (int k = 0; k < g->M && p->y_model != 1; k++) {
    if (!g->alive[k]) { g->y[k] = 0; g->active[k] = 0; continue; }
    i128 dmin = -1;
    for (int t = 0; t < p->n_proto; t++) {
      i128 d = 0;
      for (int ch = 0; ch < 3; ch++) {
        i128 e = (i128)g->cq[(size_t)k * 3 + ch] - ((i128)p->proto[t][ch] << FRAC);
        d += e * e;
      }
      if (dmin < 0 || d < dmin) dmin = d;
    }
    /* Eq. 6: y = +1 iff h(x) = tau^2 2^(2F) - d >= 0 */
    g->y[k] = (((i128)p->tau2 << (2 * FRAC)) - dmin >= 0) ? 1 : -1;
  }
  if (p->mask_rule == ORC_MASK_CLASS) {
    for (int k = 0; k < g->M; k++) g->active[k] = g->alive[k] && g->y[k] == 1;
  } else { /* BSP / EQ7: boundary superpixels (Eq. 7 at superpixel level) */
    for (int k = 0; k < g->M; k++) g->active[k] = 0;
    for (int j = 0; j < st->nby; j++)
      for (int i = 0; i < st->nbx; i++) {
        int32_t a = lab(g, i, j);
        for (int dir = 0; dir < 2; dir++) {
          int32_t b = lab(g, i + (dir == 0), j + (dir == 1));
          if (b < 0 || b == a) continue;
          if (g->y[a] != g->y[b]) { g->active[a] = 1; g->active[b] = 1; }
        }
      }
  }
}

/* ---------------------------------------------------------- per image ---- */
static void free_seg(seg_t *g) {
  free(g->X); free(g->Y); free(g->S); free(g->init); free(g->alive); free(g->active);
  free(g->victim); free(g->locked); free(g->y); free(g->cq); free(g->mq); free(g->nsnap);
  free(g->out); free(g->remap); free(g->L);
  for (int s = 0; s < ORC_MAX_STAGES; s++) {
    free(g->st[s].xs); free(g->st[s].ys); free(g->st[s].bd);
  }
}

static int build_stage(seg_t *g, int s) {
  const int b = g->p->block_size[s];
  stage_t *st = &g->st[s];
  int capx = g->W / b + g->cols + 3, capy = g->H / b + g->rows + 3;
  st->xs = (int32_t *)malloc(sizeof(int32_t) * (size_t)capx);
  st->ys = (int32_t *)malloc(sizeof(int32_t) * (size_t)capy);
  if (!st->xs || !st->ys) return ORC_E_OOM;
  int nx = orc_stage_axis(g->W, b, g->X, g->cols + 1, st->xs, capx);
  int ny = orc_stage_axis(g->H, b, g->Y, g->rows + 1, st->ys, capy);
  if (nx < 2 || ny < 2) return ORC_E_ARG;
  st->nbx = nx - 1;
  st->nby = ny - 1;
  return 0;
}

/* f3 / A32, literal image pyramid (Eq. 8 reuse with the paper's approximation): a block's
 * level value is the rounded (half up) area-weighted mean of its children's level values in
 * the next finer stage, the finest stage's blocks averaging their pixels (pixels are the
 * level of b = 1); its colour data are area x value per channel; area and position sums stay
 * exact (full-resolution coordinates make Eq. 8's position map the identity). */
static int build_pyramid_literal(seg_t *g) {
  const orc_params *p = g->p;
  for (int s = p->n_stages - 1; s >= 0; s--) {
    stage_t *st = &g->st[s];
    if (p->block_size[s] == 1) continue;
    free(st->bd);
    st->bd = (int64_t *)malloc(sizeof(int64_t) * 6 * (size_t)st->nbx * st->nby);
    if (!st->bd) return ORC_E_OOM;
    const stage_t *fn = (s + 1 < p->n_stages && p->block_size[s + 1] > 1) ? &g->st[s + 1] : NULL;
    for (int j = 0; j < st->nby; j++)
      for (int i = 0; i < st->nbx; i++) {
        int64_t *d = st->bd + ((size_t)j * st->nbx + i) * 6;
        const int x0 = st->xs[i], x1 = st->xs[i + 1], y0 = st->ys[j], y1 = st->ys[j + 1];
        int64_t pix[6];
        block_direct(g, x0, x1, y0, y1, pix); /* exact area and positions */
        int64_t cs[3] = {pix[1], pix[2], pix[3]};
        if (fn) { /* children: the finer stage's blocks inside this one */
          cs[0] = cs[1] = cs[2] = 0;
          for (int cj = 0; cj < fn->nby; cj++) {
            if (fn->ys[cj] < y0 || fn->ys[cj] >= y1) continue;
            for (int ci = 0; ci < fn->nbx; ci++) {
              if (fn->xs[ci] < x0 || fn->xs[ci] >= x1) continue;
              const int64_t *cd = fn->bd + ((size_t)cj * fn->nbx + ci) * 6;
              cs[0] += cd[1]; cs[1] += cd[2]; cs[2] += cd[3];
            }
          }
        }
        const int64_t area = pix[0];
        d[0] = area;
        for (int ch = 0; ch < 3; ch++) d[1 + ch] = area * ((2 * cs[ch] + area) / (2 * area));
        d[4] = pix[4];
        d[5] = pix[5];
      }
  }
  return 0;
}

static int build_block_sums(seg_t *g, int s) { /* O3, direct summation (b > 1 only) */
  stage_t *st = &g->st[s];
  if (g->p->block_size[s] == 1) return 0;
  if (g->p->stats_mode == ORC_STATS_PYRAMID) return st->bd ? 0 : ORC_E_ARG; /* built up front */
  st->bd = (int64_t *)malloc(sizeof(int64_t) * 6 * (size_t)st->nbx * st->nby);
  if (!st->bd) return ORC_E_OOM;
  for (int j = 0; j < st->nby; j++)
    for (int i = 0; i < st->nbx; i++)
      block_direct(g, st->xs[i], st->xs[i + 1], st->ys[j], st->ys[j + 1],
                   st->bd + ((size_t)j * st->nbx + i) * 6);
  return 0;
}

static int stop_here(seg_t *g, int kind, int s, int t, int ph) {
  orc_debug *d = g->dbg;
  if (!d || d->stop_kind != kind || d->stop_stage != s) return 0;
  if (kind == ORC_STOP_PHASE && (d->stop_sweep != t || d->stop_phase != ph)) return 0;
  dump_state(g);
  return 1;
}

static void write_sp(seg_t *g, orc_sp *sp) {
  for (int k = 0; k < g->M; k++) {
    orc_sp *o = &sp[(size_t)g->img * g->M + k];
    const int64_t *s = g->S + (size_t)k * 6;
    o->n = s[0]; o->sum_r = s[1]; o->sum_g = s[2]; o->sum_b = s[3]; o->sum_x = s[4]; o->sum_y = s[5];
    o->init_size = g->init[k];
    o->alive = (int8_t)g->alive[k];
    o->active = (int8_t)g->active[k];
    o->y = g->y[k];
    o->pad = 0;
  }
}

static int seg_image(seg_t *g, int32_t *labels_out, orc_sp *sp_out) {
  const orc_params *p = g->p;
  const int H = g->H, W = g->W, M = g->M;
  int rc = orc_grid(H, W, M, &g->rows, &g->cols);
  if (rc) return rc;
  const int r = g->rows, c = g->cols;
  g->X = (int32_t *)malloc(sizeof(int32_t) * (size_t)(c + 1));
  g->Y = (int32_t *)malloc(sizeof(int32_t) * (size_t)(r + 1));
  g->S = (int64_t *)calloc((size_t)M * 6, sizeof(int64_t));
  g->init = (int32_t *)malloc(sizeof(int32_t) * (size_t)M);
  g->alive = (uint8_t *)malloc((size_t)M);
  g->active = (uint8_t *)malloc((size_t)M);
  g->victim = (uint8_t *)calloc((size_t)M, 1);
  g->locked = (uint8_t *)calloc((size_t)M, 1);
  g->y = (int8_t *)calloc((size_t)M, 1);
  g->cq = (int64_t *)calloc((size_t)M * 3, sizeof(int64_t));
  g->mq = (int64_t *)calloc((size_t)M * 2, sizeof(int64_t));
  g->nsnap = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  g->out = (int64_t *)calloc((size_t)M, sizeof(int64_t));
  g->remap = (int32_t *)malloc(sizeof(int32_t) * (size_t)M);
  if (!g->X || !g->Y || !g->S || !g->init || !g->alive || !g->active || !g->victim ||
      !g->locked || !g->y || !g->cq || !g->mq || !g->nsnap || !g->out || !g->remap)
    return ORC_E_OOM;
  /* O1: X_i = floor(i W / c), Y_j = floor(j H / r); label j*c + i; InitSize = cell area */
  for (int i = 0; i <= c; i++) g->X[i] = (int32_t)(((int64_t)i * W) / c);
  for (int j = 0; j <= r; j++) g->Y[j] = (int32_t)(((int64_t)j * H) / r);
  for (int j = 0; j < r; j++)
    for (int i = 0; i < c; i++)
      g->init[j * c + i] = (g->X[i + 1] - g->X[i]) * (g->Y[j + 1] - g->Y[j]);
  for (int k = 0; k < M; k++) { g->alive[k] = 1; g->active[k] = 1; }
  /* cell index of each pixel column / row */
  int32_t *colcell = (int32_t *)malloc(sizeof(int32_t) * (size_t)W);
  int32_t *rowcell = (int32_t *)malloc(sizeof(int32_t) * (size_t)H);
  if (!colcell || !rowcell) { free(colcell); free(rowcell); return ORC_E_OOM; }
  for (int i = 0; i < c; i++)
    for (int x = g->X[i]; x < g->X[i + 1]; x++) colcell[x] = i;
  for (int j = 0; j < r; j++)
    for (int y = g->Y[j]; y < g->Y[j + 1]; y++) rowcell[y] = j;
  /* O4: S_1 by a pixel loop over the initial grid labels (RAPID l.9-10) */
  for (int y = 0; y < H; y++)
    for (int x = 0; x < W; x++) {
      int k = rowcell[y] * c + colcell[x];
      const uint8_t *px = g->I + ((size_t)y * W + x) * 3;
      int64_t *s = g->S + (size_t)k * 6;
      s[0] += 1; s[1] += px[0]; s[2] += px[1]; s[3] += px[2]; s[4] += x; s[5] += y;
    }
  /* O2 geometry of every stage */
  for (int s = 0; s < p->n_stages; s++) {
    rc = build_stage(g, s);
    if (rc) { free(colcell); free(rowcell); return rc; }
  }
  /* stage-0 map: the cell of each block (blocks never straddle cells, A10) */
  {
    stage_t *st = &g->st[0];
    g->L = (int32_t *)malloc(sizeof(int32_t) * (size_t)st->nbx * st->nby);
    if (!g->L) { free(colcell); free(rowcell); return ORC_E_OOM; }
    for (int j = 0; j < st->nby; j++)
      for (int i = 0; i < st->nbx; i++)
        g->L[(size_t)j * st->nbx + i] = rowcell[st->ys[j]] * c + colcell[st->xs[i]];
  }
  free(colcell);
  free(rowcell);

  if (p->stats_mode == ORC_STATS_PYRAMID) {
    int rc2 = build_pyramid_literal(g);
    if (rc2) return rc2;
    /* f3: S_1 from the coarsest level's data ("average information of each superpixel at the
     * first image level"), not from the pixels */
    const stage_t *st = &g->st[0];
    if (p->block_size[0] > 1) {
      memset(g->S, 0, sizeof(int64_t) * 6 * (size_t)M);
      for (int j = 0; j < st->nby; j++)
        for (int i = 0; i < st->nbx; i++) {
          const int64_t *d = st->bd + ((size_t)j * st->nbx + i) * 6;
          int64_t *sk = g->S + (size_t)g->L[(size_t)j * st->nbx + i] * 6;
          for (int f = 0; f < 6; f++) sk[f] += d[f];
        }
    }
  }
  prop_t *props = NULL;
  int result = 0;
  for (int s = 0; s < p->n_stages; s++) {
    stage_t *st = &g->st[s];
    if (s > 0) { /* O9: L_s(child) = L_{s-1}(parent) (RAPID l.7-8) */
      stage_t *pv = &g->st[s - 1];
      int32_t *pi = (int32_t *)malloc(sizeof(int32_t) * (size_t)st->nbx);
      int32_t *pj = (int32_t *)malloc(sizeof(int32_t) * (size_t)st->nby);
      int32_t *NL = (int32_t *)malloc(sizeof(int32_t) * (size_t)st->nbx * st->nby);
      if (!pi || !pj || !NL) { free(pi); free(pj); free(NL); result = ORC_E_OOM; break; }
      for (int i = 0; i < st->nbx; i++) {
        int k = 0;
        while (!(pv->xs[k] <= st->xs[i] && st->xs[i] < pv->xs[k + 1])) k++;
        pi[i] = k;
      }
      for (int j = 0; j < st->nby; j++) {
        int k = 0;
        while (!(pv->ys[k] <= st->ys[j] && st->ys[j] < pv->ys[k + 1])) k++;
        pj[j] = k;
      }
      for (int j = 0; j < st->nby; j++)
        for (int i = 0; i < st->nbx; i++)
          NL[(size_t)j * st->nbx + i] = g->L[(size_t)pj[j] * pv->nbx + pi[i]];
      free(pi); free(pj); free(g->L);
      g->L = NL;
      if (p->stats_mode != ORC_STATS_PYRAMID) { free(pv->bd); pv->bd = NULL; }
    }
    g->cur = s;
    result = build_block_sums(g, s);
    if (result) break;
    if (s > 0 && p->stats_mode == ORC_STATS_RECOUNT) {
      /* multi-scale CTFTPS recount: sums from the new map must equal the
       * reused ones exactly (A23) */
      int64_t *R = (int64_t *)calloc((size_t)M * 6, sizeof(int64_t));
      if (!R) { result = ORC_E_OOM; break; }
      for (int j = 0; j < st->nby; j++)
        for (int i = 0; i < st->nbx; i++) {
          int64_t d[6];
          block_data(g, s, i, j, d);
          int32_t l = g->L[(size_t)j * st->nbx + i];
          for (int f = 0; f < 6; f++) R[(size_t)l * 6 + f] += d[f];
        }
      int bad = memcmp(R, g->S, sizeof(int64_t) * 6 * (size_t)M) != 0;
      free(R);
      if (bad) { result = ORC_E_INTEGRITY; break; }
    }
    if (stop_here(g, ORC_STOP_STAGE_START, s, 0, 0)) { write_sp(g, sp_out); free(props); return 0; }
    free(props);
    props = (prop_t *)malloc(sizeof(prop_t) * ((size_t)(st->nbx / 2 + 1) * (st->nby / 2 + 1)));
    if (!props) { result = ORC_E_OOM; break; }
    for (int t = 0; t < p->sweeps; t++) {
      for (int ph = 0; ph < 4; ph++) {
        run_phase(g, s, t, ph, props);
        if (stop_here(g, ORC_STOP_PHASE, s, t, ph)) { write_sp(g, sp_out); free(props); return 0; }
      }
    }
    /* A28: merges -> prediction (s = 0) -> transition */
    if (p->size_mode == ORC_SIZE_MERGE) {
      result = merge_round(g, s);
      if (result) break;
    }
    if (stop_here(g, ORC_STOP_AFTER_MERGE, s, 0, 0)) { write_sp(g, sp_out); free(props); return 0; }
    if (s == 0 && p->mask_rule != ORC_MASK_OFF) {
      predict(g);
      if (stop_here(g, ORC_STOP_AFTER_PREDICT, s, 0, 0)) { write_sp(g, sp_out); free(props); return 0; }
    }
  }
  free(props);
  if (result) return result;
  /* final: the last stage's map at pixel resolution (upsample when the grain > 1) */
  {
    const stage_t *st = &g->st[p->n_stages - 1];
    int32_t *bx = (int32_t *)malloc(sizeof(int32_t) * (size_t)W);
    int32_t *by = (int32_t *)malloc(sizeof(int32_t) * (size_t)H);
    if (!bx || !by) { free(bx); free(by); return ORC_E_OOM; }
    for (int i = 0; i < st->nbx; i++)
      for (int x = st->xs[i]; x < st->xs[i + 1]; x++) bx[x] = i;
    for (int j = 0; j < st->nby; j++)
      for (int y = st->ys[j]; y < st->ys[j + 1]; y++) by[y] = j;
    for (int y = 0; y < H; y++)
      for (int x = 0; x < W; x++)
        labels_out[(size_t)y * W + x] = g->L[(size_t)by[y] * st->nbx + bx[x]];
    free(bx); free(by);
  }
  write_sp(g, sp_out);
  return 0;
}

static int check_params(int B, int H, int W, const orc_params *p) {
  if (B < 1 || H < 1 || W < 1 || !p) return ORC_E_ARG;
  if (p->n_superpixels < 1 || (int64_t)p->n_superpixels > (int64_t)H * W) return ORC_E_ARG;
  if (p->n_stages < 1 || p->n_stages > ORC_MAX_STAGES) return ORC_E_ARG;
  if (p->sweeps < 0 || p->sweeps > ORC_MAX_SWEEPS) return ORC_E_ARG;
  for (int s = 0; s < p->n_stages; s++) {
    if (p->block_size[s] < 1 || p->block_size[s] > 64) return ORC_E_ARG;
    if (s > 0 && (p->block_size[s] >= p->block_size[s - 1] ||
                  p->block_size[s - 1] % p->block_size[s] != 0))
      return ORC_E_ARG;
  }
  if (p->lambda_pos_q16 < 0 || p->lambda_b_q16 < 0) return ORC_E_ARG;
  if (p->size_mode < 0 || p->size_mode > 2 || p->mask_rule < 0 || p->mask_rule > 3) return ORC_E_ARG;
  if (p->size_mode != ORC_SIZE_NONE) {
    if (p->l_num < 0 || p->l_den <= 0 || p->l_num >= p->l_den) return ORC_E_ARG;
    if (p->u_den <= 0 || p->u_num <= p->u_den) return ORC_E_ARG;
  }
  if (p->mask_rule != ORC_MASK_OFF && p->y_model == 0 && (p->n_proto < 1 || p->n_proto > 4)) return ORC_E_ARG;
  if (p->y_model < 0 || p->y_model > 1) return ORC_E_ARG;
  if (p->tau2 < 0) return ORC_E_ARG;
  return ORC_OK;
}

int orc_segment(const uint8_t *image, int B, int H, int W, const orc_params *p,
                int32_t *labels_out, orc_sp *sp_out, orc_debug *dbg) {
  int rc = check_params(B, H, W, p);
  if (rc) return rc;
  int r, c;
  rc = orc_grid(H, W, p->n_superpixels, &r, &c);
  if (rc) return rc;
  if (dbg) {
    dbg->stopped = 0;
    dbg->n_moves = 0;
    dbg->n_merges = 0;
    for (int s = 0; s < ORC_MAX_STAGES; s++) { dbg->stage_victims[s] = 0; dbg->stage_merges[s] = 0; }
  }
  /* A27: images are independent; each is segmented on its own, in order */
  for (int b = 0; b < B; b++) {
    seg_t g;
    memset(&g, 0, sizeof g);
    g.I = image + (size_t)b * H * W * 3;
    g.H = H; g.W = W; g.M = p->n_superpixels; g.img = b; g.p = p; g.dbg = dbg;
    rc = seg_image(&g, labels_out + (size_t)b * H * W, sp_out);
    free_seg(&g);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* ===================================================================== f4: quality
 * Plain definitions (oracle.h).  UE: the (superpixel, segment) intersection sizes by sorting
 * the per-pixel pairs; superpixel sizes by sorting the labels.  BR: direct window scan. */
static int cmp_u64(const void *a, const void *b) {
  const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int is_boundary(const int32_t *m, int H, int W, int x, int y) {
  const int32_t v = m[(size_t)y * W + x];
  if (x > 0 && m[(size_t)y * W + x - 1] != v) return 1;
  if (x + 1 < W && m[(size_t)y * W + x + 1] != v) return 1;
  if (y > 0 && m[(size_t)(y - 1) * W + x] != v) return 1;
  if (y + 1 < H && m[(size_t)(y + 1) * W + x] != v) return 1;
  return 0;
}

int orc_quality_eval(const int32_t *labels, const int32_t *gt, int B, int H, int W, int eps, orc_quality *out) {
  if (!labels || !gt || !out || B < 1 || H < 1 || W < 1 || eps < 0) return ORC_E_ARG;
  const size_t n = (size_t)H * W;
  uint64_t *pairs = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *sps = (uint64_t *)malloc(sizeof(uint64_t) * n);
  if (!pairs || !sps) {
    free(pairs);
    free(sps);
    return ORC_E_OOM;
  }
  memset(out, 0, sizeof *out);
  out->pixels = (int64_t)B * (int64_t)n;
  for (int b = 0; b < B; b++) {
    const int32_t *L = labels + (size_t)b * n, *G = gt + (size_t)b * n;
    for (size_t i = 0; i < n; i++) {
      if (L[i] < 0 || G[i] < 0) {
        free(pairs);
        free(sps);
        return ORC_E_ARG;
      }
      pairs[i] = ((uint64_t)(uint32_t)L[i] << 32) | (uint32_t)G[i];
      sps[i] = (uint32_t)L[i];
    }
    qsort(pairs, n, sizeof(uint64_t), cmp_u64);
    qsort(sps, n, sizeof(uint64_t), cmp_u64);
    /* walk the pairs; |sp| by binary search of the sorted labels */
    size_t i = 0;
    while (i < n) {
      size_t j = i;
      while (j < n && pairs[j] == pairs[i]) j++;
      const uint64_t sp = pairs[i] >> 32;
      size_t lo = 0, hi = n;  /* first index with sps >= sp */
      while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (sps[mid] < sp) lo = mid + 1; else hi = mid;
      }
      size_t e = lo;
      while (e < n && sps[e] == sp) e++;
      const int64_t inter = (int64_t)(j - i), size = (int64_t)(e - lo);
      const int64_t rest = size - inter;
      out->leak += inter < rest ? inter : rest;
      i = j;
    }
    for (int y = 0; y < H; y++)
      for (int x = 0; x < W; x++) {
        if (!is_boundary(G, H, W, x, y)) continue;
        out->gt_boundary++;
        int hit = 0;
        for (int dy = -eps; dy <= eps && !hit; dy++)
          for (int dx = -eps; dx <= eps && !hit; dx++) {
            const int xx = x + dx, yy = y + dy;
            if (xx >= 0 && yy >= 0 && xx < W && yy < H && is_boundary(L, H, W, xx, yy)) hit = 1;
          }
        out->covered += hit;
      }
  }
  free(pairs);
  free(sps);
  return ORC_OK;
}

