/*
 * oracle.h — CPU oracle for the RAPID / CTFTPS refinement hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The
 * product path (paper_1704_02083_b200/, include/rapid.h) never does, and shares
 * no code, header, table or constant generator with it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named),
 * "Ax" = a reading listed in DESIGN.md §2 (taken from SURVEY.md §8(c)).
 *
 * Parity pins (tests/test_oracle_*.py): geometry closed forms, brute-force block
 * sums, exhaustive rounding, per-pixel brute-force energy deltas (exact integer
 * equality), exhaustive topology LUT vs flood fill, hand-worked H1-H4, invariants,
 * and the choices themselves: every Eq. 3 decision and every Eq. 4 merge of random
 * runs re-derived by brute force (tests/test_oracle_choice.py; one-token mutants of
 * either argmin fail it, tools/mutation_check.sh).
 * Parity with the paper's own outputs is unpinned (the paper prints none).
 */
#ifndef RAPID_ORACLE_H
#define RAPID_ORACLE_H
#include <stdint.h>

#define ORC_MAX_STAGES 12
#define ORC_MAX_SWEEPS 64
#define ORC_NCNT 6 /* per-phase counters, see orc_phase_counter */

enum { ORC_SIZE_NONE = 0, ORC_SIZE_HARD = 1, ORC_SIZE_MERGE = 2 };
enum { ORC_MASK_OFF = 0, ORC_MASK_CLASS = 1, ORC_MASK_BSP = 2, ORC_MASK_EQ7 = 3 };
enum { ORC_STATS_REUSE = 0, ORC_STATS_RECOUNT = 1, ORC_STATS_PYRAMID = 2 };
/* per-phase counters */
enum { ORC_C_CAND = 0,     /* gated boundary blocks of the phase colour */
       ORC_C_TOPO = 1,     /* ... that passed the simple-point test */
       ORC_C_PROP = 2,     /* proposals (dE<0 and single-move size gate ok) */
       ORC_C_SIZEREJ = 3,  /* desired moves rejected by the single-move size gate */
       ORC_C_COMMIT = 4,   /* committed moves */
       ORC_C_COMMREJ = 5 };/* proposals dropped by the all-or-nothing budget */

typedef struct {
  int32_t n_superpixels;             /* M per image */
  int32_t n_stages;                  /* <= ORC_MAX_STAGES */
  int32_t block_size[ORC_MAX_STAGES];/* descending, each divides the previous */
  int32_t sweeps;                    /* sweeps per stage (A5) */
  int64_t lambda_pos_q16;            /* lambda_pos, Q16.16 */
  int64_t lambda_b_q16;              /* lambda_b, Q16.16 */
  int32_t size_mode;                 /* ORC_SIZE_* */
  int32_t l_num, l_den;              /* lower bound l */
  int32_t u_num, u_den;              /* upper bound u (Eq. 5) */
  int32_t mask_rule;                 /* ORC_MASK_* (A22) */
  int32_t n_proto;                   /* <= 4 */
  int32_t proto[4][3];               /* RGB prototypes for h_theta (A21) */
  int64_t tau2;                      /* y=+1 iff min_k ||c-proto_k||^2 <= tau2 */
  int32_t stats_mode;                /* ORC_STATS_* (A23) */
  int32_t y_model;                   /* 0: prototype distance (A21); 1: linear model on features (A31) */
  int64_t feat_w_q16[5];             /* bias, w1..w4 (Q16.16) of the feature model */
} orc_params;

typedef struct {
  int64_t n, sum_r, sum_g, sum_b, sum_x, sum_y;
  int32_t init_size;
  int8_t alive, active, y;
  int8_t pad;
} orc_sp;

typedef struct {
  int32_t stage, sweep, phase, img;
  int32_t bi, bj; /* block column, row within the image */
  int32_t A, B;   /* local labels */
  int64_t dE_hi;  /* int128 dE = (dE_hi << 64) | dE_lo, units 2^(16+4F) */
  uint64_t dE_lo;
} orc_move;

typedef struct {
  int32_t stage, img, A, T;
  int64_t len;    /* shared edge length in pixels */
  int64_t dE_hi;
  uint64_t dE_lo;
} orc_merge;

/* stop kinds: the oracle stops and dumps the current stage map + stats */
enum { ORC_STOP_NONE = 0,
       ORC_STOP_PHASE = 1,       /* after the commit of (stage, sweep, phase) */
       ORC_STOP_STAGE_START = 2, /* after the transition into `stage`, before its phases */
       ORC_STOP_AFTER_MERGE = 3, /* after the merge round of `stage` */
       ORC_STOP_AFTER_PREDICT = 4/* after prediction (stage 0) */ };

typedef struct {
  int32_t stop_kind, stop_stage, stop_sweep, stop_phase;
  int32_t *map_out; int64_t map_cap;   /* stage map, images stacked: [B][nby][nbx] */
  int32_t map_nbx, map_nby;            /* out */
  int32_t stopped;                     /* out: 1 if the stop point was reached */
  orc_move *moves; int64_t moves_cap; int64_t n_moves;     /* committed-move log */
  orc_merge *merges; int64_t merges_cap; int64_t n_merges; /* merge log */
  int64_t *phase_counters;  /* [ORC_MAX_STAGES][ORC_MAX_SWEEPS][4][ORC_NCNT], summed over images */
  int64_t stage_victims[ORC_MAX_STAGES];
  int64_t stage_merges[ORC_MAX_STAGES];
  uint8_t *victim_out;      /* optional [B][M]: the O6/O6' victim flags at the stop point (test export) */
} orc_debug;

#define ORC_OK 0
#define ORC_E_ARG (-1)
#define ORC_E_OOM (-5)
#define ORC_E_INTEGRITY (-6)

/* Whole segmentation of B independent images u8 [B][H][W][3] -> labels [B][H][W]
 * (per-image local ids) and per-superpixel stats [B*M] (index img*M + local).
 * dbg may be NULL. Returns ORC_OK or an error. */
int orc_segment(const uint8_t *image, int B, int H, int W, const orc_params *p,
                int32_t *labels_out, orc_sp *sp_out, orc_debug *dbg);

/* Exposed pieces for the pin tests. */
int orc_grid(int H, int W, int M, int *rows, int *cols);            /* O1 */
int orc_stage_axis(int len, int b, const int32_t *cuts, int ncuts,  /* O2 */
                   int32_t *out, int cap);
int orc_yokoi_c4(int ring_mask);                                    /* A9 */
void orc_round_mean(int64_t S, int64_t n, int64_t *q);              /* O5 */
void orc_colour_mean(int64_t S, int64_t n, int64_t *q);             /* O5 + A33 clamp */
/* O6 steps 2-6 for one block in isolation (see oracle.c) */
int orc_block_move(const int32_t *win, const int64_t *means, const int64_t *d, const int64_t *e,
                   const orc_params *p, int32_t *B_out, int64_t *dE_hi, uint64_t *dE_lo);
/* segmentation quality against a ground-truth segment map (the
 * standard metrics of "Peer"; definitions as SPEC §Operations states them in words).
 * labels, gt: int32 [B][H][W], per-image ids >= 0; each image is scored on its own and the
 * counts are summed over the batch.
 *   UE: leak = sum over images, GT segments S and superpixels sp meeting S of
 *       min(|sp n S|, |sp \ S|);  UE = leak / (B H W).
 *   BR(eps): a pixel is a boundary pixel of a map if one of its in-image 4-neighbours has
 *       another id; BR = (#GT boundary pixels with a superpixel boundary pixel within
 *       Chebyshev distance eps) / (#GT boundary pixels), 1 when there is none. */
typedef struct {
  int64_t pixels, leak, gt_boundary, covered;
} orc_quality;
int orc_quality_eval(const int32_t *labels, const int32_t *gt, int B, int H, int W, int eps, orc_quality *out);
#endif