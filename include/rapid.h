/*
 * rapid.h — C ABI of the B200-native RAPID / CTFTPS superpixel refinement library.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   The coarse-to-fine topology-preserving superpixel refinement (CTFTPS, §2.1)
 *   as modified by RAPID (§3): superpixels start as a regular grid (RAPID l.1,
 *   P:124); at every block stage (RAPID l.5-8) each boundary block may be
 *   relabelled to a 4-neighbouring superpixel (Eq. 3) under the energy of Eq. 1
 *   (colour + lambda_pos position + lambda_b boundary length, Eq. 2) if the move
 *   keeps every superpixel 4-connected (E_topo) and, in the size-regularity modes,
 *   the superpixel above l*InitSize (E_size P:68 / §3.1); undersized superpixels are
 *   merged into the contiguous superpixel of least merged energy within u*InitSize
 *   (Eqs. 4-5); after the coarsest stage a classifier (Eq. 6) gates
 *   which superpixels are refined later (Eq. 7); coarsest-level
 *   statistics are reused at finer levels (Eq. 8).
 *   The exact deterministic schedule (2x2 parity-coloured sweeps, frozen per-phase
 *   fixed-point means, all-or-nothing size budget, ordered merge rounds) and every reading
 *   of an ambiguous passage are listed in DESIGN.md §2.  Output label maps are bit-exact
 *   with the CPU oracle (oracle/) under those readings.
 *
 * Conventions
 *   - All entry points return int status (RAPID_OK = 0, negative = error, see below);
 *     nothing throws across the ABI; argument validation happens before any launch.
 *   - Device pointers are CUDA device addresses on the ctx's device.  Host pointers are
 *     ordinary (preferably pinned) host memory.  `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).
 *   - Ownership: images and label buffers belong to the caller and must stay valid until
 *     the stream work completes; the ctx owns every internal buffer.
 *   - Threading: one ctx per concurrently used stream; calls on one ctx are not reentrant.
 */
#ifndef RAPID_H
#define RAPID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAPID_MAX_STAGES 12
#define RAPID_MAX_SWEEPS 64
#define RAPID_MAX_PROTO 4
#define RAPID_NCNT 6

/* status codes */
#define RAPID_OK 0
#define RAPID_E_ARG (-1)       /* null pointer, bad sizes, bad stage list, l>=1, u<=1, ... */
#define RAPID_E_CAPACITY (-2)  /* B*H*W or B*M exceeds the capacity given to rapid_init */
#define RAPID_E_RANGE (-3)     /* values that could overflow the integer energy parts */
#define RAPID_E_CUDA (-4)      /* a CUDA call failed; rapid_last_error() has the message */
#define RAPID_E_OOM (-5)       /* device allocation failed */
#define RAPID_E_INTEGRITY (-6) /* RECOUNT mode found reused sums != recount (never expected) */
#define RAPID_E_STATE (-7)     /* stats/profile requested before any segmentation */

/* size_mode: how E_size is handled */
#define RAPID_SIZE_NONE 0  /* lambda_s = 0: no size limit (CTFTPS case 1) */
#define RAPID_SIZE_HARD 1  /* lambda_s = inf: moves below l*InitSize rejected (case 2) */
#define RAPID_SIZE_MERGE 2 /* RAPID regularity optimisation: merge instead (§3.1) */

/* mask_rule: which blocks are refined after the coarsest stage (RAPID l.3-4, l.14) */
#define RAPID_MASK_OFF 0   /* everything is refined (CTFTPS) */
#define RAPID_MASK_CLASS 1 /* superpixels with y=+1 (config text: ROI-like colour) */
#define RAPID_MASK_BSP 2   /* "boundary superpixels": a 4-adjacent superpixel of the other class */
#define RAPID_MASK_EQ7 3   /* block-level Eq. 7: a neighbour with another label and another class */

/* stats_mode */
#define RAPID_STATS_REUSE 0   /* RAPID: coarsest-level sums reused (Eq. 8, exact here) */
#define RAPID_STATS_RECOUNT 1 /* multi-scale CTFTPS: recount at every stage (checked equal) */
#define RAPID_STATS_PYRAMID 2 /* literal image pyramid — block colour data are area x
                                 the rounded box mean of the next finer level, S_1 from
                                 the coarsest level, reused by Eq. 8 (the paper's approximation;
                                 A32) */

/* how the prediction step (RAPID l.3-4, Eq. 6) computes y of each superpixel */
#define RAPID_Y_PROTO 0    /* distance of the mean colour to the prototypes (A21) */
#define RAPID_Y_FEATURES 1 /* linear h_theta on the 4 features of P:271 (A31) */

/* per-phase counters (rapid_run_info.phase) */
#define RAPID_C_CAND 0    /* gated boundary blocks of the phase colour */
#define RAPID_C_TOPO 1    /* ... that passed the simple-point test */
#define RAPID_C_PROP 2    /* proposals: dE<0 and the single-move size gate passed */
#define RAPID_C_SIZEREJ 3 /* desired moves rejected by the single-move size gate */
#define RAPID_C_COMMIT 4  /* committed moves */
#define RAPID_C_COMMREJ 5 /* proposals dropped by the all-or-nothing size budget */

typedef struct rapid_ctx rapid_ctx; /* opaque; owns all device workspace */

/* Parameters of one segmentation call.  Integers only, so results are bit-reproducible. */
typedef struct {
  uint32_t struct_size;      /* = sizeof(rapid_params) (ABI check) */
  uint32_t batch;            /* B >= 1 independent images of H x W (A27) */
  uint32_t n_superpixels;    /* M per image; grid r x c = M with the squarest cells */
  uint32_t n_stages;         /* 1..RAPID_MAX_STAGES */
  uint32_t block_size[RAPID_MAX_STAGES]; /* descending, 1..64, each divides the previous;
                                            the last is the final grain (Table 1) */
  uint32_t sweeps;           /* parity sweeps per stage, 0..RAPID_MAX_SWEEPS (A5, A25) */
  uint8_t pad0_[4];          /* explicit padding (ignored; zeroed in the graph-cache key) */
  int64_t lambda_pos_q16;    /* lambda_pos in Q16.16, 0..2^31-1 */
  int64_t lambda_b_q16;      /* lambda_b in Q16.16 per ordered pixel pair, 0..2^31-1 (A3) */
  uint32_t size_mode;        /* RAPID_SIZE_* */
  uint32_t l_num, l_den;     /* lower size bound l = l_num/l_den < 1 (default 1/4) */
  uint32_t u_num, u_den;     /* upper size bound u = u_num/u_den > 1 (Eq. 5; default 3/2) */
  uint32_t mask_rule;        /* RAPID_MASK_* */
  uint32_t n_proto;          /* 1..4 when mask_rule != OFF */
  uint8_t proto_rgb[RAPID_MAX_PROTO][3]; /* prototypes of h_theta (A21) */
  uint8_t pad_[8];           /* explicit padding (ignored; zeroed in the graph-cache key) */
  int64_t tau2;              /* y=+1 iff min_k ||c - proto_k||^2 <= tau2 (Eq. 6; intensity^2) */
  uint32_t stats_mode;       /* RAPID_STATS_* */
  uint32_t y_model;          /* RAPID_Y_* */
  /* RAPID_Y_FEATURES: y = +1 iff w[0] 2^16 + sum_i w[i] f_i >= 0 with the features f1..f4 in
   * Q16 (absolute and comparative brightness, intra- and extra-region dissimilarity; A31)
   * and w in Q16.16, |w| < 2^31 (a model file's bias and weights, rounded) */
  int64_t feat_w_q16[5];
} rapid_params;

/* Per-superpixel result, index img*M + local id. */
typedef struct {
  int64_t n, sum_r, sum_g, sum_b, sum_x, sum_y; /* exact integer sums (x = column) */
  double mean_r, mean_g, mean_b, mean_x, mean_y; /* sum / n (0 when n == 0) */
  int32_t init_size;                            /* InitSize (cell area) */
  int8_t alive, active, y;                      /* y in {-1,+1}, 0 = not predicted */
  int8_t pad_;
} rapid_sp_stat;

typedef struct {
  int32_t status;            /* status of the last segmentation (deferred errors) */
  uint32_t batch, H, W, n_superpixels, n_stages, sweeps;
  uint32_t grid_rows, grid_cols;
  uint32_t stage_nbx[RAPID_MAX_STAGES], stage_nby[RAPID_MAX_STAGES];
  uint64_t stage_tiles[RAPID_MAX_STAGES];        /* tiles of the stage map */
  uint64_t stage_active_tiles[RAPID_MAX_STAGES]; /* tiles on the worklist */
  uint64_t stage_victims[RAPID_MAX_STAGES];      /* victims at the stage's merge round */
  uint64_t stage_merges[RAPID_MAX_STAGES];
  uint64_t stage_sweeps_run[RAPID_MAX_STAGES];   /* sweeps actually executed (exact early exit) */
  uint64_t stage_window_blocks[RAPID_MAX_STAGES];/* blocks within distance 1 of a block whose label
                                                    can pass the gate (profiling level 2; else 0) */
  uint64_t alive, active;                        /* after the run */
  uint64_t phase[RAPID_MAX_STAGES][RAPID_MAX_SWEEPS][4][RAPID_NCNT]; /* RAPID_C_* */
} rapid_run_info;

/* Kernel timing (profiling mode): per kernel class and stage. */
#define RAPID_K_PYRAMID 0
#define RAPID_K_SNAPSHOT 1
#define RAPID_K_PROPOSE 2
#define RAPID_K_COMMIT 3
#define RAPID_K_MERGE 4
#define RAPID_K_PREDICT 5
#define RAPID_K_TRANSITION 6
#define RAPID_K_FINAL 7
#define RAPID_K_PHASESET 8 /* snapshot+scan+eval+commit of every phase of the stage, as one interval */
#define RAPID_K_EVAL 9     /* K4b candidate evaluation (RAPID_K_PROPOSE is the K4a scan) */
#define RAPID_NK 10
typedef struct {
  uint64_t launches[RAPID_NK][RAPID_MAX_STAGES];
  double ms[RAPID_NK][RAPID_MAX_STAGES];
  uint64_t total_launches; /* every kernel of the last segmentation */
} rapid_profile;

/* Create a context on CUDA device `device`, sized for at most `max_pixels_total` = B*H*W
 * pixels and `max_superpixels_total` = B*M superpixels per call.  *out = NULL on error. */
int rapid_init(rapid_ctx **out, int device, uint64_t max_pixels_total,
               uint64_t max_superpixels_total);

/* Segment image (device, u8 [B][H][W][3], RGB, row-major) into labels_out (device, int32
 * [B][H][W], per-image local ids in [0, M); merged-away ids are absent).  Only enqueues
 * work on `stream`; returns after validation and launch. */
int rapid_segment(rapid_ctx *ctx, const uint8_t *image, int32_t H, int32_t W,
                  const rapid_params *params, int32_t *labels_out, void *stream);

/* Same, end to end from host buffers: copies image_host to the device, segments, copies
 * the labels back into labels_host, and synchronises `stream` before returning. */
int rapid_segment_host(rapid_ctx *ctx, const uint8_t *image_host, int32_t H, int32_t W,
                       const rapid_params *params, int32_t *labels_host, void *stream);

/* A stream of n independent segmentations from host buffers, all with the same H, W and
 * params: images_host[k] (u8 [B][H][W][3]) -> labels_host[k] (int32 [B][H][W]), k = 0..n-1.
 * Equivalent to n rapid_segment_host calls, but pipelined over two device buffer pairs and
 * two copy streams: the labels of segmentation k travel to the host while the image of k+1
 * is copied in and segmented (copies of each direction stay in order; host buffers should be
 * pinned for the copies to overlap).  Segmentations run on `stream`; returns after every
 * label buffer is written, with the first error status of any of them (RAPID_E_INTEGRITY when
 * a RECOUNT check failed).  rapid_stats afterwards reports the last segmentation.
 * Errors: RAPID_E_ARG (n < 1, a null buffer), otherwise as rapid_segment_host. */
int rapid_segment_host_stream(rapid_ctx *ctx, const uint8_t *const *images_host, int32_t *const *labels_host,
                              int32_t n, int32_t H, int32_t W, const rapid_params *params, void *stream);

/* segmentation quality (the metrics of the paper's §4.2) of a label
 * map against a ground-truth segment map, on the GPU.  labels: device int32 [B][H][W],
 * per-image ids in [0, M); gt: device int32 [B][H][W], per-image segment ids >= 0.  Each
 * image is scored on its own; counts are summed over the batch:
 *   UE  = sum over images, segments S and superpixels sp meeting S of
 *         min(|sp n S|, |sp \ S|), divided by B*H*W (under-segmentation error);
 *   BR  = (# GT boundary pixels with a superpixel boundary pixel within Chebyshev distance
 *         eps) / (# GT boundary pixels), 1 when there is none; a boundary pixel of a map is a
 *         pixel with an in-image 4-neighbour of another id (boundary recall).
 * Enqueues on `stream`, synchronises it and writes *out_host.  Errors: RAPID_E_ARG (bad
 * sizes, eps < 0, or an id out of range found on the device), RAPID_E_CAPACITY (more distinct
 * (superpixel, segment) pairs than the histogram holds: 2^26), RAPID_E_CUDA, RAPID_E_OOM.
 * The workspace (pair histogram, sizes, one byte per pixel) is allocated on first use. */
typedef struct {
  double ue, br;
  uint64_t pixels, leak_px, gt_boundary_px, covered_px, pairs;
} rapid_quality_result;
int rapid_quality(rapid_ctx *ctx, const int32_t *labels, const int32_t *gt, int32_t B, int32_t H, int32_t W,
                  int32_t M, int32_t eps, rapid_quality_result *out_host, void *stream);

/* Synchronise the last segmentation's stream and copy per-superpixel stats (up to
 * `capacity` entries; out_host may be NULL) and run info (may be NULL) to the host.
 * Returns the deferred status of that segmentation (e.g. RAPID_E_INTEGRITY). */
int rapid_stats(rapid_ctx *ctx, rapid_sp_stat *out_host, uint64_t capacity,
                rapid_run_info *info_host);

/* Profiling: level 1 = CUDA events bracket every kernel class per stage; level 2 also
 * counts each stage's window blocks (rapid_run_info.stage_window_blocks; extra kernels);
 * level 3 = coarse: events bracket only each stage's whole phase set (RAPID_K_PHASESET) and the
 * kernel classes outside the phase loop, none between the K3/K4/K5 launches (the nested events
 * of level 1 add ~7 us per launch group to that interval). */
int rapid_set_profiling(rapid_ctx *ctx, int enable);
int rapid_get_profile(rapid_ctx *ctx, rapid_profile *out_host); /* synchronises */

void rapid_free(rapid_ctx *ctx); /* synchronises first; NULL is a no-op */
const char *rapid_status_string(int status);
const char *rapid_last_error(const rapid_ctx *ctx);

/* ---- debug (parity bisection against the oracle; not for production use) ---------- */
#define RAPID_STOP_NONE 0
#define RAPID_STOP_PHASE 1        /* after the commit of (stage, sweep, phase) */
#define RAPID_STOP_STAGE_START 2  /* after the transition into `stage` */
#define RAPID_STOP_AFTER_MERGE 3  /* after the merge round of `stage` */
#define RAPID_STOP_AFTER_PREDICT 4
/* The next segmentation stops at the given point (labels_out is then undefined);
 * rapid_debug_map copies the stage map [B][nby][nbx] there to the host. */
int rapid_debug_stop(rapid_ctx *ctx, int kind, int stage, int sweep, int phase);
int rapid_debug_map(rapid_ctx *ctx, int32_t *host, uint64_t capacity, int32_t *nbx,
                    int32_t *nby);

#ifdef __cplusplus
}
#endif
#endif /* RAPID_H */
