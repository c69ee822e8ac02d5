/*
 * tsa.h -- C ABI of libtsa: B200-native (sm_100a) Tsallis-entropy multilevel
 * thresholding of CT slices, the data-parallel hot path of arXiv 2012.10684
 * ("GPU acceleration of patient-specific airway image segmentation").
 *
 * Problem statement (PAPER.md v2; line numbers of /root/reference/PAPER.md):
 *   image in -> threshold selected by maximising Tsallis entropy -> Algorithm 1
 *   applied, generalised per slice to
 *   k thresholds of the 1-D gray-level histogram (BASELINE.json:north_star):
 *     c_i   = #{voxels of slice z with value i}, i < bins
 *     p_i   = c_i / N
 *     class C_0 = [0,t_1], C_j = [t_j+1, t_{j+1}], C_k = [t_k+1, bins-1]
 *     A_j   = sum_{i in C_j} (p_i / P_j)^q,  S_j = (1 - A_j)/(q - 1)
 *             (q == 1: S_j = -sum (p_i/P_j) ln(p_i/P_j))
 *     phi   = S_0 (+) S_1 (+) ... (+) S_k,  x (+) y = x + y + (1-q) x y
 *             (TSA_OBJ_SUM_PLUS_PRODUCT: sum S_j + (1-q) prod S_j)
 *     t*    = argmax phi over 0 <= t_1 < ... < t_k <= bins-2, every class
 *             non-empty, lowest tuple on exact ties
 *     label = #{ j : v > t*_j }  (Algorithm 1 with T = t+1 for k = 1)
 *   The readings behind these lines are DESIGN.md R1-R17.
 *
 * Conventions for every entry point:
 *   - Every data pointer is a DEVICE pointer on the current CUDA device unless
 *     its comment says "host".  Layouts are C-contiguous.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are asynchronous on that stream: they validate arguments on the
 *     host, enqueue kernels and return; they never synchronise, never allocate
 *     or free device memory and keep no global mutable state, so a whole
 *     tsa_segment call can be captured in a CUDA graph.
 *   - The caller owns every buffer, including the workspace (size from the
 *     matching *_workspace_size call, 256-byte aligned).
 *   - Argument errors return TSA_ERR_INVALID_ARG before anything is enqueued.
 *     Data-dependent errors are reported per slice in slice_status (the call
 *     itself returns TSA_OK): TSA_ERR_LEVEL_OVERFLOW when any voxel >= bins
 *     (never clamped), TSA_ERR_NO_VALID_SPLIT when fewer than k+1 bins are
 *     non-empty.  A failed slice gets thresholds -1, objective NaN, labels 0.
 *   - CUDA launch failures return TSA_ERR_CUDA, transport (NCCL) failures of
 *     the multi-GPU calls TSA_ERR_NCCL; tsa_last_error() gives detail
 *     (thread-local).
 */
#ifndef TSA_H
#define TSA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSA_VERSION 1
#define TSA_KMAX 4
#define TSA_BINS_MAX 4096
#define TSA_KEY_NONE 0xFFFFFFFFFFFFFFFFull /* partial key of "no valid tuple" */

typedef enum {
  TSA_OK = 0,
  TSA_ERR_INVALID_ARG = 1,
  TSA_ERR_LEVEL_OVERFLOW = 2,
  TSA_ERR_NO_VALID_SPLIT = 3,
  TSA_ERR_WORKSPACE = 4,
  TSA_ERR_CUDA = 5,
  TSA_ERR_NCCL = 6
} tsa_status;

typedef enum { TSA_U8 = 1, TSA_U16 = 2 } tsa_dtype;

/* R1: the k >= 2 objective.  PSEUDO_ADDITIVE is the paper's two-class rule
 * folded over k+1 classes (default); SUM_PLUS_PRODUCT is the multilevel
 * literature's alternative. */
typedef enum { TSA_OBJ_PSEUDO_ADDITIVE = 0, TSA_OBJ_SUM_PLUS_PRODUCT = 1 } tsa_objective;

/* Which tuples the exhaustive search evaluates.  FULL: every t_1<...<t_k in
 * [0, bins-2] (C(bins-1,k) tuples, invalid ones skipped).  CANONICAL: only
 * tuples whose every t_j is a non-empty bin (C(m-1,k) tuples, m = non-empty
 * bins).  Both return the same (bit-identical) t* and score: tuples that
 * differ only by empty bins describe the same partition, evaluate to the same
 * value bit for bit, and the lowest of them is the canonical one. */
typedef enum { TSA_ENUM_CANONICAL = 0, TSA_ENUM_FULL = 1, TSA_ENUM_DP = 2 } tsa_enumeration;
/* TSA_ENUM_DP: not an enumeration but an exact
 * interval dynamic programme over the canonical positions, O(k m^2) class
 * terms: maximises sum_j g(C_j), g = ln A (q < 1), -ln A (q > 1), S (q == 1),
 * which orders tuples as phi does (phi = (prod A_j - 1)/(1 - q), R1).  Returns
 * the lexicographically smallest optimum of that sum; it differs from the
 * exhaustive argmax only on partitions whose objectives differ by rounding.
 * PSEUDO_ADDITIVE only (INVALID_ARG otherwise); one work unit per slice. */

typedef struct {
  const void *volume;   /* [nz][ny][nx] u8 or u16, device */
  int32_t dtype;        /* tsa_dtype */
  int64_t nx, ny, nz;   /* > 0; nx*ny < 2^31; nz <= 65535 */
  int32_t bins;         /* L: 2..256 for u8, 2..4096 for u16 */
  int32_t k;            /* thresholds per slice, 1..4, k <= bins-1 */
  double q;             /* entropic index q (alpha), > 0 and finite; q == 1 is Shannon */
  int32_t objective;    /* tsa_objective */
  int32_t enumeration;  /* tsa_enumeration */
  int32_t units_per_slice; /* search work units per slice (0 = library heuristic) */
  /* tsa_segment schedule (0 = library default for every field):
   *   pipeline     2 = compact: three kernels (histogram partials + class-term table,
   *                one CTA per slice for tables/search/argmax/phi, labels);
   *                1 = one persistent fused kernel (the same work overlapped
   *                through a dependency-ordered task queue); both need k <= 2,
   *                bins <= 1024, CANONICAL, PSEUDO_ADDITIVE, nx*ny % 16 == 0,
   *                16-byte aligned volume and labels;
   *                3 = stream: ONE persistent kernel whose io CTAs stream
   *                histogram chunks and label chunks while its search CTAs
   *                run each slice's tables and exhaustive search (k = 2,
   *                CANONICAL, PSEUDO_ADDITIVE, nx*ny % 16 == 0, aligned);
   *                4 = overlap: the staged kernels on slabs of slices over
   *                the caller's stream and a second stream the call creates,
   *                so the histogram / labels of one slab overlap the search of
   *                another (any problem; staged while the stream is being
   *                captured into a CUDA graph);
   *                -1 = staged: one kernel per stage (any problem);
   *                0 = overlap for k = 2 above 1024 bins with >= 16 slices,
   *                else compact whenever eligible, else staged
   *   slab_slices  fused: slices per pipeline slab; compact: histogram CTAs
   *                per SM (default 4); stream: histogram / label chunks per
   *                slice (default ~256 K voxels each); overlap: number of
   *                slabs (default 8, at most 64)
   *   label_lag    fused: rounds by which labelling trails the histogram;
   *                stream: slices by which labelling trails the histogram
   *                (default 16); compact: ignored */
  int32_t pipeline;
  int32_t slab_slices;
  int32_t label_lag;
} tsa_problem;

typedef struct {
  int32_t *thresholds;   /* [nz][k], required; t_1<...<t_k in [0,bins-2]; -1 on slice error */
  uint8_t *labels;       /* [nz][ny][nx] or NULL = skip labelling */
  double *objective;     /* [nz] or NULL; phi(t*) recomputed in the definition's order; NaN on error */
  uint32_t *histogram;   /* [nz][bins] or NULL (then kept in the workspace) */
  int32_t *slice_status; /* [nz] or NULL; tsa_status per slice */
} tsa_outputs;

/* Validate a problem (host only, no CUDA calls).  TSA_OK or TSA_ERR_INVALID_ARG. */
tsa_status tsa_validate(const tsa_problem *p);

/* Bytes of workspace tsa_segment needs for this problem (0 if invalid). */
size_t tsa_workspace_size(const tsa_problem *p);

/* Which implementation tsa_segment runs for this problem: 4 = overlap (staged
 * kernels on two streams), 3 = stream (one
 * persistent kernel), 2 = compact (3 kernels), 1 = persistent fused kernel,
 * -1 = staged (one kernel per stage), 0 = invalid problem.  (Labels must also
 * be 16-byte aligned for 1, 2 and 3.) */
int32_t tsa_pipeline_kind(const tsa_problem *p);

/* The whole hot path on one stream:
 * histogram -> tables (prefix scans) -> exhaustive search -> argmax/finalize
 * -> labels. */
tsa_status tsa_segment(const tsa_problem *p, const tsa_outputs *out, void *workspace,
                       size_t workspace_bytes, void *stream);

/* ---- stage calls (parity tests, ncu, tuple sharding) ------------------- */

/* a1: hist[z][i] = #{v == i} over the slice's in-range voxels; slice_status[z]
 * = TSA_OK or TSA_ERR_LEVEL_OVERFLOW.  Both outputs are fully overwritten. */
tsa_status tsa_histogram(const tsa_problem *p, uint32_t *hist, int32_t *slice_status,
                         void *stream);

/* Workspace for tsa_search of nz slices of bins bins (same for every unit range). */
size_t tsa_search_workspace_size(int64_t nz, int64_t voxels_per_slice, int32_t bins, int32_t k,
                                 double q, int32_t objective, int32_t enumeration);

/* Units per slice the library would pick for this shape (what units_per_slice=0 means). */
int32_t tsa_default_units(int64_t nz, int32_t bins, int32_t k, int32_t enumeration);

/* a2+a3: prefix-scan tables and the exhaustive search over work units
 * [unit_begin, unit_end) of units_per_slice units per slice.  Unit u of slice z
 * covers a fixed, rank-independent range of the slice's tuples, so disjoint
 * unit ranges on different GPUs partition the tuple space.
 *   hist            [nz][bins] (from tsa_histogram)
 *   slice_status    [nz] in/out: slices not TSA_OK are skipped; TSA_ERR_NO_VALID_SPLIT
 *                   is set when fewer than k+1 bins are non-empty
 *   part_score      [unit_end-unit_begin][nz] f64 out: best score per unit (score = phi-
 *                   monotone comparison quantity, higher is better; -inf if none)
 *   part_key        [unit_end-unit_begin][nz] u64 out: packed tuple of that score:
 *                   sum_j t_j << 12*(k-1-j) (integer order == lexicographic order);
 *                   TSA_KEY_NONE if none. */
tsa_status tsa_search(const uint32_t *hist, int32_t *slice_status, int64_t nz,
                      int64_t voxels_per_slice, int32_t bins, int32_t k, double q,
                      int32_t objective, int32_t enumeration, int32_t units_per_slice,
                      int32_t unit_begin, int32_t unit_end, double *part_score,
                      uint64_t *part_key, void *workspace, size_t workspace_bytes,
                      void *stream);

/* The class-size constants of every search kernel (a2/a3), exposed so tests
 * can check them against the definition.  A class of n voxels contributes
 * A = W / n^q (q != 1; PAPER.md:581-591 with p_i/P_j = c_i/n, R11)
 * or S = ln n - W/n (q == 1, R6); the library computes n^-q, ln n and 1/n
 * from a 33 KB table (j^-q or ln j and 1/j for j <= 2^11, 2^(-s q)) and a
 * degree-6 (q > 10: 12) polynomial in d = r/(j 2^s) < 2^-10, n = 2^s j + r
 * -- no N-sized table.
 *   n      [count] u32 class sizes (0 gives NaN)
 *   a      [count] f64 out: n^-q (q != 1) or ln n (q == 1)
 *   b      [count] f64 out or NULL: 1/n (q == 1 only; untouched otherwise)
 *   workspace  tsa_class_consts_workspace_size() bytes */
size_t tsa_class_consts_workspace_size(void);
tsa_status tsa_class_consts(const uint32_t *n, int64_t count, double q, double *a, double *b,
                            void *workspace, size_t workspace_bytes, void *stream);

/* a4 (partial): merge nparts [nparts][nz] partials into [nz] under the total
 * order (score desc, key asc).  Used before a cross-rank exchange. */
tsa_status tsa_merge(const double *part_score, const uint64_t *part_key, int32_t nparts,
                     int64_t nz, double *score, uint64_t *key, void *stream);

/* a4: merge partials, decode t*, recompute phi(t*) from the histogram in the
 * definition's order, write out->thresholds / objective / slice_status
 * (out->labels and out->histogram are ignored). */
tsa_status tsa_finalize(const uint32_t *hist, const int32_t *slice_status, int64_t nz,
                        int32_t bins, int32_t k, double q, int32_t objective,
                        const double *part_score, const uint64_t *part_key, int32_t nparts,
                        const tsa_outputs *out, void *stream);

/* a5: labels[z][y][x] = #{j : v > thresholds[z][j]}; 0 for slices whose
 * slice_status (may be NULL = all OK) is not TSA_OK. */
tsa_status tsa_label(const tsa_problem *p, const int32_t *thresholds,
                     const int32_t *slice_status, uint8_t *labels, void *stream);

/* Host-buffer convenience: copies a HOST volume (pinned recommended) to the
 * device in slabs, runs tsa_segment per slab and copies thresholds, objective,
 * status and (if labels_host != NULL) labels back: compute on stream0,
 * copy-out on stream1, copy-in on a stream the call creates and destroys,
 * ordered by events over three device slab buffers, so the H2D and D2H copy engines
 * and the kernels run concurrently.  Device scratch (dev_buf, dev_bytes) comes from the
 * caller: tsa_segment_host_scratch_size() bytes.  Blocks until done. */
size_t tsa_segment_host_scratch_size(const tsa_problem *p, int64_t slab_slices);
tsa_status tsa_segment_host(const tsa_problem *p_host_volume, int64_t slab_slices,
                            int32_t *thresholds_host, double *objective_host,
                            int32_t *status_host, uint8_t *labels_host, void *dev_buf,
                            size_t dev_bytes, void *stream0, void *stream1);

/* ---- q sweep: one histogram, the search and labels for several q --------
 * PAPER.md:564 ("the alpha coefficient can be adjusted and plays a critical
 * role in tuning"); BASELINE.json config 3 sweeps q in {0.5, ..., 1.5}.
 * Equivalent, output for output, to nq tsa_segment calls on the same volume
 * with p->q replaced by qs[i] (bit-identical; tested), but the volume is
 * histogrammed once: a1 once, a2-a5 per q, always one kernel per stage.
 *   qs    host array [nq] of q values (each > 0 and finite), nq in 1..64
 *   outs  host array [nq] of tsa_outputs; outs[i] receives the results of
 *         qs[i] (thresholds required; labels / objective / slice_status
 *         optional; every non-NULL histogram receives the volume's histogram)
 *   workspace  tsa_sweep_workspace_size(p, qs, nq) bytes (p->q is ignored) */
size_t tsa_sweep_workspace_size(const tsa_problem *p, const double *qs, int32_t nq);
tsa_status tsa_segment_sweep(const tsa_problem *p, const double *qs, int32_t nq,
                             const tsa_outputs *outs, void *workspace, size_t workspace_bytes,
                             void *stream);

/* ---- multi-GPU: one process per GPU, slices or tuples sharded ------------
 * (SURVEY.md §8(b),(e); "job distribution ... reduction of
 * results from different devices", Table "multiple" PAPER.md:726-739.)
 *
 * A tsa_comm is an all-gather transport between nranks processes, each
 * driving one GPU.  tsa_comm_init builds it on NCCL (libnccl.so.2, loaded
 * at the first call with dlopen; the communicator is owned by the tsa_comm
 * and freed by tsa_comm_destroy -- the one object the library allocates).
 * tsa_comm_init_custom wraps a caller-provided all-gather instead (any
 * transport: MPI, gloo, shared memory; the tests use it to run two ranks on
 * one GPU, which NCCL refuses).
 *
 * Slab partition (tsa_slab_range): rank r owns slices [r c, min(nz, (r+1) c)),
 * c = ceil(nz / nranks); trailing ranks may own none.
 *
 * tsa_segment_sharded, on `stream`, with `slab` = this rank's slices (slab->nz
 * = z1 - z0, may be 0 with volume NULL in TUPLES mode) and nz_total slices in
 * the whole volume:
 *   TSA_SHARD_SLICES  slices are independent problems: the rank segments its
 *                     slab with no exchange (tsa_segment); every output refers
 *                     to the slab.  The comm is only checked (rank, nranks).
 *   TSA_SHARD_TUPLES  the tuple space of EVERY slice is split over the ranks
 *                     (large k): histogram of the own slab -> all-gather of
 *                     the histograms and statuses -> exhaustive search of the
 *                     rank's share of the work units of all nz_total slices
 *                     -> per-slice merge -> all-gather of the (score, key)
 *                     partials -> merge under (score desc, key asc) and
 *                     phi(t*) in the definition's order (tsa_finalize) ->
 *                     labels of the own slab.  out->thresholds [nz_total][k],
 *                     objective [nz_total], slice_status [nz_total] and
 *                     histogram [nz_total][bins] (optional) are identical on
 *                     every rank; out->labels is the own slab [z1-z0][ny][nx].
 *                     Work units per slice: slab->units_per_slice, else a
 *                     rank-independent default (never the local SM count), so
 *                     the unit ranges partition the same space on every rank
 *                     and the result is bit-identical to one GPU.
 * Exchanged bytes per call (TUPLES): nranks c (4 bins + 4) + 16 nranks nz_total.
 * Transport failures return TSA_ERR_NCCL with detail in tsa_last_error().
 * The call blocks only as much as the transport does (NCCL: asynchronous on
 * the stream; a custom all-gather decides). */
typedef struct tsa_comm tsa_comm;
typedef enum { TSA_SHARD_SLICES = 0, TSA_SHARD_TUPLES = 1 } tsa_shard_mode;
#define TSA_COMM_ID_BYTES 128

/* Custom all-gather: gather `bytes` from every rank's `send` into `recv`
 * (rank-major, nranks * bytes), device pointers, ordered after prior work on
 * `stream` and before later work on it.  Return 0 on success. */
typedef int (*tsa_allgather_fn)(void *user, const void *send, void *recv, size_t bytes,
                                void *stream);

/* id: host buffer of TSA_COMM_ID_BYTES; rank 0 creates it, every rank passes
 * the same bytes to tsa_comm_init (the caller distributes them). */
tsa_status tsa_comm_unique_id(unsigned char id[TSA_COMM_ID_BYTES]);
tsa_status tsa_comm_init(tsa_comm **comm, int32_t nranks, int32_t rank,
                         const unsigned char id[TSA_COMM_ID_BYTES]);
tsa_status tsa_comm_init_custom(tsa_comm **comm, int32_t nranks, int32_t rank,
                                tsa_allgather_fn allgather, void *user);
tsa_status tsa_comm_destroy(tsa_comm *comm);
/* 1 = NCCL, 2 = custom, 0 = NULL comm */
int32_t tsa_comm_kind(const tsa_comm *comm);

/* host: [z0, z1) of `rank` (the partition tsa_segment_sharded expects) */
tsa_status tsa_slab_range(int64_t nz_total, int32_t nranks, int32_t rank, int64_t *z0, int64_t *z1);

/* Work units per slice TSA_SHARD_TUPLES uses (identical on every rank). */
int32_t tsa_sharded_units(const tsa_problem *slab, int64_t nz_total, int32_t nranks);

size_t tsa_sharded_workspace_size(const tsa_problem *slab, int64_t nz_total, int32_t shard_mode,
                                  const tsa_comm *comm);
tsa_status tsa_segment_sharded(const tsa_problem *slab, int64_t nz_total, const tsa_outputs *out,
                               int32_t shard_mode, tsa_comm *comm, void *workspace,
                               size_t workspace_bytes, void *stream);

/* ---- 2-D Tsallis thresholding: the paper's own formulation -------------
 * (readings DESIGN.md R18-R22)
 *   g(x,y)   = floor( sum_{3x3} f / 9 ), replicate border
 *   h[i][j]  = #{(x,y) : f = i, g = j}
 *   class 1  = {i <= t, j <= s}, class 2 = {i > t, j > s}
 *   H_c      = (1 - sum_{class c} (p_ij / P_c)^q) / (q - 1)      (q == 1: Shannon)
 *   phi(t,s) = H_1 + H_2 + (1 - q) H_1 H_2
 *   (t*,s*)  = argmax over 0 <= t, s <= bins-2 with both classes non-empty,
 *              lowest (t,s) in row-major order on exact ties        (R21)
 *   label    = [f > t*]  ("only t is used as the threshold value")
 * Conventions as above (device pointers, caller-owned buffers and workspace,
 * asynchronous on `stream`, argument errors before any launch, per-slice
 * data errors: TSA_ERR_LEVEL_OVERFLOW if any f >= bins or g >= bins,
 * TSA_ERR_NO_VALID_SPLIT if no (t,s) has two non-empty classes). */
typedef struct {
  const void *volume;   /* [nz][ny][nx] u8, device */
  int64_t nx, ny, nz;   /* > 0; nx <= 65535; nz <= 65535; nx*ny < 2^31 */
  int32_t bins;         /* L: 2..256 */
  double q;             /* > 0 and finite; q == 1 is Shannon */
  int32_t cluster;      /* CTAs per slice (one thread-block cluster each): 0 = library
                           default, else 4..8 (the L x L histogram is split by f-rows
                           over the cluster's shared memory) */
} tsa2d_problem;

/* TSA_OK or TSA_ERR_INVALID_ARG (host only). */
tsa_status tsa2d_validate(const tsa2d_problem *p);

/* Bytes of workspace tsa2d_segment / tsa2d_histogram need (0 if invalid). */
size_t tsa2d_workspace_size(const tsa2d_problem *p);

/* CTAs per cluster the library uses for this problem (0 if invalid): the
 * explicit `cluster` if set, else the smallest of 4..8 whose CTAs each count
 * <= 65536 pixels in one round (4 for 512x512) and whose shared-memory plan
 * fits; slices too large for that count in rounds of <= 65535 pixels. */
int32_t tsa2d_cluster_size(const tsa2d_problem *p);

/* The whole 2-D path: mean image, 2-D histogram, exhaustive (t,s) search,
 * argmax, phi(t*,s*) recomputed from the definition, labels.
 *   out->thresholds   [nz][2] (t*, s*), required; -1 on slice error
 *   out->labels       [nz][ny][nx] u8 or NULL: [f > t*], 0 on slice error
 *   out->objective    [nz] f64 or NULL: phi(t*,s*); NaN on slice error
 *   out->histogram    [nz][bins][bins] u32 or NULL: h
 *   out->slice_status [nz] or NULL */
tsa_status tsa2d_segment(const tsa2d_problem *p, const tsa_outputs *out, void *workspace,
                         size_t workspace_bytes, void *stream);

/* The 2-D histogram alone: hist [nz][bins][bins] u32 (required), slice_status
 * [nz] (required): TSA_OK or TSA_ERR_LEVEL_OVERFLOW. */
tsa_status tsa2d_histogram(const tsa2d_problem *p, uint32_t *hist, int32_t *slice_status,
                           void *workspace, size_t workspace_bytes, void *stream);

/* The mean image alone: g [nz][ny][nx] u8. */
tsa_status tsa2d_mean3x3(const tsa2d_problem *p, uint8_t *g, void *stream);

/* ---- HU input: pre-processing fused into the histogram and label passes ---
 * (readings DESIGN.md R23-R25)
 *   lo, hi = volume-wide min / max of the voxels != background
 *   g(v)   = 0 for the background; else round-half-away(255 (v-lo)/(hi-lo)),
 *            0 when hi == lo                                    (the 8-bit image)
 * then the 1-D path on g with 256 bins: thresholds are 8-bit levels, labels
 * #{j : g(v) > t_j}.  The volume is read twice (HU histogram + window pass,
 * label pass); the 8-bit image is never materialised.
 * Requirements: nx*ny % 16 == 0, nz <= 65535, volume (and labels) 16-byte aligned.  HU
 * values outside [-4096, 4095] make their slice TSA_ERR_LEVEL_OVERFLOW (they
 * still take part in the window). */
typedef struct {
  const int16_t *volume; /* [nz][ny][nx] HU, device */
  int64_t nx, ny, nz;
  int32_t background;    /* HU of "outside the detector" (the paper: -2000); in [-4096, 4095] */
  int32_t k;             /* thresholds per slice, 1..4 */
  double q;              /* entropic index, as tsa_problem */
  int32_t objective;     /* tsa_objective */
  int32_t enumeration;   /* tsa_enumeration */
} tsa_hu_problem;

size_t tsa_hu_workspace_size(const tsa_hu_problem *p);

/* The whole path on HU input.  out: as tsa_segment with bins = 256
 * (thresholds [nz][k] in 8-bit levels, labels, objective, histogram [nz][256]
 * of g, slice_status).  window: device int32[2] = (lo, hi) or NULL. */
tsa_status tsa_hu_segment(const tsa_hu_problem *p, const tsa_outputs *out, int32_t *window,
                          void *workspace, size_t workspace_bytes, void *stream);

/* The two phases of tsa_hu_segment, for slices sharded over ranks (the
 * window is volume-wide, so ranks exchange it: an all-reduce of (min lo,
 * max hi) between the phases):
 *   tsa_hu_histogram  HU histograms of the slab into the workspace and the
 *                     slab's window -> window_out (device int32[2]; (INT_MAX,
 *                     INT_MIN) when the slab has no non-background voxel)
 *   tsa_hu_finish     8-bit histograms under window_in (device int32[2]), the
 *                     search, finalize and labels -> out (as tsa_hu_segment)
 * Same workspace for both (tsa_hu_workspace_size), left untouched between. */
tsa_status tsa_hu_histogram(const tsa_hu_problem *p, int32_t *window_out, void *workspace,
                            size_t workspace_bytes, void *stream);
tsa_status tsa_hu_finish(const tsa_hu_problem *p, const int32_t *window_in, const tsa_outputs *out,
                         void *workspace, size_t workspace_bytes, void *stream);

/* The pre-processing step alone: gray [nz][ny][nx] u8 = g(v); window as above. */
tsa_status tsa_hu_preprocess(const tsa_hu_problem *p, uint8_t *gray, int32_t *window,
                             void *workspace, size_t workspace_bytes, void *stream);

/* ---- Morphology: opening and the top-hat mask --------------------------
 * (readings DESIGN.md R26-R28)
 * Per slice, grayscale, structuring element disk(r) = {dy^2 + dx^2 <= r^2}:
 *   ERODE   out = min over the disk, samples outside the slice = 255
 *   DILATE  out = max over the disk, outside = 0
 *   OPEN    out = dilate(erode(in))                    (A o B = (A (-) B) (+) B)
 *   TOPHAT  out = max(in - open(in), 0)                (the chest mask, white top-hat)
 * in / out: [nz][ny][nx] u8, device, may not alias; nz <= 65535.  radius 0..10 (the paper:
 * 10).  OPEN and TOPHAT need tsa_morph_workspace_size() bytes (the eroded
 * volume); ERODE / DILATE need none (workspace may be NULL). */
typedef enum { TSA_MORPH_ERODE = 0, TSA_MORPH_DILATE = 1, TSA_MORPH_OPEN = 2, TSA_MORPH_TOPHAT = 3 } tsa_morph_op;

size_t tsa_morph_workspace_size(int64_t nx, int64_t ny, int64_t nz, int32_t op);

tsa_status tsa_morph(const uint8_t *in, uint8_t *out, int64_t nx, int64_t ny, int64_t nz,
                     int32_t radius, int32_t op, void *workspace, size_t workspace_bytes,
                     void *stream);

const char *tsa_status_string(tsa_status s);
const char *tsa_last_error(void);
int32_t tsa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TSA_H */
