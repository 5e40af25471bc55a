/*
 * esom.h -- C ABI of libesom.so, the sm_100a EmbedSOM hot path.
 *
 * Each entry point replaces one reference function of `embedview`
 * (/root/reference/pkg/src/embedview).  The reference has no FFI of its own
 * (it is Python + numba); the binding a maintainer adds is a ctypes stub,
 * shown in INTEGRATION.md and implemented in
 * paper_2201_00701_b200/_lib.py.
 *
 * Conventions
 *  - All pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    row-major, C-contiguous: points n×d f32, landmarks g×d f32, layout g×2
 *    f32, neighbour lists n×k (int32 indices, f32 squared distances).
 *  - Calls are asynchronous on `stream` and never allocate: scratch comes
 *    from a caller-owned workspace sized by the *_workspace_bytes helpers.
 *  - Return 0 on success, else ESOM_ERR_*; esom_last_error() (thread-local)
 *    holds the message.  PARAM maps to ParameterError, INPUT to InputError.
 *  - Non-finite inputs raise a device flag (*nonfinite_flag |= 1) instead
 *    of the reference's host-side np.isfinite pass (ref: knn.py:196-197);
 *    the host wrapper turns it into InputError("non-finite input").
 */
#ifndef ESOM_H
#define ESOM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESOM_ABI_VERSION 1
#define ESOM_OK 0
#define ESOM_ERR_PARAM 1
#define ESOM_ERR_INPUT 2
#define ESOM_ERR_CUDA 3
#define ESOM_ERR_UNSUPPORTED 4

typedef struct CUstream_st *esom_stream_t; /* == cudaStream_t */
#ifndef __CUDACC__
typedef esom_stream_t cudaStream_t;
#endif

int esom_version(void);
const char *esom_last_error(void);

/* Diagnostic: when non-NULL, the tensor-core screens atomically add the
 * number of candidates they re-evaluate exactly to *counter (device int32). */
void esom_set_tc_stats(int32_t *counter);

/* Diagnostic kernel timing: esom_timing_begin(1) clears and starts recording
 * CUDA events on the launching stream around the hot kernels (knn_tc2_kernel,
 * knn_gemm_kernel, knn_exact_group_kernel, project_kernel);
 * esom_timing_query(name, &launches) synchronizes and returns their summed
 * milliseconds.  esom_timing_begin(0) stops recording. */
void esom_timing_begin(int32_t on);
/* Number of kernels libesom has launched so far (process-wide counter). */
int64_t esom_launch_count(void);
double esom_timing_query(const char *name, int32_t *launches);

/* Bytes of scratch for esom_knn / esom_bmu_accumulate (with_pairs = 0) or
 * for a prepared model (with_pairs = 1: packed landmark tiles + the packed
 * upper-triangular pair table). */
size_t esom_workspace_bytes(int32_t g, int32_t d, int32_t k, int32_t with_pairs);

/* Exact k nearest landmarks per point, rows ascending by (sqdist, index).
 * Replaces knn_base / knn_bitonic / knn (ref: knn.py:201-243; the two
 * reference backends are bit-identical, so is this).  1 <= k <= g. */
int esom_knn(const float *X, int64_t n, int32_t d, const float *L, int32_t g, int32_t k,
             int32_t *idx, float *sqd, int32_t *nonfinite_flag,
             void *workspace, size_t ws_bytes, cudaStream_t stream);

/* Score rows n×k f64 from ascending squared distances.
 * Replaces _score_rows / scores (ref: projection.py:38-65, 124-142). */
int esom_scores(const float *sqd, int64_t n, int32_t k, double *out, cudaStream_t stream);

/* Faithful projection of precomputed neighbour rows and scores, the mixed
 * f32/f64 contract of _project_rows (ref: projection.py:68-121); used by
 * project_point / project_neighbors (ref: projection.py:189-217). */
int esom_project(const float *X, int64_t n, int32_t d, const float *hi, const float *lo,
                 int32_t g, const int32_t *idx, const double *scores, int32_t k, float *xy,
                 cudaStream_t stream);

/* Per-model preparation of esom_embed_prepared: landmark tiles, tensor-core
 * operands (rows ordered along the Morton curve of the layout lo, which
 * keeps the screen's k-th-distance bound tight for trained SOMs; lo may be
 * NULL = index order), the g×g pair table (0.5/hd2) and f64 rows.  Re-run
 * whenever hi or lo changes. */
#define ESOM_PREPARE_KEEP_ORDER 1  /* lo unchanged since the last preparation of this workspace */
int esom_prepare_model(const float *hi, const float *lo, int32_t g, int32_t d, int32_t k, int32_t flags,
                       void *workspace, size_t ws_bytes, int32_t *nonfinite_flag, cudaStream_t stream);

/* Per-call scratch of esom_embed_prepared for n points: the neighbour rows
 * of one L2-resident chunk of points (scan -> projection). */
size_t esom_point_workspace_bytes(int64_t n, int32_t d, int32_t k);

/* Embed on a prepared model: exact k-NN + scores + projection -> xy (n×2
 * f32).  Per chunk of points: the k-NN (d <= 32: tensor-core screen, BMU
 * sort, exact re-evaluation; d > 32: operand split, GEMM screen, BMU sort,
 * exact re-evaluation) and the projection kernel -- esom_embed_launches()
 * counts them.  Replaces embed (ref: projection.py:220-245).  Optional
 * outputs (NULL to skip): bmu (n int32 = idx[:,0]); batch-SOM statistics in
 * exact int64 fixed point -- acc_S (g×d: += round(x_i 2^acc_fx_bits) per
 * BMU) and acc_C (g: += 1) -- so they are independent of accumulation order
 * and of the split of points over ranks; qe_sum (f64 += nearest squared
 * distance, ref: som.py:71-79).  k <= 64, 0 <= acc_fx_bits <= 60. */
int esom_embed_prepared(const float *X, int64_t n, int32_t d, const float *hi, const float *lo,
                        int32_t g, int32_t k, const void *model_ws, void *point_ws,
                        size_t point_ws_bytes, float *xy, int32_t *bmu, int64_t *acc_S,
                        int64_t *acc_C, int32_t acc_fx_bits, double *qe_sum, int32_t *nonfinite_flag,
                        cudaStream_t stream);

/* esom_embed_prepared with options.  flags: ESOM_EMBED_BMU_ORDER = visit
 * points grouped by nearest landmark in the projection (neighbour rows and
 * pair-table entries shared across a warp; pays a BMU counting sort -- worth
 * it when most points are far from tightly packed landmarks, e.g. a trained
 * SOM).  far_count (nullable, device int32): += points that took the f64
 * far-point distance path -- the caller's signal for the next frame's flag. */
#define ESOM_EMBED_BMU_ORDER 1
int esom_embed_prepared_ex(const float *X, int64_t n, int32_t d, const float *hi, const float *lo,
                           int32_t g, int32_t k, const void *model_ws, void *point_ws,
                           size_t point_ws_bytes, float *xy, int32_t *bmu, int64_t *acc_S,
                           int64_t *acc_C, int32_t acc_fx_bits, double *qe_sum, int32_t *nonfinite_flag,
                           int32_t flags, int32_t *far_count, cudaStream_t stream);

/* Number of kernels one esom_embed_prepared(n, ...) call launches (evidence
 * for the benchmark's launch count). */
int32_t esom_embed_launches(int64_t n, int32_t g, int32_t d, int32_t k);

/* esom_prepare_model + esom_embed_prepared in one workspace of
 * esom_embed_workspace_bytes(n, g, d, k) bytes. */
size_t esom_embed_workspace_bytes(int64_t n, int32_t g, int32_t d, int32_t k);
int esom_embed(const float *X, int64_t n, int32_t d, const float *hi, const float *lo, int32_t g,
               int32_t k, void *workspace, size_t ws_bytes, float *xy, int32_t *bmu,
               int64_t *acc_S, int64_t *acc_C, int32_t acc_fx_bits, double *qe_sum,
               int32_t *nonfinite_flag, cudaStream_t stream);

/* Batch-SOM statistics only (BMU pass, no projection): acc_S/acc_C/qe_sum
 * as in esom_embed_prepared; bmu optional.  Workspace from esom_workspace_bytes(.., 0). */
int esom_bmu_accumulate(const float *X, int64_t n, int32_t d, const float *hi, int32_t g,
                        void *workspace, size_t ws_bytes, int32_t *bmu, int64_t *acc_S,
                        int64_t *acc_C, int32_t acc_fx_bits, double *qe_sum, int32_t *nonfinite_flag,
                        cudaStream_t stream);

/* Online trainers: the sample indices are drawn on the host from the
 * caller's Rng (ref: som.py:57, graphmodel.py:96) and applied in order.
 * hi_inout g×d f32 is updated in place.  Workspace: esom_tick_workspace_bytes. */
size_t esom_tick_workspace_bytes(int32_t g, int32_t d);
int esom_som_tick(const float *X, int32_t d, const int64_t *sample_idx, int32_t B,
                  float *hi_inout, const float *lo, int32_t g, double sigma, double alpha,
                  void *workspace, size_t ws_bytes, cudaStream_t stream);   /* ref: som.py:44-68 */
int esom_kmeans_tick(const float *X, int32_t d, const int64_t *sample_idx, int32_t B,
                     float *hi_inout, int32_t g, double alpha_km, void *workspace,
                     size_t ws_bytes, cudaStream_t stream);                 /* ref: graphmodel.py:87-102 */

/* Batch-SOM landmark update from (all-reduced) int64 fixed-point statistics
 * (S = acc_S 2^-acc_fx_bits, C = acc_C).  NEW -- no reference function
 * (SURVEY.md §8a T3).  mode 0 mean-field hi_j += (alpha/B)(num_j - den_j
 * hi_j); mode 1 Kohonen hi_j = num_j/den_j.  Deterministic: a fixed
 * reduction order per landmark. */
int esom_batch_som_update(const int64_t *acc_S, const int64_t *acc_C, int32_t acc_fx_bits,
                          const float *lo, int32_t g, int32_t d, double sigma, double alpha,
                          int32_t mode, float *hi_inout, cudaStream_t stream);

/* Page-lock / release a caller-owned host range in place (cudaHostRegister):
 * repeated host inputs then DMA straight from the caller's buffer.  Errors
 * are returned (and cleared), never left pending. */
int esom_host_register(void *p, size_t bytes);
int esom_host_unregister(void *p);

/* ---- data formats either side of the path ---- */

/* Frame colours: rint((X[:, color_dim] - lo) / span * 255) as u8, 128 when
 * span <= 0 (lo, span = the column's min and max - min).  Replaces
 * color_channel (ref: engine.py:144-153); bit-exact. */
int esom_color_channel(const float *X, int64_t n, int32_t d, int32_t color_dim, double lo, double span,
                       uint8_t *out, cudaStream_t stream);

/* FramePoints wire record, the bytes protocol.encode(FramePoints(frame_id,
 * xy, colors)) returns (ref: protocol.py:205-210, 216-218): u32 length, tag
 * 0x31, u32 frame_id, u32 n, n×2 f32, n u8 -- esom_frame_points_bytes(n) =
 * 13 + 9n bytes.  `out` (16-byte aligned) may be device memory or mapped
 * pinned host memory (written over PCIe by the kernel: zero-copy send). */
size_t esom_frame_points_bytes(int64_t n);
/* Device-side address of a page-locked host buffer (cudaHostGetDevicePointer),
 * NULL if the buffer is not mapped. */
void *esom_mapped_device_ptr(void *host_ptr);
int esom_frame_points_pack(const float *xy, const uint8_t *colors, int64_t n, uint32_t frame_id,
                           uint8_t *out, cudaStream_t stream);

/* FCS DATA segment -> f32 (ref: io.py:113-126; $BYTEORD "4,3,2,1" =
 * big_endian 1, "1,2,3,4" = 0), with the finiteness check of
 * Dataset.from_points (ref: core.py:38-40).  raw/out 16-byte aligned
 * (raw = the DATA bytes copied into device staging); count = n*d values. */
int esom_fcs_decode(const void *raw, int64_t count, int32_t big_endian, float *out,
                    int32_t *nonfinite_flag, cudaStream_t stream);

/* Per-dimension f64 min, max, mean and population sd of X (ref: core.py:57-69
 * compute_dim_stats).  Deterministic blocked sums (not numpy's sequential
 * order: mean/sd agree to ~1e-15 relative; min/max exactly). */
size_t esom_dim_stats_workspace_bytes(int64_t n, int32_t d);
int esom_dim_stats(const float *X, int64_t n, int32_t d, double *mn, double *mx, double *mean,
                   double *sd, void *workspace, size_t ws_bytes, cudaStream_t stream);

/* Per-dimension transform (ref: io.py:200-225 apply_transform): kind[c] 0
 * none, 1 minmax, 2 zscore, 3 affine (a[c] * x + b[c]); f64 arithmetic op
 * for op like numpy, rounded to f32.  All arrays device, length d. */
int esom_apply_transform(const float *X, int64_t n, int32_t d, const int32_t *kind, const double *a,
                         const double *b, const double *mn, const double *mx, const double *mean,
                         const double *sd, float *out, int32_t *nonfinite_flag, cudaStream_t stream);

/* Landmark-side graph ops, f64.
 * One force-layout step (ref: graphmodel.py:138-192 net_forces + layout_tick):
 * lo g×2 f32, edges pairs e×2 int32 (i < j) with rest lengths, and a CSR of
 * signed edge ids per landmark (csr_ptr g+1, csr_edge: e for the first
 * endpoint, -e-1 for the second, in edge order); pinned g u8 or NULL.
 * vel_inout g×2 f64 is updated; lo_out g×2 f32; forces_or_null g×2 f64. */
int esom_layout_tick(const float *lo, int32_t g, const int32_t *pairs, const float *rest,
                     const int32_t *csr_ptr, const int32_t *csr_edge, const uint8_t *pinned,
                     double stiffness, double repulsion, double eps, double damping, double dt,
                     double *vel_inout, float *lo_out, double *forces_or_null, cudaStream_t stream);

/* hi row for a landmark added at layout position (px, py): inverse-distance
 * weights over the layout (ref: som.py:82-101); out d f32. */
int esom_fit_hi(const float *hi, const float *lo, int32_t g, int32_t d, double px, double py, double eps,
                float *out, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ESOM_H */
