/*
 * lpd_nystrom.h — C ABI of the B200 Nyström-factor library (liblpd_nystrom.so).
 *
 * This is the drop-in boundary for the LPD-SVM reference's factor path. Every
 * entry point below replaces a named reference interface:
 *
 *   lpd_compute_g_csr / lpd_compute_g_dense
 *       replace lpdsvm::compute_G
 *       (reference proj/include/lpdsvm/factor.hpp:50-55, proj/src/factor.cpp:83-110):
 *       G = Z(points, landmarks) · L, written row-major into a caller buffer.
 *   lpd_set_basis_csr / lpd_set_basis_dense
 *       receive the (landmarks, landmark_norms, L, params) arguments of the same
 *       call (factor.hpp:53-54). Split out so one basis (one γ) serves many row
 *       batches and devices: the reference calls compute_G once per γ
 *       (proj/src/factor.cpp:129-133, proj/src/modelsel.cpp:180-190).
 *   lpd_decision_values
 *       replaces the held-out scoring loop d[r][p] = G_r · w_p
 *       (proj/src/modelsel.cpp:123-140) and the warm-start/KKT sweeps that read
 *       G·w (proj/src/dcd.cpp:91-102, 150-172).
 *
 * Conventions: plain pointers and sizes only, no CUDA or C++ types. Matrices
 * are row-major fp64 with an explicit leading dimension in elements. Sparse
 * points use CSR with 0-based int32 column indices, the flattened form of the
 * reference's std::vector<Feature> (proj/include/lpdsvm/dataio.hpp:14-24).
 * Functions never throw; they return an LPD_* status and leave a message
 * retrievable with lpd_last_error() (thread-local).
 *
 * Threading: a context is used by one host thread at a time (the reference calls
 * compute_G from a single thread, factor.cpp:131-132; the library runs its own
 * host threads per device and per delivery inside each call). Calls on different
 * contexts may run concurrently; the *_device entry points enqueue on the
 * caller's stream, and two such calls must not run concurrently on different
 * streams of the same device (the large-d GEMMs rendezvous across their CTAs).
 */
#ifndef LPD_NYSTROM_H
#define LPD_NYSTROM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPD_OK 0
#define LPD_ERR_INVALID_ARGUMENT 1 /* reference: std::invalid_argument (factor.cpp:87,91; kernel.cpp:10-15) */
#define LPD_ERR_CUDA 2             /* device / driver failure: std::runtime_error */
#define LPD_ERR_UNSUPPORTED 3      /* valid input outside this build's kernel envelope */
#define LPD_ERR_OUT_OF_MEMORY 4
#define LPD_ERR_NO_DEVICE 5

/* Fault-injection sites (lpd_inject_fault; tests) */
#define LPD_FAULT_NONE 0
#define LPD_FAULT_ALLOC 1  /* a device allocation fails: LPD_ERR_OUT_OF_MEMORY */
#define LPD_FAULT_LAUNCH 2 /* a factor-kernel launch fails: LPD_ERR_CUDA */
#define LPD_FAULT_D2H 3    /* a device-to-host transfer of G fails: LPD_ERR_CUDA */

#define LPD_OUT_F64 0
#define LPD_OUT_F32 1

#define LPD_PRECISION_AUTO 0 /* per basis: high when the fast path's error estimate > 5e-5 */
#define LPD_PRECISION_FAST 1 /* tensor-core split-fp16 path (K1 / panel path) */
#define LPD_PRECISION_HIGH 2 /* fp64 Z (direct distance) + fp64 DMMA projection */

typedef struct lpd_context lpd_context;

/* One stored feature of a sparse point: the layout of the reference's lpdsvm::Feature
 * {int32 index (0-based); double value} (proj/include/lpdsvm/dataio.hpp:14-19), so a
 * std::vector<Feature>'s storage is an array of these. */
typedef struct lpd_feature {
    int32_t index;
    double value;
} lpd_feature;

/* Per-call phase timings (seconds, host wall clock unless noted). */
typedef struct lpd_timings {
    double total_seconds;     /* whole call */
    double h2d_seconds;       /* sum over devices of host->device copy time (events) */
    double kernel_seconds;    /* sum over devices of prep + factor kernel time (events) */
    double d2h_seconds;       /* sum over devices of device->host copy time (events) */
    double host_copy_seconds; /* pinned staging -> caller buffer memcpy time (wall) */
    int64_t rows;             /* rows computed */
    int64_t launches;         /* kernel launches issued */
    int32_t devices;          /* devices used */
    int32_t reserved;
} lpd_timings;

const char* lpd_last_error(void);
/* Test hook (the reference has no fault injection): the `after`-th next pass
 * through `site` (process-wide, once) fails the way the real CUDA failure would; the call
 * returns the error, in-flight work of the call is drained, and the context stays usable.
 * site = LPD_FAULT_NONE disarms. Also armed by LPD_FAULT_INJECT=<alloc|launch|d2h>:<after>
 * at context creation. */
int lpd_inject_fault(int site, int after);
int lpd_version(void);
/* Number of visible CUDA devices (0 on a machine without a GPU; never fails). */
int lpd_device_count(void);

/* num_devices <= 0: use LPD_NUM_GPUS from the environment if set, else all visible. */
int lpd_context_create(lpd_context** out, int num_devices);
/* Explicit device ordinals (one process per GPU: pass the local rank's device). */
int lpd_context_create_devices(lpd_context** out, const int* device_ids, int count);
int lpd_context_destroy(lpd_context* ctx);
int lpd_context_num_devices(const lpd_context* ctx);

/* Basis: B landmarks with d features, L (B x b_eff, row-major, ld = b_eff), gamma > 0.
 * Replicated to every device of the context. Landmark norms are recomputed on the
 * device from the same values the tensor cores see (the caller's fp64 norms are
 * not needed). */
int lpd_set_basis_dense(lpd_context* ctx, const double* landmarks, int64_t B, int64_t d,
                        int64_t ld, const double* L, int64_t b_eff, double gamma);
int lpd_set_basis_csr(lpd_context* ctx, int64_t B, int64_t d, const int64_t* indptr,
                      const int32_t* indices, const double* values, const double* L,
                      int64_t b_eff, double gamma);

/* Basis from device-resident fp64 landmarks (B x d, ld) and L (B x b_eff) on device
 * `device_index`. stream: cudaStream_t as void* (NULL = library stream, synchronised).
 * Shapes unchanged from the previous basis reuse the device buffers (no allocation). */
int lpd_set_basis_device(lpd_context* ctx, int device_index, const double* landmarks_dev,
                         int64_t B, int64_t d, int64_t ld, const double* L_dev, int64_t b_eff,
                         double gamma, void* stream);

/* Precision of the factor path (default LPD_PRECISION_AUTO, or the LPD_PRECISION environment
 * variable: auto | fast | high). The fast path holds G within ~2x its estimate
 * 2^-22*sqrt(lambda_max)*||L||_F/sqrt(B) of the fp64 reference (row-normwise; the lambda_j are
 * read off L's column norms 1/sqrt(lambda_j)); the high path computes Z in fp64 by direct distance and
 * G = Z*L on the fp64 tensor cores, for the ill-conditioned bases of small gamma with the
 * reference default tau = 1e-12 (proj/include/lpdsvm/factor.hpp:59). Applies from the next
 * lpd_set_basis_* call. */
int lpd_set_precision(lpd_context* ctx, int mode);
/* The current basis' choice: *high = 1 on the high-precision path; *estimate = the fast
 * path's row-error estimate 2^-22*sqrt(lambda_max)*||L||_F/sqrt(B) from L's column norms. */
int lpd_basis_precision(const lpd_context* ctx, int* high, double* estimate);

/* G (n x b_eff, leading dimension ldg >= b_eff) for host rows; rows are sharded
 * across the context's devices, results streamed back into G. */
int lpd_compute_g_dense(lpd_context* ctx, const double* X, int64_t n, int64_t d, int64_t ldx,
                        double* G, int64_t ldg, lpd_timings* timings);
int lpd_compute_g_csr(lpd_context* ctx, int64_t n, int64_t d, const int64_t* indptr,
                      const int32_t* indices, const double* values, double* G, int64_t ldg,
                      lpd_timings* timings);

/* The same for rows in the reference's own storage (no intermediate CSR): rows[i] points at
 * nnz[i] features of point i (a std::vector<Feature>'s data(), strictly ascending indices,
 * dataio.hpp:20-24), indices in [0, d). Chunks are densified by the library's host threads
 * into pinned memory and copied up while earlier chunks compute and deliver. */
int lpd_compute_g_rows(lpd_context* ctx, int64_t n, int64_t d, const lpd_feature* const* rows,
                       const int64_t* nnz, double* G, int64_t ldg, lpd_timings* timings);

/* Device-resident variant: X_dev (n x d fp64, ld ldx) and G_dev on device
 * `device_index` of the context; out_dtype LPD_OUT_F64 or LPD_OUT_F32; stream is a
 * cudaStream_t passed as void* (NULL = the library's stream, synchronised before
 * return). scratch may be NULL (library allocates) . */
int lpd_compute_g_device(lpd_context* ctx, int device_index, const double* X_dev, int64_t n,
                         int64_t ldx, void* G_dev, int64_t ldg, int out_dtype, void* stream);

/* Decision values D (n x P, ld = ldd) = G (n x b_eff, ld = ldg) · Wᵀ, W (P x b_eff, ld = b_eff).
 * All pointers are device pointers on device_index; g_dtype LPD_OUT_F64/F32. fp64
 * accumulation. */
int lpd_decision_values_device(lpd_context* ctx, int device_index, const void* G_dev,
                               int g_dtype, int64_t n, int64_t b_eff, int64_t ldg,
                               const double* W_dev, int64_t P, double* D_dev, int64_t ldd,
                               void* stream);

/* Host variant of the above (copies in/out). */
int lpd_decision_values(lpd_context* ctx, const double* G, int64_t n, int64_t b_eff, int64_t ldg,
                        const double* W, int64_t P, double* D, int64_t ldd);

/* One-vs-one prediction (K5): the basis must have been set with L := betasᵀ
 * (B x P, P = num_classes*(num_classes-1)/2, the reference's OvoModel::betas
 * transposed, proj/include/lpdsvm/multiclass.hpp:57-68). Computes the decision values
 * Z(x, landmarks)·betasᵀ on the device and the majority vote
 * (proj/src/multiclass.cpp:153-168); classes[i] receives the winning class INDEX
 * (into the model's LabelMap) for row i. Replaces lpdsvm::ovo_predict
 * (multiclass.cpp:170-200). num_classes <= 2048. */
int lpd_predict_ovo_dense(lpd_context* ctx, const double* X, int64_t n, int64_t d, int64_t ldx,
                          int64_t num_classes, int32_t* classes);
int lpd_predict_ovo_csr(lpd_context* ctx, int64_t n, int64_t d, const int64_t* indptr,
                        const int32_t* indices, const double* values, int64_t num_classes,
                        int32_t* classes);

/* Per-point decision values of a trained one-vs-one model (K8): replaces
 * lpdsvm::decision_values (proj/include/lpdsvm/multiclass.hpp:84-86,
 * proj/src/multiclass.cpp:137-151), which Python Model.decision_values calls once per
 * point (proj/bindings/module.cpp:157-171). The model is set once: B landmarks with d
 * features (dense ld, or CSR), betas (P x B row-major, the OvoModel::betas of
 * multiclass.hpp:63), gamma. Then D[i][p] = sum_j exp(-gamma*||x_i - b_j||^2)*betas[p][j]
 * for n points (D row-major, ld = ldd >= P), in fp64 with the reference's operation
 * order (direct squared distance in ascending feature order, products rounded then
 * added, exp, then the dot with betas in ascending j): equal to the reference up to the
 * last ulp of exp. Points may have a different feature width d than the landmarks
 * (missing features are zeros, as in the sparse merge of squared_distance,
 * dataio.cpp:38-58); CSR indices outside [0, d) are LPD_ERR_INVALID_ARGUMENT. Runs on
 * the context's first device. */
int lpd_set_model_dense(lpd_context* ctx, const double* landmarks, int64_t B, int64_t d, int64_t ld,
                        const double* betas, int64_t P, double gamma);
int lpd_set_model_csr(lpd_context* ctx, int64_t B, int64_t d, const int64_t* indptr,
                      const int32_t* indices, const double* values, const double* betas, int64_t P,
                      double gamma);
int lpd_model_decision_values_dense(lpd_context* ctx, const double* X, int64_t n, int64_t d,
                                    int64_t ldx, double* D, int64_t ldd);
int lpd_model_decision_values_csr(lpd_context* ctx, int64_t n, int64_t d, const int64_t* indptr,
                                  const int32_t* indices, const double* values, double* D,
                                  int64_t ldd);

/* The one-vs-one vote on given decision values (D: n x P host, row-major, ld = ldd,
 * P = num_classes*(num_classes-1)/2): classes[i] = the winning class INDEX, with the
 * reference's rule (proj/src/multiclass.cpp:153-168: a strictly positive decision votes
 * for the pair's first class, anything else for the second; most votes wins, ties to
 * the smaller index). The same device kernel ovo_predict's K5 path ends with. */
int lpd_ovo_vote(lpd_context* ctx, const double* D, int64_t n, int64_t ldd, int64_t num_classes,
                 int32_t* classes);

/* Kernel block K[i][j] = exp(-gamma * max(0, norms_a[i] + norms_b[j] - 2<a_i, b_j>)) in fp64
 * with the reference's operation order (K7; replaces lpdsvm::kernel_block,
 * proj/include/lpdsvm/kernel.hpp:26-32, proj/src/kernel.cpp:31-57, whose main caller is
 * the landmark Gram matrix of build_factor_with_landmarks, factor.cpp:121-126). Rows are
 * CSR; pass a_indptr / b_indptr = NULL to give dense row-major fp64 rows (ld = d) in
 * a_values / b_values. out is m x n row-major (ld = ldo), host memory. Runs on the
 * context's first device. */
int lpd_kernel_block(lpd_context* ctx, int64_t m, const int64_t* a_indptr, const int32_t* a_indices,
                     const double* a_values, const double* norms_a, int64_t n,
                     const int64_t* b_indptr, const int32_t* b_indices, const double* b_values,
                     const double* norms_b, int64_t d, double gamma, double* out, int64_t ldo);

/* Resident G (config 5, solver sweeps). With keep_resident on, lpd_compute_g_* also
 * leaves the fp32 G (bit-identical to the fp64 G it returns) on the devices, row-sharded
 * like the computation, until the next call; lpd_resident_shape reports n = 0 when the
 * last call could not keep it (HBM short). */
int lpd_set_keep_resident(lpd_context* ctx, int enable);
int lpd_resident_shape(const lpd_context* ctx, int64_t* n, int64_t* b_eff);
/* D[i][p] = sum_j G[rows[i]][j] * W[p][j] (W is P x b_eff, D is count x P), each sum in
 * ascending j with every product rounded then added — the reference's scoring loop
 * (proj/src/modelsel.cpp:129-136) bit for bit: the held-out scoring of cross-validation
 * (modelsel.cpp:123-140) and the gradients 1 - y_i G_i.w of reactivation_pass
 * (proj/src/dcd.cpp:150-172). */
int lpd_resident_gw(lpd_context* ctx, const int32_t* rows, int64_t count, const double* W,
                    int64_t P, double* D);
/* The same D for the P = num_classes*(num_classes-1)/2 pair vectors of a one-vs-one model
 * (W in the reference's pair order, multiclass.cpp:24-32), then the reference's vote
 * (multiclass.cpp:153-168) on the device: classes[i] = the winning class index of listed
 * row i. cross_validate's held-out scoring (modelsel.cpp:123-140) without shipping D. */
int lpd_resident_vote(lpd_context* ctx, const int32_t* rows, int64_t count, const double* W,
                      int64_t num_classes, int32_t* classes);
/* w[j] = sum_i coef[i] * G[rows[i]][j] (fp64, deterministic order): rebuild_w of the
 * warm starts (proj/src/dcd.cpp:91-102). */
int lpd_resident_gtv(lpd_context* ctx, const int32_t* rows, const double* coef, int64_t count,
                     double* w);
/* W[s][j] = sum_i coef[i][s] * G[rows[i]][j] for `sets` coefficient vectors at once (coef is
 * count x sets row-major, W is sets x b_eff): one read of the listed rows serves every set.
 * The warm starts of every (fold, pair) problem of cross_validate at a new C
 * (proj/src/modelsel.cpp:104-112 -> dcd.cpp:91-102, 115-121) in one pass. */
int lpd_resident_gtv_sets(lpd_context* ctx, const int32_t* rows, const double* coef, int64_t count,
                          int64_t sets, double* W);
/* q[i] = sum_j G[i][j]^2 for every row of the resident G (n values), fp64 in ascending j with
 * each product rounded then added: make_binary_problem's q_diag (proj/src/dcd.cpp:60-89,
 * row.squaredNorm()), bit-identical to a sequential host pass over the returned fp64 G. */
int lpd_resident_row_sqnorms(lpd_context* ctx, double* q);

/* Last kernel timing of the fused factor kernel on device_index (milliseconds,
 * CUDA events around the launch on its stream), for benchmarks. */
double lpd_last_factor_kernel_ms(const lpd_context* ctx, int device_index);

/* Sum of the fused factor kernel's durations (CUDA events recorded on its launch
 * stream around every device-path launch, up to 512 since the last reset) and the
 * launch count. Synchronises on the recorded events. reset != 0 clears the record. */
int lpd_factor_kernel_stats(lpd_context* ctx, int device_index, double* total_ms,
                            int64_t* launches, int reset);

#ifdef __cplusplus
}
#endif

#endif /* LPD_NYSTROM_H */
