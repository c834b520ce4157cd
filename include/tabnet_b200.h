/*
 * tabnet_b200.h — C ABI of libtabnet_b200.so, the B200 (sm_100a) engine for
 * TabNet batch predict + feature-mask explain.
 *
 * This is the drop-in boundary for the reference's hot path
 *   /root/reference/pkg/src/tabserve/model/network.py:195-267  TabNetModel.apply
 *   /root/reference/pkg/src/tabserve/model/network.py:269-281  TabNetModel.forward
 *   /root/reference/pkg/src/tabserve/model/sparsemax.py:13-41  sparsemax
 *   /root/reference/pkg/src/tabserve/model/io.py:22-36         crc32c (.tbnt trailer)
 * The reference is pure Python/NumPy and has no FFI of its own; these entry
 * points are what a ctypes binding inside tabserve.model would call
 * (INTEGRATION.md shows that stub).  No torch types cross this boundary: plain
 * pointers, sizes and an opaque cudaStream_t passed as void*.
 *
 * Error convention (errors.py:4-41): every call returns a tbn_status; the
 * Python shim maps TBN_ERR_INVALID_INPUT -> InvalidInputError,
 * TBN_ERR_CONFIG -> ConfigurationError, TBN_ERR_CUDA/UNSUPPORTED -> DeviceError.
 * tbn_last_error() gives the thread-local message of the last failure.
 */
#ifndef TABNET_B200_H
#define TABNET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TBN_ABI_VERSION 2

typedef enum {
  TBN_OK = 0,
  TBN_ERR_INVALID_INPUT = 1, /* width mismatch, non-finite feature, rows < 1   (network.py:207-211) */
  TBN_ERR_CONFIG = 2,        /* inconsistent config / params                   (config.py:29-41, network.py:110-114) */
  TBN_ERR_CUDA = 3,          /* CUDA runtime failure or no device                                         */
  TBN_ERR_UNSUPPORTED = 4,   /* shape outside the compiled kernel instances                               */
  /* .tbnt stream errors, the ModelFormatError family of io.py:60-112 / errors.py:20-33 */
  TBN_ERR_FORMAT = 5,        /* ModelFormatError: bad magic, trailing bytes, metadata, size mismatch   */
  TBN_ERR_FORMAT_VERSION = 6,/* FormatVersionError: version != 1                                       */
  TBN_ERR_TRUNCATED = 7,     /* TruncatedStreamError: stream ends inside the header or a section        */
  TBN_ERR_CHECKSUM = 8       /* ChecksumError: CRC-32C trailer mismatch                                  */
} tbn_status;

/* Arithmetic of the FC contractions.  Everything else (GLU, sparsemax, prior,
 * aggregation, softmax) is fp32 on CUDA cores in every mode. */
typedef enum {
  TBN_PREC_TF32X3 = 0, /* tcgen05 kind::tf32, hi/lo split, 3 MMAs: fp32-faithful (parity mode, default) */
  TBN_PREC_TF32 = 1,   /* tcgen05 kind::tf32, 1 MMA                                                   */
  TBN_PREC_BF16 = 2,   /* tcgen05 kind::f16 (bf16 operands), 1 MMA                                    */
  TBN_PREC_FP32 = 3    /* CUDA-core fp32 FFMA kernel (no tensor cores; reference-precision check)     */
} tbn_precision;

/* tbn_config.flags.  TBN_CFG_REGRESSION: identity head, n_classes must be 1.
 * An extension: the reference only has the
 * softmax classifier (config.py:32-33 enforces n_classes >= 2).  The output
 * is logits (rows, 1) = d_sum @ head_W + head_b; probabilities (if requested)
 * receive the same value and predicted_class is 0.  Its oracle is column 0 of
 * the reference logits of a 2-class model sharing head_W[:, 0] / head_b[0]. */
#define TBN_CFG_REGRESSION 1

/* apply() flags (network.py:195-196) */
#define TBN_FLAG_NORMALIZED 1u      /* input is already normalized: skip the frozen affine        */
#define TBN_FLAG_BATCH_STATS 2u     /* negative control: normalize with this batch's mean/var     */
/* Launch geometry (no effect on any output bit): by default a batch is spread
 * over every SM (one partial row tile each: the shortest latency for a small
 * batch).  PACKED gives each CTA full row tiles on as few SMs as the batch
 * needs, so several batches in flight on different streams share the GPU
 * (the steady-state serving shape: e.g. 8 x 8,192-row batches per B200). */
#define TBN_FLAG_PACKED 4u

typedef struct {
  int32_t feature_count; /* F            (config.py:20)  */
  int32_t n_classes;     /* C >= 2       (config.py:21)  */
  int32_t n_d;           /* decision width               */
  int32_t n_a;           /* attention width              */
  int32_t n_steps;       /* S                            */
  int32_t flags;         /* TBN_CFG_* (0 = the reference's classifier)          */
  double gamma;          /* prior relaxation (config.py:26) */
} tbn_config;

/* Output views; any pointer may be NULL to skip that output.
 *   logits, probabilities : (rows, C) row-major float32
 *   masks                 : (S, rows, F) step-major float32  (network.py:231)
 *   importance            : (rows, F) float32
 *   predicted_class       : (rows,) int32, argmax with lowest-index ties */
typedef struct {
  float* logits;
  float* probabilities;
  float* masks;
  float* importance;
  int32_t* predicted_class;
} tbn_outputs;

typedef struct {
  double* logits;
  double* probabilities;
  double* masks;
  double* importance;
  int32_t* predicted_class;
} tbn_outputs_f64;

typedef struct tbn_model tbn_model;

/* Library identity. */
int32_t tbn_abi_version(void);
const char* tbn_last_error(void);                   /* thread-local, never NULL */
int32_t tbn_device_count(void);                     /* 0 when no CUDA device is usable */
/* Create the device's primary CUDA context now (a server's warm-up; the
 * cold-start split of tools/cold_start.py).  Optional: every call creates it
 * on first use. */
tbn_status tbn_device_init(int32_t device);

/* Build a device-resident model from the reference's params dict
 * (network.py:71-97 names and shapes, row-major float64, used as x @ W) and
 * frozen normalization stats (network.py:104-107).  n_params entries of
 * (names[i], values[i], sizes[i] = element count).  Packs weights once for the
 * chosen precision (K0) and uploads them to `device`. */
tbn_status tbn_model_create(const tbn_config* cfg, const char* const* names,
                            const double* const* values, const int64_t* sizes,
                            int32_t n_params, const double* norm_mean,
                            const double* norm_var, int32_t precision,
                            int32_t device, tbn_model** out);
void tbn_model_destroy(tbn_model* model);
tbn_status tbn_model_info(const tbn_model* model, tbn_config* cfg,
                          int32_t* precision, int32_t* device);

/* Device workspace needed by tbn_forward for `rows` rows (>= 256 bytes). */
size_t tbn_workspace_bytes(const tbn_model* model, int64_t rows, uint32_t flags);

/* TabNetModel.apply (network.py:195-267) on device: normalize, S+1 feature
 * transformers, S attentive steps with sparsemax, head/softmax, importance.
 * Async forward on `stream` (a cudaStream_t; NULL = legacy default stream).
 * x: device float32 (rows, F) row-major.  Outputs are device pointers.
 * A non-finite input sets *err_flag (int32, may be NULL) to 1 with a plain
 * store; the caller zeroes it before and checks it after synchronizing
 * (tbn_forward_host does).  It may point to device memory or to device-mapped
 * page-locked host memory.
 * Per-row results are bitwise independent of `rows`, tile position, grid size
 * and concurrency (invariance.py:56-82). */
tbn_status tbn_forward(const tbn_model* model, const float* x, int64_t rows,
                       uint32_t flags, const tbn_outputs* out, int32_t* err_flag,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Synchronous host-buffer forward (the reference-facing call, replacing the
 * body of TabNetModel.apply network.py:195-267 incl. its validation :204-211): stages x
 * through pinned memory on a per-thread stream, runs tbn_forward, copies the
 * outputs back, and returns TBN_ERR_INVALID_INPUT on non-finite input.
 * Reentrant: safe from many host threads at once. */
tbn_status tbn_forward_host(const tbn_model* model, const float* x, int64_t rows,
                            uint32_t flags, const tbn_outputs* out);
/* Same with the reference's float64 arrays on both sides (numpy apply path). */
tbn_status tbn_forward_host_f64(const tbn_model* model, const double* x, int64_t rows,
                                uint32_t flags, const tbn_outputs_f64* out);

/* Row-wise sparsemax on device (sparsemax.py:13-41): z, out (rows, n) fp32. */
tbn_status tbn_sparsemax(const float* z, int64_t rows, int32_t n, float* out,
                         void* stream);
/* Host-buffer sparsemax: float64 in/out, computed on device in float64, any
 * width (the reference helper's precision, sparsemax.py:13-41). */
tbn_status tbn_sparsemax_host_f64(const double* z, int64_t rows, int32_t n, double* out);

/* Per-partition column means on device: values (partitions*rows_per_partition,
 * width) fp32, out (partitions, width) float64 (fixed-order fp64 sums).  The
 * per-batch mean importance of stability_score (interpret/stability.py:103-106)
 * over one forward of all partitions' rows. */
tbn_status tbn_partition_mean(const float* values, int64_t rows_per_partition, int32_t partitions,
                              int32_t width, double* out, void* stream);

/* CRC-32C (Castagnoli, reflected 0x82F63B78) as io.py:22-36, hardware
 * accelerated on the host CPU when SSE4.2 is present.  Pure host code. */
uint32_t tbn_crc32c(const uint8_t* data, size_t n, uint32_t crc);

/* ---- .tbnt model streams (io.py:43-112; pure host code) ----------------
 * tbn_tbnt_parse replaces load_model (io.py:60-112): header, sections, CRC,
 * metadata JSON, ModelConfig / TabNetModel invariants, in the reference's
 * order and error classes (TBN_ERR_TRUNCATED / FORMAT / FORMAT_VERSION /
 * CHECKSUM / CONFIG).  The handle owns float64 copies of every parameter in
 * param_order and of the normalization stats. */
typedef struct tbn_tbnt tbn_tbnt;
tbn_status tbn_tbnt_parse(const uint8_t* data, size_t n, tbn_tbnt** out);
void tbn_tbnt_free(tbn_tbnt* t);
/* ModelConfig fields (lambda_sparse, seed beside tbn_config), model_version, #params */
tbn_status tbn_tbnt_info(const tbn_tbnt* t, tbn_config* cfg, double* lambda_sparse, int64_t* seed,
                         const char** model_version, int32_t* n_params);
/* parameter i of param_order: name, ndim, dims (<= 8), row-major float64 data */
tbn_status tbn_tbnt_param(const tbn_tbnt* t, int32_t i, const char** name, int32_t* ndim,
                          int64_t* dims, const double** data);
tbn_status tbn_tbnt_norm(const tbn_tbnt* t, const double** mean, const double** var);
/* The cold-start path: parse + verify the stream and build the device model
 * (weights packed for `precision` and uploaded to `device`) in one call, no
 * Python-side parsing.  cfg_flags = TBN_CFG_REGRESSION serves head column
 * `head_column` of the stored classifier as an identity head (TabNetRegressor). */
tbn_status tbn_model_create_from_tbnt(const uint8_t* data, size_t n, int32_t precision, int32_t device,
                                      int32_t cfg_flags, int32_t head_column, tbn_model** out);

/* ---- device preprocessing (data/preprocess.py:68-122, the numeric tail) ----
 * The host maps each raw cell to one float64 code (the string -> level lookup
 * stays on the host): standardize/passthrough -> the value or NaN if missing,
 * ordinal -> the plan's level integer or -1, onehot -> the category index or -1.
 * tbn_preprocess expands (rows x ncols) device codes into the model's float32
 * input (rows x width): median imputation, (v - mean) / std in float64 rounded
 * once (= the reference's float64 matrix cast to float32), ordinal values,
 * one-hot blocks of `width` levels, columns in plan order. */
#define TBN_PREP_STANDARDIZE 0
#define TBN_PREP_PASSTHROUGH 1
#define TBN_PREP_ORDINAL 2
#define TBN_PREP_ONEHOT 3
typedef struct {
  int32_t kind;     /* TBN_PREP_*                                  */
  int32_t width;    /* one-hot: number of categories; else 1       */
  double median;    /* imputation value (standardize, passthrough) */
  double mean;      /* standardize                                 */
  double std;       /* standardize (ddof=1, never 0)               */
} tbn_prep_column;
typedef struct tbn_prep tbn_prep;
tbn_status tbn_prep_create(const tbn_prep_column* cols, int32_t ncols, int32_t device, tbn_prep** out);
void tbn_prep_destroy(tbn_prep* plan);
int32_t tbn_prep_width(const tbn_prep* plan);
tbn_status tbn_preprocess(const tbn_prep* plan, const double* codes, int64_t rows, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TABNET_B200_H */
