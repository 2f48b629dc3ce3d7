/*
 * splitq.h — C-ABI of the B200 (sm_100a) SplitQ split-linear hot path.
 *
 * Plain pointers and sizes only (no torch / numpy types). Device pointers are
 * CUDA device addresses owned by the caller; host pointers are only read
 * during the call. Every function returns SPLITQ_OK (0) or a negative status;
 * splitq_last_error() returns the thread-local message of the last failure.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/modquant/):
 *
 *   splitq_layer_create     SplitLayer (layer.py:46-97) + the weight half of
 *                           forward_with_cache (layer.py:137-163), done once:
 *                           the caller passes the integer weight codes and
 *                           fp64 column scales of Q(R), Q(W_t/d_t), Q(W_v/d_v),
 *                           Q(u*), Q(gate*v) exactly as compute_params /
 *                           fake_quantize define them (quantizer.py:104-155).
 *   splitq_forward          forward(layer, batch) (layer.py:175-177 via
 *                           forward_with_cache :118-172) on a device batch.
 *   splitq_quantize_rows    compute_params + fake_quantize with PER_TOKEN
 *                           granularity (quantizer.py:104-155), returning the
 *                           integer codes, scales and zero points.
 *   splitq_mocd_*           vision_score / init_transform column max /
 *                           percentile_rank / text_score (mocd.py:72-150,
 *                           transform.py:89).
 *
 * Error mapping used by the Python shim: SPLITQ_ERR_INVALID,
 * SPLITQ_ERR_UNSUPPORTED and SPLITQ_ERR_DATA -> ValueError (same messages as
 * the reference where it has them); SPLITQ_ERR_CUDA / SPLITQ_ERR_NCCL ->
 * RuntimeError.
 */
#ifndef SPLITQ_H_
#define SPLITQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPLITQ_OK 0
#define SPLITQ_ERR_INVALID (-1)     /* bad argument / shape (ValueError) */
#define SPLITQ_ERR_UNSUPPORTED (-2) /* spec the GPU path does not implement (ValueError) */
#define SPLITQ_ERR_CUDA (-3)        /* CUDA runtime failure (RuntimeError) */
#define SPLITQ_ERR_DATA (-4)        /* data-dependent failure found on device (ValueError) */
#define SPLITQ_ERR_NCCL (-5)        /* NCCL failure (RuntimeError) */

/* element types of activation inputs / outputs */
#define SPLITQ_F16 0
#define SPLITQ_F32 1
#define SPLITQ_F64 2
#define SPLITQ_BF16 3

/* device error word bits returned by splitq_read_status */
#define SPLITQ_STATUS_NONFINITE 1  /* "non-finite value in matrix" (tensor.py:39-40) */
#define SPLITQ_STATUS_SCALE 2      /* "scales must be positive" (quantizer.py:72-73) */
#define SPLITQ_STATUS_TAG 4        /* "tags must be 0 (text) or 1 (vision)" (tensor.py:71-72) */
#define SPLITQ_STATUS_LR_RANGE 8   /* low-rank fp16 operand overflow */

/* forward flags */
#define SPLITQ_FWD_RAW 1     /* y receives raw accumulators (see splitq_forward) */
#define SPLITQ_FWD_PROFILE 2 /* record stage events on the stream (splitq_profile_read) */
#define SPLITQ_FWD_UNPACKED 4 /* main GEMM streams the int8 weight copy instead of the packed
                                 4-bit codes (W <= 4 bits); for A/B parity checks */

typedef struct splitq_layer_s* splitq_layer_t;

/* QuantSpec (quantizer.py:27-57). bits in [2, 8]; identity (None) and bits > 8
 * are rejected with SPLITQ_ERR_UNSUPPORTED. Activations are PER_TOKEN,
 * weights PER_CHANNEL (the only granularities that factor out of a GEMM). */
typedef struct {
  int32_t bits;
  int32_t symmetric;
} splitq_qspec_t;

/* Layer description. Index sets and transform scales are host arrays; weight
 * code matrices are host int8 arrays in the reference orientation
 * (K rows x N cols, row-major), scales are host fp64, one per column. */
typedef struct {
  int64_t d_in, d_out;
  int64_t n_main, n_text, n_vision;
  const int64_t* c_main; /* ChannelPartition (mocd.py:19-42) */
  const int64_t* c_text;
  const int64_t* c_vision;
  const double* scale_main; /* Transform.scale (transform.py:37-39) */
  const double* scale_text;
  const double* scale_vision;
  splitq_qspec_t act;    /* layer.act_spec */
  splitq_qspec_t weight; /* layer.weight_spec */
  int32_t aux_bits_floor; /* AUX_BITS_FLOOR (layer.py:38) */
  int32_t use_cws, use_mac;
  int64_t r_cws, r_mac;
  const int8_t* q_main; const double* s_main;     /* n_main x d_out : Q(R) or Q(P^-1 W_m) */
  const int8_t* q_text; const double* s_text;     /* n_text x d_out : Q_aux(W_t / d_t) */
  const int8_t* q_vision; const double* s_vision; /* n_vision x d_out */
  const int8_t* q_us; const double* s_us;         /* n_main x r_cws : Q_aux(u*) */
  const int8_t* q_vs; const double* s_vs;         /* r_cws x d_out : Q_aux(gate * v_base) */
  const int8_t* q_uc; const double* s_uc;         /* n_main x r_mac */
  const int8_t* q_vc; const double* s_vc;         /* r_mac x d_out */
} splitq_layer_desc_t;

/* Offsets (bytes, from the workspace base) of every intermediate the forward
 * writes, so tests can read the codes / scales back. -1 = not present. */
typedef struct {
  int64_t total_bytes;
  int64_t status;                                  /* int32 error word */
  int64_t text_idx, text_rows, n_text;             /* int32 */
  int64_t a_main; int64_t ld_main;                 /* int8 codes [T x ld_main]; column c is
                                                      channel c when main_natural (outlier
                                                      columns hold don't-care codes) */
  int64_t s_main, sf_main, zp_main, lrs_main, rho; /* f64, f32, i32, f32, f32 per row */
  int64_t a_text; int64_t ld_text;
  int64_t s_text, sf_text, zp_text;
  int64_t a_vision; int64_t ld_vision;
  int64_t s_vision, sf_vision, zp_vision;
  int64_t a_mac;                                   /* int8 codes [n_text_rows x ld_main] */
  int64_t s_mac, zp_mac, lrs_mac;                  /* per compact text row */
  int64_t lr_a; int64_t k_lr;                      /* fp16 [T x k_lr] low-rank operand */
  int32_t code_centered_main;                      /* 1: codes stored as (q - zp) s8; 0: q as u8 */
  int32_t code_centered_aux;
  int32_t main_natural;                            /* 1: main / MAC codes in natural channel order */
  int32_t reserved;
  int64_t acc_scratch, acc_scratch_bytes;          /* split-K partial accumulators (decode-sized calls) */
  int64_t a_main_fp4;                              /* E2M1 copy of the main codes [tokens x ld_main / 2]
                                                      (A2 x W3 / W2 layers, prefill: kind::mxf4 GEMM; -1 if none) */
} splitq_ws_layout_t;

const char* splitq_last_error(void);
int splitq_version(void);
int splitq_device_sm_count(int device, int* out);

int splitq_layer_create(const splitq_layer_desc_t* desc, int device, splitq_layer_t* out);
int splitq_layer_destroy(splitq_layer_t layer);
int splitq_workspace_layout(splitq_layer_t layer, int64_t tokens, splitq_ws_layout_t* out);

/* y = forward(layer, batch). x: device [tokens x x_ld] of x_dtype (d_in valid
 * columns); tags: device uint8 [tokens] (0 text, 1 vision); y: device
 * [tokens x y_ld] of y_dtype (F32 / F16 / BF16). With SPLITQ_FWD_RAW, y must
 * hold 2 consecutive [tokens x y_ld] 32-bit planes: the int32 main-channel
 * accumulator sum_k (q_a - z_a) * q_w and the fp32 auxiliary accumulator
 * (outlier + low-rank branches, scaled by 1 / (rho_i kappa_j)).
 * Asynchronous on `stream` (cudaStream_t); call splitq_read_status to
 * surface data-dependent errors. */
int splitq_forward(splitq_layer_t layer, const void* x, int x_dtype, int64_t x_ld,
                   const uint8_t* tags, int64_t tokens, void* y, int y_dtype, int64_t y_ld,
                   void* workspace, size_t workspace_bytes, void* stream, int flags);

/* Stage times of the SPLITQ_FWD_PROFILE calls since the last read, summed:
 * stage_ms[0] = row compaction + K1 quantizer, [1] = low-rank first stages,
 * [2] = split GEMM. CUDA events on the launch stream; synchronises. */
int splitq_profile_read(splitq_layer_t layer, double* stage_ms, int32_t* calls);

/* Synchronise `stream` and read the device error word of the workspace;
 * returns SPLITQ_ERR_DATA (with the reference's message) when it is set. */
int splitq_read_status(void* workspace, void* stream, int32_t* status_out);

/* Standalone per-token quantizer (PER_TOKEN compute_params + codes):
 * x device [rows x x_ld], codes device int8 [rows x codes_ld] (stored as
 * (q - zp) when centered, else q as u8), scales device f64 [rows],
 * zero_points device int32 [rows], status device int32 [1]. */
int splitq_quantize_rows(const void* x, int x_dtype, int64_t x_ld, int64_t rows, int64_t cols,
                         splitq_qspec_t spec, int8_t* codes, int64_t codes_ld, double* scales,
                         int32_t* zero_points, int32_t* status, int32_t* centered_out,
                         void* stream);

/* Raw tcgen05 int8 GEMM (the forward's main-path kernel in raw mode):
 * C[m][n] = sum_k A[m][k] * B[n][k]; A, B K-major int8 (a_signed selects
 * s8 / u8 for A, B is s8), C int32 [m x ldc]. */
int splitq_gemm_i8(const int8_t* a, int64_t lda, int a_signed, const int8_t* b, int64_t ldb,
                   int32_t* c, int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream);

/* MOCD calibration statistics (mocd.py:72-150; transform.py:89).
 * x device [tokens x x_ld] (x_dtype), tags device uint8. All asynchronous. */

/* vision_max[c] = max over vision rows of |x[:, c]| (vision_score,
 * mocd.py:72-77); all_max[c] = max over all rows (the init_transform
 * statistic, transform.py:89). fp64 [dim]; status: SPLITQ_STATUS_* bits. */
int splitq_mocd_absmax(const void* x, int x_dtype, int64_t x_ld, const uint8_t* tags,
                       int64_t tokens, int64_t dim, double* vision_max, double* all_max,
                       int32_t* status, void* stream);
/* percentile_rank numerators (mocd.py:92-111): counts[i][j] =
 * #{l in cand : |x[r_i, l]| <= |x[r_i, cand[j]]|} for the text rows
 * r_i = text_rows[i], i < *n_text (device count, max_text rows allocated);
 * uint16 [max_text x n_cand], row-major. fp16 / bf16 rows: a 32K-key
 * histogram per row (SPLITQ_MOCD_RC_SORT=1 selects the sort path used for
 * fp32 / fp64 rows). */
int splitq_mocd_rank_counts(const void* x, int x_dtype, int64_t x_ld, const int32_t* text_rows,
                            const int32_t* n_text, int64_t max_text, const int32_t* cand,
                            int64_t n_cand, uint16_t* counts, void* stream);
/* out[c][r] = in[r][c] (uint16), out row stride ld_out. */
int splitq_mocd_transpose_u16(const uint16_t* in, int64_t rows, int64_t cols, uint16_t* out,
                              int64_t ld_out, void* stream);
/* text_score (mocd.py:141-150) for the channel rows [c0, c1) of counts_t:
 * _kmeans_1d (mocd.py:114-138) of counts_t[c][0..n_text) / n_cand,
 * evaluated with numpy's exact float64 arithmetic (quantile init,
 * pairwise-sum means). counts_t: uint16 [>= c1 x ld] (transposed counts of
 * a channel range); n_cand: the rank denominator |C'| (the counts lie in
 * 1..n_cand); scores fp64, scores[c] written for c in [c0, c1). Rows that
 * start 16-byte aligned are read in whole 16-byte vectors: the buffer must
 * extend to the next multiple of 8 tokens past each such row (ld a multiple
 * of 8, as mocd_gpu allocates it).
 * The library keeps one device scratch buffer per device for the compacted
 * cluster members (k x 512 x ceil8(n_text / 512) uint16 per resident CTA),
 * grown on demand under a lock held through the launch. */
int splitq_mocd_text_score(const uint16_t* counts_t, int64_t ld, int64_t n_cand, int64_t n_text,
                           int k, int max_iter, int64_t c0, int64_t c1, double* scores,
                           void* stream);
/* select_topk (mocd.py:80-89): ascending indices of the k largest scores,
 * ties to the lower index. flags: int32 [n] scratch, out: int64 [k]. */
int splitq_mocd_topk(const double* scores, int64_t n, int64_t k, int32_t* flags, int64_t* out,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLITQ_H_ */
