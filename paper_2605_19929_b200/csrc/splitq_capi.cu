// C-ABI implementation (include/splitq.h): layer packing, workspace layout and
// the launch sequence of the split-linear forward on one CUDA stream:
//   compact_text_rows -> K1 quantize -> LR1 (CWS) -> LR1 (MAC) -> split GEMM
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/splitq.h"
#include "gemm2_sm100.cuh"
#include "quantize.cuh"
#include "quantize_fast.cuh"
#include "k1w.cuh"
#include "gemv_decode.cuh"
#include "tma_host.cuh"
#include "nvtx.cuh"

using namespace splitq;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(SPLITQ_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));     \
  } while (0)

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// tile N: up to 160 with the fp32 aux accumulator (two main buffers + one aux
// buffer = 3 bn TMEM columns), up to 256 without it (two main buffers)
int tile_n(int64_t n, bool aux) {
  if (const char* e = getenv("SPLITQ_TILE_N")) {  // experiments: force the tile width
    const int f = atoi(e);
    if (f >= 32 && f % 32 == 0 && f <= (aux ? G2_BN : G2_BN_MAX)) return f;
  }
  if (aux) {  // 160-wide tiles unless the last tile would waste > 5 % of the columns
    const int64_t r160 = round_up(n, G2_BN);
    if (n > 128 && r160 * 100 > n * 105) return 128;
  }
  return (int)std::min<int64_t>(aux ? G2_BN : G2_BN_MAX, round_up(n, 32));
}

// calls with at most this many token rows run the GEMMs swap-AB (decode)
constexpr int64_t kSwapMaxRows = 128;
inline bool use_swap(int64_t T) { return T <= kSwapMaxRows && !getenv("SPLITQ_NO_SWAP"); }
// token tile of a swap-AB launch: N of the MMA (multiple of 16, <= 128)
inline int swap_bn(int64_t T) { return (int)std::min<int64_t>(128, std::max<int64_t>(16, (T + 15) / 16 * 16)); }

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cache[device] = v;
  }
  return cache[device];
}

// QuantSpec -> device spec (quantizer.py:41-51). Codes are stored centred
// (q - zp) as s8 whenever that fits (symmetric, or asymmetric <= 7 bits),
// otherwise as u8 with the zero point applied in the GEMM epilogue.
int make_spec(splitq_qspec_t s, QSpecDev* out, const char* what) {
  if (s.bits < 2 || s.bits > 8)
    return fail(SPLITQ_ERR_UNSUPPORTED,
                "%s: the GPU path supports integer bit widths 2..8 (got %d); identity and "
                ">8-bit specs stay on the CPU reference",
                what, s.bits);
  if (s.symmetric) {
    out->qmin = -(1 << (s.bits - 1)) + 1;
    out->qmax = (1 << (s.bits - 1)) - 1;
    out->sym = 1;
    out->centered = 1;
  } else {
    out->qmin = 0;
    out->qmax = (1 << s.bits) - 1;
    out->sym = 0;
    out->centered = s.bits <= 7 ? 1 : 0;
  }
  return SPLITQ_OK;
}

splitq_qspec_t with_floor(splitq_qspec_t s, int floor_bits) {  // quantizer.py:53-57
  if (s.bits < floor_bits) s.bits = floor_bits;
  return s;
}

struct DevBuf {
  std::vector<void*> ptrs;
  int alloc(void** out, size_t bytes) {
    *out = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) return fail(SPLITQ_ERR_CUDA, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    ptrs.push_back(*out);
    return SPLITQ_OK;
  }
  template <typename T>
  int upload(T** out, const T* host, size_t count) {
    int rc = alloc(reinterpret_cast<void**>(out), count * sizeof(T));
    if (rc) return rc;
    if (count) {
      cudaError_t e = cudaMemcpy(*out, host, count * sizeof(T), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return fail(SPLITQ_ERR_CUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
    }
    return SPLITQ_OK;
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
};

// K x N row-major centred codes -> N x ld K-major (zero padded) + column sums.
// With a row map, code row k lands at K position kmap[k] (the natural channel
// index of main channel k; the other positions stay zero).
void transpose_codes(const int8_t* q, int64_t K, int64_t N, int64_t ld, std::vector<int8_t>& out,
                     std::vector<int32_t>& colsum, const int64_t* kmap = nullptr) {
  out.assign((size_t)N * ld, 0);
  colsum.assign((size_t)N, 0);
  for (int64_t k = 0; k < K; ++k) {
    const int8_t* src = q + k * N;
    const int64_t kk = kmap ? kmap[k] : k;
    for (int64_t n = 0; n < N; ++n) {
      out[(size_t)n * ld + kk] = src[n];
      colsum[n] += src[n];
    }
  }
}

// E2M1 nibble of a small integer code k in [-3, 3]: |k| 0, 1, 2, 3 -> 0x0, 0x2,
// 0x4, 0x5 (exponent / mantissa of 0, 1, 2, 3), sign in bit 3. Element 2i of a
// K-major row sits in the low nibble of byte i (A and B alike, so the dot
// products do not depend on the nibble order within a byte).
uint8_t e2m1_of(int k) {
  static const uint8_t mag[4] = {0x0, 0x2, 0x4, 0x5};
  return (uint8_t)(mag[k < 0 ? -k : k] | (k < 0 ? 0x8 : 0x0));
}

double pow2_ceil(double v) {  // smallest power of two >= v (v > 0)
  int e;
  const double m = std::frexp(v, &e);  // v = m * 2^e, m in [0.5, 1)
  return m == 0.5 ? std::ldexp(1.0, e - 1) : std::ldexp(1.0, e);
}

}  // namespace

struct splitq_layer_s {
  int device = 0;
  int64_t d_in = 0, d_out = 0, n_main = 0, n_text = 0, n_vis = 0, r_s = 0, r_c = 0;
  QSpecDev act{}, aux{};
  int use_cws = 0, use_mac = 0;
  // Main-path codes live in natural channel order: column c of the code rows
  // is channel c (outlier channels carry don't-care codes against all-zero
  // weight rows), so K1 needs no gather and the GEMM K is d_in.
  int64_t k_nat = 0;
  int64_t ld_main = 0, ld_text = 0, ld_vis = 0;
  int64_t r_s16 = 0, r_c16 = 0, k_lr = 0;  // k_lr = K of the fp16 auxiliary GEMM
  int64_t kt16 = 0, kv16 = 0, off_t = 0, off_v = 0, off_s = 0, off_c = 0, r_s8 = 0;
  DevBuf mem;
  int* c_main = nullptr; double* d_main = nullptr; float* d_main32 = nullptr;
  float* d_main_lo32 = nullptr;  // fl32(d_main - d_main32): the compensated MAC pass (K1, wide aux codes)
  int k3_ok = 0;  // smoothing scales within the fp32 fast path's range
  int* c_text = nullptr; double* d_text = nullptr;
  int* c_vis = nullptr; double* d_vis = nullptr;
  int8_t* b_main = nullptr; float* s_main = nullptr; int* cs_main = nullptr;
  uint8_t* bp_main = nullptr;  // packed 4-bit main weights [d_out x ld_main / 2] (W <= 4 bits)
  uint8_t* bf4_main = nullptr; // E2M1 main weights [d_out x ld_main / 2] (A2 x W3 / W2: kind::mxf4)
  int wmax = 0;                // max |main weight code| (bounds the int32 main accumulator)
  int8_t* b_us = nullptr; float* s_us = nullptr; int* cs_us = nullptr;
  int8_t* b_uc = nullptr; float* s_uc = nullptr; int* cs_uc = nullptr;
  __half* b_lr = nullptr; float* kappa = nullptr;
  // stage timing (SPLITQ_FWD_PROFILE): 4 events per profiled call
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // prefill: the MAC first stage runs on a side stream beside the CWS one
  // (fork / join events on the caller's stream; graph-capture safe)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::mutex side_mu;  // creation + the fork / join enqueues (host threads may share a layer)
};

namespace {

int pack_weight(splitq_layer_s* L, const int8_t* q, const double* s, int64_t K, int64_t N,
                int64_t ld, int8_t** b, float** sc, int** cs, double extra_div = 1.0,
                const std::vector<double>* per_col_div = nullptr, const int64_t* kmap = nullptr) {
  std::vector<int8_t> t;
  std::vector<int32_t> colsum;
  transpose_codes(q, K, N, ld, t, colsum, kmap);
  std::vector<float> sf((size_t)N);
  for (int64_t n = 0; n < N; ++n) {
    double v = s[n] / extra_div;
    if (per_col_div) v /= (*per_col_div)[n];
    sf[n] = (float)v;
  }
  int rc = L->mem.upload(b, t.data(), t.size());
  if (!rc) rc = L->mem.upload(sc, sf.data(), sf.size());
  if (!rc) rc = L->mem.upload(cs, colsum.data(), colsum.size());
  return rc;
}

int validate_index_set(const int64_t* c, int64_t n, int64_t dim, const char* name) {
  for (int64_t i = 0; i < n; ++i) {
    if (c[i] < 0 || c[i] >= dim) return fail(SPLITQ_ERR_INVALID, "%s index out of range", name);
    if (i && c[i] <= c[i - 1]) return fail(SPLITQ_ERR_INVALID, "%s must be strictly ascending", name);
  }
  return SPLITQ_OK;
}

int check_codes(const int8_t* q, int64_t count, const QSpecDev& s, const char* name) {
  // centred weight codes: symmetric in [qmin, qmax]; asymmetric in
  // [qmin - zp, qmax - zp], a subset of [-(qmax-qmin), qmax-qmin]
  const int lo = s.sym ? s.qmin : -(s.qmax - s.qmin), hi = s.sym ? s.qmax : s.qmax - s.qmin;
  for (int64_t i = 0; i < count; ++i)
    if (q[i] < lo || q[i] > hi) return fail(SPLITQ_ERR_INVALID, "%s code out of range", name);
  return SPLITQ_OK;
}

}  // namespace

extern "C" {

const char* splitq_last_error(void) { return g_last_error.c_str(); }
int splitq_internal_fail(int code, const char* msg) { return fail(code, "%s", msg); }
int splitq_version(void) { return 1; }

int splitq_device_sm_count(int device, int* out) {
  if (!out) return fail(SPLITQ_ERR_INVALID, "null output");
  *out = sm_count(device);
  return SPLITQ_OK;
}

int splitq_layer_create(const splitq_layer_desc_t* d, int device, splitq_layer_t* out) {
  if (!d || !out) return fail(SPLITQ_ERR_INVALID, "null argument");
  *out = nullptr;
  if (d->d_in <= 0 || d->d_out <= 0) return fail(SPLITQ_ERR_INVALID, "empty layer");
  if (d->n_main + d->n_text + d->n_vision != d->d_in)
    return fail(SPLITQ_ERR_INVALID, "channel sets must cover exactly 0..dim-1");
  if (d->n_main < d->n_text || d->n_main < d->n_vision)
    return fail(SPLITQ_ERR_INVALID, "main set must be at least as large as each outlier set");
  QSpecDev act, wsp, aux, waux;
  int rc = make_spec(d->act, &act, "act_spec");
  if (!rc) rc = make_spec(d->weight, &wsp, "weight_spec");
  if (rc) return rc;
  const int floor_bits = d->aux_bits_floor;
  rc = make_spec(with_floor(d->act, floor_bits), &aux, "act_spec (aux floor)");
  if (!rc) rc = make_spec(with_floor(d->weight, floor_bits), &waux, "weight_spec (aux floor)");
  if (rc) return rc;
  // centred weight codes must fit int8: symmetric codes lie in [qmin, qmax]
  // (W8 sym: -127..127, the reference's DEFAULT_WEIGHT_SPEC, layer.py:41),
  // asymmetric ones in [-(qmax - qmin), qmax - qmin]
  auto w_fits = [](const QSpecDev& s) { return s.sym ? s.qmax <= 127 : s.qmax - s.qmin <= 127; };
  if (!w_fits(wsp) || !w_fits(waux))
    return fail(SPLITQ_ERR_UNSUPPORTED, "weight codes must fit int8 (asymmetric 8-bit weights unsupported)");
  if (d->use_cws && (d->r_cws <= 0 || d->r_cws > std::min(d->n_main, d->d_out)))
    return fail(SPLITQ_ERR_INVALID, "branch rank exceeds min(path width, d_out)");
  if (d->use_mac && (d->r_mac <= 0 || d->r_mac > std::min(d->n_main, d->d_out)))
    return fail(SPLITQ_ERR_INVALID, "branch rank exceeds min(path width, d_out)");
  if ((rc = validate_index_set(d->c_main, d->n_main, d->d_in, "c_main"))) return rc;
  if ((rc = validate_index_set(d->c_text, d->n_text, d->d_in, "c_text"))) return rc;
  if ((rc = validate_index_set(d->c_vision, d->n_vision, d->d_in, "c_vision"))) return rc;
  {
    std::vector<char> seen((size_t)d->d_in, 0);
    for (auto [c, n] : {std::pair<const int64_t*, int64_t>{d->c_main, d->n_main},
                        {d->c_text, d->n_text}, {d->c_vision, d->n_vision}})
      for (int64_t i = 0; i < n; ++i) {
        if (seen[c[i]]) return fail(SPLITQ_ERR_INVALID, "channel sets must be pairwise disjoint");
        seen[c[i]] = 1;
      }
  }
  if ((rc = check_codes(d->q_main, d->n_main * d->d_out, wsp, "q_main"))) return rc;
  if (d->n_text && (rc = check_codes(d->q_text, d->n_text * d->d_out, waux, "q_text"))) return rc;
  if (d->n_vision && (rc = check_codes(d->q_vision, d->n_vision * d->d_out, waux, "q_vision")))
    return rc;

  CUDA_TRY(cudaSetDevice(device));
  auto* L = new splitq_layer_s();
  L->device = device;
  L->d_in = d->d_in;
  L->d_out = d->d_out;
  L->n_main = d->n_main;
  L->n_text = d->n_text;
  L->n_vis = d->n_vision;
  L->act = act;
  L->aux = aux;
  L->use_cws = d->use_cws ? 1 : 0;
  L->use_mac = d->use_mac ? 1 : 0;
  L->r_s = L->use_cws ? d->r_cws : 0;
  L->r_c = L->use_mac ? d->r_mac : 0;
  L->k_nat = L->d_in;
  L->ld_main = round_up(L->d_in, 16);
  L->ld_text = round_up(std::max<int64_t>(L->n_text, 1), 16);
  L->ld_vis = round_up(std::max<int64_t>(L->n_vis, 1), 16);
  L->r_s16 = round_up(L->r_s, 16);
  L->r_c16 = round_up(L->r_c, 16);
  // auxiliary fp16 operand segments: [text hi|lo|hi][vision hi|lo|hi][CWS hi|lo][MAC]
  // (the CWS first stage is split hi / lo: the branch can carry a large share
  // of the output, so fp16 rounding of it alone would exceed the tolerance)
  L->kt16 = round_up(L->n_text, 16);
  L->kv16 = round_up(L->n_vis, 16);
  L->off_t = 0;
  L->off_v = 3 * L->kt16;
  L->off_s = L->off_v + 3 * L->kv16;
  // segments start at multiples of 8 halves (16 B: LR1 stores 8 columns at a
  // time); the fp16 MMA K step is 16 and a stage 64, so only the total pads
  L->r_s8 = round_up(L->r_s, 8);
  L->off_c = L->off_s + 2 * L->r_s8;
  L->k_lr = (L->off_c + L->r_c) ? round_up(L->off_c + L->r_c, 64) : 0;

  auto cleanup = [&](int code) {
    L->mem.release();
    delete L;
    return code;
  };
  auto to_i32 = [](const int64_t* c, int64_t n) {
    std::vector<int32_t> v((size_t)n);
    for (int64_t i = 0; i < n; ++i) v[i] = (int32_t)c[i];
    return v;
  };
  {
    auto ct = to_i32(d->c_text, d->n_text), cv = to_i32(d->c_vision, d->n_vision);
    // main tables in natural channel order, padded to ld_main: index c -> c
    // (padding -> 0) and the smoothing scale of main channel c, NaN for
    // outlier channels and padding (NaN never wins a min / max, so K1 reads
    // whole groups without masks; quantize_fast.cuh, k1v3.cuh)
    std::vector<int32_t> cm((size_t)L->ld_main, 0);
    for (int64_t c = 0; c < L->d_in; ++c) cm[c] = (int32_t)c;
    std::vector<double> dm((size_t)L->ld_main, std::nan(""));
    for (int64_t k = 0; k < d->n_main; ++k) dm[d->c_main[k]] = d->scale_main[k];
    std::vector<float> dm32((size_t)L->ld_main, std::nanf("")), dmlo((size_t)L->ld_main, 0.f);
    for (int64_t c = 0; c < L->ld_main; ++c) {
      dm32[c] = (float)dm[c];
      if (dm[c] == dm[c]) dmlo[c] = (float)(dm[c] - (double)dm32[c]);
    }
    L->k3_ok = 1;
    for (int64_t k = 0; k < d->n_main; ++k)
      if (!(d->scale_main[k] > 1e-30 && d->scale_main[k] < 1e30)) L->k3_ok = 0;
    if ((rc = L->mem.upload(&L->d_main32, dm32.data(), dm32.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->d_main_lo32, dmlo.data(), dmlo.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->c_main, cm.data(), cm.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->c_text, ct.data(), ct.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->c_vis, cv.data(), cv.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->d_main, dm.data(), dm.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->d_text, d->scale_text, d->n_text))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->d_vis, d->scale_vision, d->n_vision))) return cleanup(rc);
  }
  const int64_t N = d->d_out;
  if ((rc = pack_weight(L, d->q_main, d->s_main, d->n_main, N, L->ld_main, &L->b_main, &L->s_main,
                        &L->cs_main, 1.0, nullptr, d->c_main)))
    return cleanup(rc);
  for (int64_t i = 0; i < d->n_main * N; ++i) L->wmax = std::max(L->wmax, std::abs((int)d->q_main[i]));
  // centred codes must also fit signed 4 bits; packed rows are 16-byte multiples
  bool fits4 = wsp.qmax - wsp.qmin <= 15 && L->ld_main % 32 == 0;
  for (int64_t i = 0; fits4 && i < d->n_main * N; ++i) fits4 = d->q_main[i] >= -8 && d->q_main[i] <= 7;
  if (fits4 && !getenv("SPLITQ_UNPACKED_W")) {
    // W <= 4 bits: the main GEMM streams 4-bit codes (two per byte; byte i of
    // each 32-bit word holds codes 8g+i and 8g+4+i), unpacked in SMEM
    std::vector<uint8_t> bp((size_t)N * (L->ld_main / 2), 0);
    std::vector<int8_t> full((size_t)N * L->ld_main, 0);
    for (int64_t k = 0; k < d->n_main; ++k) {
      const int64_t kk = d->c_main[k];
      for (int64_t n = 0; n < N; ++n) full[(size_t)n * L->ld_main + kk] = d->q_main[k * N + n];
    }
    for (int64_t n = 0; n < N; ++n) {
      const int8_t* src = full.data() + (size_t)n * L->ld_main;
      uint8_t* dst = bp.data() + (size_t)n * (L->ld_main / 2);
      for (int64_t g = 0; g < L->ld_main / 8; ++g)
        for (int i = 0; i < 4; ++i)
          dst[4 * g + i] = (uint8_t)((src[8 * g + i] & 0xF) | ((src[8 * g + 4 + i] & 0xF) << 4));
    }
    if ((rc = L->mem.upload(&L->bp_main, bp.data(), bp.size()))) return cleanup(rc);
  }
  // A2 activations (centred codes in [-3, 3]) against weight codes in [-3, 3]
  // (W3 / W2): both exact in E2M1, so the prefill main GEMM can run on
  // kind::mxf4 (2x the int8 MMA rate) with unit block scales
  bool fits_e2m1 = act.centered && act.qmax - act.qmin <= 3 && L->ld_main % 32 == 0;
  for (int64_t i = 0; fits_e2m1 && i < d->n_main * N; ++i) fits_e2m1 = d->q_main[i] >= -3 && d->q_main[i] <= 3;
  if (fits_e2m1) {
    std::vector<uint8_t> bf((size_t)N * (L->ld_main / 2), 0);
    for (int64_t k = 0; k < d->n_main; ++k) {
      const int64_t kk = d->c_main[k];
      for (int64_t n = 0; n < N; ++n)
        bf[(size_t)n * (L->ld_main / 2) + kk / 2] |= (uint8_t)(e2m1_of(d->q_main[k * N + n]) << (4 * (kk & 1)));
    }
    if ((rc = L->mem.upload(&L->bf4_main, bf.data(), bf.size()))) return cleanup(rc);
  }
  if (L->k_lr) {
    // Low-rank first stage: A_lr[i, c] = (S_a[i] / rho_i) * (S_u[c] / sigma_c) * acc[i, c]
    // with sigma_c a power of two bounding |A_lr| by 2^15 (fp16-safe for any input).
    // Second stage B_lr (fp16, d_out x k_lr, K-major):
    //   CWS  cols [0, r_s):          qv_s[c, j] * sigma_c / kappa_j          (exact)
    //   MAC  cols [r_s16, r_s16+r_c): qv_c[c, j] * (S_vc[j]/colf[j]) * sigma'_c / kappa_j
    // and the epilogue adds rho_i * (kappa_j * colf[j]) * f[i, j], colf = S_vs (or S_vc).
    const int64_t K = d->n_main;
    auto sigmas = [&](const int8_t* qu, const double* su, int64_t r, const QSpecDev& a) {
      std::vector<double> sg((size_t)r, 1.0);
      for (int64_t c = 0; c < r; ++c) {
        int mx = 0;
        for (int64_t k = 0; k < K; ++k) mx = std::max(mx, std::abs((int)qu[k * r + c]));
        const double bound = 2.0 * su[c] * (double)K * (double)(a.qmax - a.qmin) * (double)mx;
        sg[c] = bound > 0 ? pow2_ceil(bound / 32768.0) : 1.0;
      }
      return sg;
    };
    std::vector<double> sig_s, sig_c;
    if (L->r_s) {
      if ((rc = check_codes(d->q_us, K * L->r_s, waux, "q_us")) ||
          (rc = check_codes(d->q_vs, L->r_s * N, waux, "q_vs")))
        return cleanup(rc);
      sig_s = sigmas(d->q_us, d->s_us, L->r_s, act);
      if ((rc = pack_weight(L, d->q_us, d->s_us, K, L->r_s, L->ld_main, &L->b_us, &L->s_us,
                            &L->cs_us, 1.0, &sig_s, d->c_main)))
        return cleanup(rc);
    }
    if (L->r_c) {
      if ((rc = check_codes(d->q_uc, K * L->r_c, waux, "q_uc")) ||
          (rc = check_codes(d->q_vc, L->r_c * N, waux, "q_vc")))
        return cleanup(rc);
      sig_c = sigmas(d->q_uc, d->s_uc, L->r_c, aux);
      if ((rc = pack_weight(L, d->q_uc, d->s_uc, K, L->r_c, L->ld_main, &L->b_uc, &L->s_uc,
                            &L->cs_uc, 1.0, &sig_c, d->c_main)))
        return cleanup(rc);
    }
    // B_aux (fp16, d_out x k_lr, K-major), per column j with colf = S_vs[j]
    // (or the first present branch scale) and kappa_j a power of two:
    //   text   [hi | hi | lo] of q_t[k, j] * (S_t[j] / colf) / kappa_j
    //   vision [hi | hi | lo] of q_v[k, j] * (S_v[j] / colf) / kappa_j
    //   CWS    q_vs[c, j] * sigma_c / kappa_j                      (exact)
    //   MAC    q_vc[c, j] * (S_vc[j] / colf) * sigma'_c / kappa_j
    // and the epilogue adds rho_i * (kappa_j * colf) * R_aux[i, j].
    std::vector<__half> blr((size_t)N * L->k_lr, __float2half(0.f));
    std::vector<float> kap((size_t)N);
    std::vector<double> row((size_t)L->k_lr);
    for (int64_t j = 0; j < N; ++j) {
      const double colf = L->r_s ? d->s_vs[j]
                          : L->n_text ? d->s_text[j]
                          : L->r_c ? d->s_vc[j]
                          : L->n_vis ? d->s_vision[j] : 1.0;
      std::fill(row.begin(), row.end(), 0.0);
      double mx = 0.0;
      for (int64_t k = 0; k < L->n_text; ++k) {
        row[L->off_t + k] = (double)d->q_text[k * N + j] * (d->s_text[j] / colf);
        mx = std::max(mx, std::fabs(row[L->off_t + k]));
      }
      for (int64_t k = 0; k < L->n_vis; ++k) {
        row[L->off_v + k] = (double)d->q_vision[k * N + j] * (d->s_vision[j] / colf);
        mx = std::max(mx, std::fabs(row[L->off_v + k]));
      }
      for (int64_t c = 0; c < L->r_s; ++c) {
        row[L->off_s + c] = (double)d->q_vs[c * N + j] * sig_s[c];
        mx = std::max(mx, std::fabs(row[L->off_s + c]));
      }
      for (int64_t c = 0; c < L->r_c; ++c) {
        row[L->off_c + c] = (double)d->q_vc[c * N + j] * (d->s_vc[j] / colf) * sig_c[c];
        mx = std::max(mx, std::fabs(row[L->off_c + c]));
      }
      const double kappa = mx > 0 ? pow2_ceil(mx) : 1.0;
      __half* dst = blr.data() + (size_t)j * L->k_lr;
      auto split3 = [&](int64_t off, int64_t n, int64_t k16) {
        for (int64_t k = 0; k < n; ++k) {
          const double v = row[off + k] / kappa;
          const __half hi = __double2half(v);
          const __half lo = __double2half(v - (double)__half2float(hi));
          dst[off + k] = hi;
          dst[off + k16 + k] = hi;
          dst[off + 2 * k16 + k] = lo;
        }
      };
      split3(L->off_t, L->n_text, L->kt16);
      split3(L->off_v, L->n_vis, L->kv16);
      for (int64_t c = 0; c < L->r_s; ++c)
        dst[L->off_s + c] = dst[L->off_s + L->r_s8 + c] = __double2half(row[L->off_s + c] / kappa);
      for (int64_t c = 0; c < L->r_c; ++c) dst[L->off_c + c] = __double2half(row[L->off_c + c] / kappa);
      kap[j] = (float)(kappa * colf);
    }
    if ((rc = L->mem.upload(&L->b_lr, blr.data(), blr.size()))) return cleanup(rc);
    if ((rc = L->mem.upload(&L->kappa, kap.data(), kap.size()))) return cleanup(rc);
  }
  *out = L;
  return SPLITQ_OK;
}

int splitq_layer_destroy(splitq_layer_t L) {
  if (!L) return SPLITQ_OK;
  cudaSetDevice(L->device);
  for (cudaEvent_t e : L->ev_pool) cudaEventDestroy(e);
  if (L->fork) cudaEventDestroy(L->fork);
  if (L->join) cudaEventDestroy(L->join);
  if (L->side) cudaStreamDestroy(L->side);
  L->mem.release();
  delete L;
  return SPLITQ_OK;
}

// LR1 split-K scratch of the decode GEMV: int32 [32 x r_s], [32 x r_c] + counters
// (one per channel block and n-tile)
static int64_t gv_scratch_bytes(const splitq_layer_s* L) {
  return 4 * (GV_MAX_ROWS * (L->r_s + L->r_c) + 4 * ((L->r_s + 15) / 16 + (L->r_c + 15) / 16));
}

// split-K scratch: the CWS first stage's slices first, the MAC stage's at this offset
static int64_t lr1_scratch_off(const splitq_layer_s* L, int64_t T) { return round_up(8 * T * L->r_s * 4, 256); }

int splitq_workspace_layout(splitq_layer_t L, int64_t T, splitq_ws_layout_t* o) {
  if (!L || !o) return fail(SPLITQ_ERR_INVALID, "null argument");
  if (T <= 0) return fail(SPLITQ_ERR_INVALID, "batch must contain at least one token");
  std::memset(o, 0xff, sizeof(*o));  // -1 everywhere
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = off;
    off = round_up(off + bytes, 256);
    return at;
  };
  // status word, MAC row count and (decode GEMV) the LR1 split-K partials +
  // arrival counters: one contiguous block zeroed by one memset per forward
  o->status = take(32 + gv_scratch_bytes(L));
  o->n_text = o->status + 16;
  o->text_idx = take(4 * T);
  o->text_rows = take(4 * T);
  o->ld_main = L->ld_main;
  o->a_main = take(T * L->ld_main);
  o->s_main = take(8 * T);
  o->sf_main = take(4 * T);
  o->zp_main = take(4 * T);
  o->lrs_main = take(4 * T);
  o->rho = take(4 * T);
  o->ld_text = L->ld_text;
  o->ld_vision = L->ld_vis;
  if (L->n_text) {
    o->a_text = take(T * L->ld_text);
    o->s_text = take(8 * T);
    o->sf_text = take(4 * T);
    o->zp_text = take(4 * T);
  }
  if (L->n_vis) {
    o->a_vision = take(T * L->ld_vis);
    o->s_vision = take(8 * T);
    o->sf_vision = take(4 * T);
    o->zp_vision = take(4 * T);
  }
  if (L->use_mac) {
    o->a_mac = take(T * L->ld_main);
    o->s_mac = take(8 * T);
    o->zp_mac = take(4 * T);
    o->lrs_mac = take(4 * T);
  }
  o->k_lr = L->k_lr;
  if (L->k_lr) o->lr_a = take(2 * T * L->k_lr);
  {
    // split-K scratch (int32 + fp32 partial accumulators) for launches whose
    // tile count cannot fill the GPU (decode-sized calls); shared by the LR1
    // and split-GEMM launches, which run in sequence on one stream
    const int64_t pairs = sm_count(L->device) / 2;
    const int64_t m_tiles = (T + 255) / 256;
    int64_t need = 0;
    const int64_t bn = tile_n(L->d_out, L->k_lr > 0);
    const bool swap = T <= kSwapMaxRows;
    const int64_t kmax = 8;  // split-K slices the scratch holds
    if (swap || m_tiles * ((L->d_out + bn - 1) / bn) * 2 <= pairs)
      need = std::max(need, kmax * T * L->d_out * 8);
    // (the two LR1 launches may run concurrently: each has its own slices)
    if ((L->r_s || L->r_c) && (swap || m_tiles * 2 <= pairs))
      need = std::max(need, lr1_scratch_off(L, T) + kmax * T * L->r_c * 4);
    o->acc_scratch_bytes = need;
    o->acc_scratch = need ? take(need) : -1;
  }
  o->a_main_fp4 = L->bf4_main ? take(T * L->ld_main / 2) : -1;
  o->total_bytes = off;
  o->code_centered_main = L->act.centered;
  o->main_natural = 1;
  o->code_centered_aux = L->aux.centered;
  return SPLITQ_OK;
}

}  // extern "C"

namespace {


struct GemmLaunch {
  G2Maps maps;
  G2Params p;
};

// Persistent launch: one CTA pair per two SMs (cluster of 2).
inline bool raw_unpacked(int flags) { return (flags & SPLITQ_FWD_UNPACKED) != 0; }

unsigned long long* g2_trace_last = nullptr;

// programmatic dependent launch of the GEMM-side kernels (SPLITQ_NO_PDL=1 disables)
bool pdl_enabled() {
  static const bool on = !getenv("SPLITQ_NO_PDL");
  return on;
}
int g2_trace_ctas = 0;

int launch_gemm(GemmLaunch& g, int device, int64_t max_rows, cudaStream_t stream,
                void* scratch = nullptr, int64_t scratch_bytes = 0) {
  static bool attr[64][2] = {};
  const int pk = g.p.packed_b ? 1 : 0;
  if (device >= 0 && device < 64 && !attr[device][pk]) {
    CUDA_TRY(cudaFuncSetAttribute(pk ? splitq_gemm2_kernel<true> : splitq_gemm2_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, G2_SMEM_BYTES));
    attr[device][pk] = true;
  }
  const int64_t m_tiles = ((g.p.swap ? g.p.N : max_rows) + G2_BM - 1) / G2_BM;
  const int64_t n_tiles = ((g.p.swap ? max_rows : g.p.N) + g.p.bn - 1) / g.p.bn;
  const int64_t tiles = m_tiles * n_tiles;
  if (tiles == 0) return SPLITQ_OK;
  const int64_t avail = sm_count(device) / 2;
  // Split-K when the tiles cannot fill the GPU (decode): each work item is a
  // K range of a tile, partial sums land in the scratch with RED atomics and a
  // finalize pass applies the epilogue.
  const int stages = g.p.k_aux / 64 + (g.p.k_main + 127) / 128;
  const bool has_aux = g.p.k_aux > 0;
  const int64_t slice = max_rows * g.p.N;
  g.p.k_split = 1;
  int final_mode = g.p.mode;
  // LR1 (N = rank, short rows of tiles): the split's scratch pass and extra
  // launch only pay for long K or very few tiles (7B q-proj LR1 at 8192
  // tokens: 71 us split vs 52 us unsplit; down-proj, K = 18944: split wins
  // up to ~8192 tokens)
  const bool split_ok = g.p.mode != G2_LR1 || stages >= 64 || tiles * 8 <= avail;
  if (scratch && split_ok && tiles * 2 <= avail && stages >= 2 && !getenv("SPLITQ_NO_SPLITK")) {
    int ks = (int)std::min<int64_t>(stages, std::max<int64_t>(2, avail / tiles));
    while (ks > 1 && ks * slice * (has_aux ? 8 : 4) > scratch_bytes) --ks;  // slices must fit
    if (ks > 1) {
      g.p.k_split = ks;
      g.p.acc_i32 = reinterpret_cast<int*>(scratch);
      g.p.acc_f32 = reinterpret_cast<float*>(reinterpret_cast<int*>(scratch) + ks * slice);
      g.p.ld_acc = g.p.N;
      g.p.acc_slice = slice;
      g.p.mode = G2_ACC;
    }
  }
  // wide N (gate / up: B beyond an L2 partition): m-fastest tile groups
  // whose A slab is ~32 MB (measured on the 7B gate / up GEMMs: group of 16-32
  // m-tiles 4.8-4.9 ms, row-major 5.4 ms, 64: 5.2-5.4 ms, 128: 6.0 ms)
  g.p.tile_gm = 0;
  if (!g.p.swap && n_tiles >= 64 && m_tiles > 1) {
    const int64_t slab = (int64_t)G2_BM * (g.p.k_main + 2 * (int64_t)g.p.k_aux);  // A bytes per m-tile
    int gm = (int)std::max<int64_t>(4, std::min<int64_t>(64, (32LL << 20) / slab));
    if (getenv("SPLITQ_TILE_GM")) gm = atoi(getenv("SPLITQ_TILE_GM"));
    g.p.tile_gm = gm;
  }
  const int64_t items = tiles * g.p.k_split;
  const int pairs = (int)std::min<int64_t>(items, avail);
#ifdef G2_TRACE
  static unsigned long long* trace_buf = nullptr;
  if (!trace_buf) cudaMalloc(&trace_buf, 148 * 8 * 8);
  // SPLITQ_TRACE_MODE=<G2 mode number>: trace only launches of that mode
  const char* tm = getenv("SPLITQ_TRACE_MODE");
  if (!tm || atoi(tm) == g.p.mode) {
    cudaMemsetAsync(trace_buf, 0, 148 * 8 * 8, stream);
    g.p.trace = trace_buf;
    g2_trace_last = trace_buf;
    g2_trace_ctas = 2 * pairs;
  }
#endif
  // programmatic dependent launch (set-up and first weight loads overlap the
  // preceding kernel's tail; see the kernel head)
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.stream = stream;
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(pk ? G2_THREADS_PACKED : G2_THREADS);
  cfg.dynamicSmemBytes = G2_SMEM_BYTES;
  if (pk) CUDA_TRY(cudaLaunchKernelEx(&cfg, splitq_gemm2_kernel<true>, g.maps, g.p));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, splitq_gemm2_kernel<false>, g.maps, g.p));
  if (g.p.mode == G2_ACC) {
    const int64_t total = max_rows * g.p.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4L * sm_count(device));
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, g2_finalize_kernel, g.p, final_mode, has_aux ? 1 : 0));
    g.p.mode = final_mode;
  }
  return SPLITQ_OK;
}

// Decode-sized calls (T <= gemv_max_rows()): warp-MMA GEMV kernels
// (gemv_decode.cuh) instead of the tensor-core tiles. The kernels take up to
// GV_MAX_ROWS = 32 rows (4 n-tiles). Measured on the 7B decode step (seven
// projections): batch 16 369 us GEMV vs 401 us tcgen05 swap-AB, batch 32
// 501 vs 414 us, so the default cut is 16. SPLITQ_GEMV_MAX_ROWS (read per
// call; 0 disables) overrides it.
int gemv_max_rows() {
  const char* e = getenv("SPLITQ_GEMV_MAX_ROWS");
  return std::min(e ? atoi(e) : 16, GV_MAX_ROWS);
}

constexpr int kGvSmemBudget = 216 * 1024;  // dynamic; + 8 KB static partials

inline int gv_ntiles(int64_t rows) { return rows <= 8 ? 1 : rows <= 16 ? 2 : 4; }

// GEMV launch shape from the token rows, the weight row bytes and the aux K;
// false when the staged rows leave no room for a 2-deep ring
// ctas_per_sm: CTAs each SM should hold (the launch's CTAs over the SMs):
// the ring takes what SMEM is left for that many; deeper rings keep more
// weight bytes in flight per SM (the GEMV streams at ring / latency)
bool gv_shape(int64_t rows, bool packed, int64_t row_bytes, int k_aux, GvArgs* g, int* smem,
              int ctas_per_sm = 1) {
  g->srows = (int)std::max<int64_t>(1, std::min<int64_t>(rows, 8 * gv_ntiles(rows)));
  g->nbox = (int)((row_bytes + 127) / 128);
  g->nbox_aux = k_aux / 64;
  g->units_main = (g->nbox + GV_BPU - 1) / GV_BPU;
  g->units_aux = (g->nbox_aux + GV_BPU - 1) / GV_BPU;
  g->act_stride = packed ? g->nbox * 256 + 16 : g->nbox * 128 + 64;
  g->aux_stride = k_aux ? g->nbox_aux * 128 + 64 : 0;
  const int fixed = gv_smem_bytes(g->srows, g->act_stride, g->aux_stride, 0);
  const int budget = std::min(kGvSmemBudget, 227 * 1024 / std::max(ctas_per_sm, 1) - 9 * 1024);
  g->stages = std::min(GV_MAX_STAGES, (budget - fixed) / (GV_BPU * GV_BOX_BYTES));
  if (g->stages < 2)  // too many CTAs per SM asked for: the largest ring one CTA fits
    g->stages = std::min(GV_MAX_STAGES, (kGvSmemBudget - fixed) / (GV_BPU * GV_BOX_BYTES));
  *smem = gv_smem_bytes(g->srows, g->act_stride, g->aux_stride, g->stages);
  return g->stages >= 2;
}

template <bool PACKED, bool ASIGNED, bool LR1, int NT>
int launch_gv_t(const GvMaps& maps, const G2Params& p, const GvArgs& g, int smem, int device, cudaStream_t s) {
  auto* kern = gv_kernel<PACKED, ASIGNED, LR1, NT>;
  static bool attr[64] = {};
  if (device >= 0 && device < 64 && !attr[device]) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kGvSmemBudget));
    attr[device] = true;
  }
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GV_THREADS, smem));
  if (per_sm < 1) return SPLITQ_ERR_UNSUPPORTED;
  const int blocks = (p.N + 15) / 16;
  const int grid = std::min(blocks * g.ksplit, per_sm * sm_count(device));
  // programmatic dependent launch: the CTAs start (and fill their weight
  // rings) while the preceding kernel finishes; they wait before reading its
  // outputs. SPLITQ_NO_PDL=1 launches plainly.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(GV_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps, p, g, blocks));
  return SPLITQ_OK;
}

template <bool PACKED, bool ASIGNED, bool LR1>
int launch_gv_n(const GvMaps& maps, const G2Params& p, const GvArgs& g, int smem, int rows, int device,
                cudaStream_t s) {
  switch (gv_ntiles(rows)) {
    case 1: return launch_gv_t<PACKED, ASIGNED, LR1, 1>(maps, p, g, smem, device, s);
    case 2: return launch_gv_t<PACKED, ASIGNED, LR1, 2>(maps, p, g, smem, device, s);
    default: return launch_gv_t<PACKED, ASIGNED, LR1, 4>(maps, p, g, smem, device, s);
  }
}

// whether a GEMV launch's staged rows and a 2-deep weight ring fit one CTA
bool gv_fits(int64_t rows, bool packed, int64_t row_bytes, int k_aux) {
  GvArgs g{};
  int smem;
  return gv_shape(rows, packed, row_bytes, k_aux, &g, &smem);
}

// One GEMV launch, planned: tensor maps, K split, SMEM.
struct GvPlan {
  GvMaps maps;
  G2Params p;
  GvArgs g;
  int smem;
  int blocks;
};

// weights: [N x row_bytes] (packed 4-bit or int8 codes); aux weights b_lr [N x k_aux] fp16;
// rows: the launch's token rows (an upper bound when p.m_count is device-side)
int gv_plan(GvPlan& pl, const G2Params& p, const GvArgs& g, int rows, const void* w, int64_t row_bytes,
            const __half* xb, bool packed, bool lr1, int device) {
  pl.p = p;
  pl.g = g;
  const int k_aux = lr1 ? 0 : p.k_aux;
  if (!gv_shape(rows, packed, row_bytes, k_aux, &pl.g, &pl.smem)) return fail(SPLITQ_ERR_UNSUPPORTED, "GEMV shape");
  pl.blocks = (p.N + 15) / 16;
  // LR1 (few channel blocks, long K): split K over CTAs only as far as one
  // CTA's ring cannot hold its range (a split adds the integer atomics, the
  // arrival counter and the read-back to the chain; a ring-sized range is one
  // round trip). SPLITQ_GV_KSPLIT (read per call, tests) forces the split.
  pl.g.ksplit = 1;
  if (lr1 && pl.g.red) {
    const char* e = getenv("SPLITQ_GV_KSPLIT");
    const int by_ring = (pl.g.units_main + pl.g.stages - 1) / std::max(pl.g.stages, 1);
    pl.g.ksplit = std::max(1, std::min({e ? atoi(e) : by_ring, pl.g.units_main,
                                        sm_count(device) / std::max(pl.blocks, 1)}));
  }
  // more CTAs than SMs: size the ring so that up to 2 fit an SM
  const int per_sm = std::min(2, (pl.blocks * pl.g.ksplit + sm_count(device) - 1) / sm_count(device));
  if (per_sm > 1 && !gv_shape(rows, packed, row_bytes, k_aux, &pl.g, &pl.smem, per_sm))
    return fail(SPLITQ_ERR_UNSUPPORTED, "GEMV shape");
  bool ok = make_map_2d(&pl.maps.w, w, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p.N, row_bytes, row_bytes, 16, 128);
  pl.maps.x = pl.maps.w;
  if (ok && k_aux)
    ok = make_map_2d(&pl.maps.x, xb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p.N, k_aux, 2 * (int64_t)k_aux, 16, 64);
  if (!ok) return fail(SPLITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (GEMV)");
  return SPLITQ_OK;
}

int launch_gv(G2Params p, GvArgs g, int rows, const void* w, int64_t row_bytes, const __half* xb, bool packed,
              bool a_signed, bool lr1, int device, cudaStream_t s) {
  GvPlan pl;
  int rc = gv_plan(pl, p, g, rows, w, row_bytes, xb, packed, lr1, device);
  if (rc) return rc;
  const GvMaps& maps = pl.maps;
  const int smem = pl.smem;
  if (lr1) return a_signed ? launch_gv_n<false, true, true>(maps, pl.p, pl.g, smem, rows, device, s)
                           : launch_gv_n<false, false, true>(maps, pl.p, pl.g, smem, rows, device, s);
  if (packed) return a_signed ? launch_gv_n<true, true, false>(maps, pl.p, pl.g, smem, rows, device, s)
                              : launch_gv_n<true, false, false>(maps, pl.p, pl.g, smem, rows, device, s);
  return a_signed ? launch_gv_n<false, true, false>(maps, pl.p, pl.g, smem, rows, device, s)
                  : launch_gv_n<false, false, false>(maps, pl.p, pl.g, smem, rows, device, s);
}

// Both LR1 GEMVs (CWS, MAC) in one launch (gv_lr1_pair_kernel)
template <bool AS1, bool AS2, int NT>
int launch_gv_pair_t(const GvPlan& a, const GvPlan& b, int device, cudaStream_t s) {
  auto* kern = gv_lr1_pair_kernel<AS1, AS2, NT>;
  static bool attr[64] = {};
  if (device >= 0 && device < 64 && !attr[device]) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kGvSmemBudget));
    attr[device] = true;
  }
  const int smem = std::max(a.smem, b.smem);
  const int ga = a.blocks * a.g.ksplit, gb = b.blocks * b.g.ksplit;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(ga + gb));
  cfg.blockDim = dim3(GV_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a.maps, a.p, a.g, a.blocks, b.maps, b.p, b.g, b.blocks, ga));
  return SPLITQ_OK;
}

int launch_gv_pair(const GvPlan& a, bool as1, const GvPlan& b, bool as2, int rows, int device, cudaStream_t s) {
  const int nt = gv_ntiles(rows);
#define GV_PAIR(A, B)                                                           \
  (nt == 1 ? launch_gv_pair_t<A, B, 1>(a, b, device, s)                          \
           : nt == 2 ? launch_gv_pair_t<A, B, 2>(a, b, device, s) : launch_gv_pair_t<A, B, 4>(a, b, device, s))
  if (as1) return as2 ? GV_PAIR(true, true) : GV_PAIR(true, false);
  return as2 ? GV_PAIR(false, true) : GV_PAIR(false, false);
#undef GV_PAIR
}

// K-major int8 operand, box of box_rows rows x 128 bytes (128-B swizzle)
bool map_i8(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
            uint32_t box_rows) {
  return make_map_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols, ld, box_rows, 128);
}
// K-major fp16 operand, box of box_rows rows x 64 elements
bool map_f16(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld_elems,
             uint32_t box_rows) {
  return make_map_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, rows, cols, ld_elems * 2, box_rows,
                     64);
}

// tile N: up to 160 with the fp32 aux accumulator (two main buffers + one aux
// buffer = 3 bn TMEM columns), up to 256 without it (two main buffers)

// i8 MMA instruction descriptor for the pair (M = 256), f16 likewise
uint32_t idesc_i8(bool a_signed, int bn) { return make_idesc(2, a_signed ? 1u : 0u, 1, G2_BM, bn); }
uint32_t idesc_f16(int bn) { return make_idesc(1, 0, 0, G2_BM, bn); }

}  // namespace


namespace {

template <typename T, bool GA, int G>
int launch_k1_g(const K1Params& k, int d_in, cudaStream_t stream) {
  const size_t smem = k1_group_smem(d_in, (int)sizeof(T), G);
  static bool attr[64] = {};  // per device: the attribute is per-context
  int device = 0;
  CUDA_TRY(cudaGetDevice(&device));
  if (device < 0 || device >= 64 || !attr[device]) {
    CUDA_TRY(cudaFuncSetAttribute(k1_group_kernel<T, GA, G>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    if (device >= 0 && device < 64) attr[device] = true;
  }
  constexpr int NG = K1G_WARPS / G;
  const unsigned grid = (unsigned)((k.T + NG - 1) / NG);
  k1_group_kernel<T, GA, G><<<grid, K1G_WARPS * 32, smem, stream>>>(k, d_in);
  CUDA_TRY(cudaGetLastError());
  return SPLITQ_OK;
}

template <typename T, bool GA>
int launch_k1_t(const K1Params& k, int d_in, cudaStream_t s) {
  // rows per group of G warps: keep one row's SMEM at most ~1/8 of the CTA budget
  const int row_bytes = d_in * (int)sizeof(T);
  int G = row_bytes <= 12 * 1024 ? 1 : row_bytes <= 24 * 1024 ? 2
        : row_bytes <= 48 * 1024 ? 4 : 8;
  if (getenv("SPLITQ_K1_G")) G = std::max(G, atoi(getenv("SPLITQ_K1_G")));
  if (k1_group_smem(d_in, (int)sizeof(T), G) > 200 * 1024) return SPLITQ_ERR_UNSUPPORTED;
  switch (G) {
    case 1: return launch_k1_g<T, GA, 1>(k, d_in, s);
    case 2: return launch_k1_g<T, GA, 2>(k, d_in, s);
    case 4: return launch_k1_g<T, GA, 4>(k, d_in, s);
    default: return launch_k1_g<T, GA, 8>(k, d_in, s);
  }
}

template <bool GA>
int launch_k1_dt(const K1Params& k, int d_in, cudaStream_t s) {
  switch (k.x_dtype) {
    case IN_F16: return launch_k1_t<__half, GA>(k, d_in, s);
    case IN_BF16: return launch_k1_t<__nv_bfloat16, GA>(k, d_in, s);
    case IN_F32: return launch_k1_t<float, GA>(k, d_in, s);
    default: return launch_k1_t<double, GA>(k, d_in, s);
  }
}

// K1 warp-per-row (fp16 / bf16 rows, d_in % 8 == 0, 16-B aligned rows):
// fp32 fast path with certified exact fp64 fallback (k1w.cuh).
unsigned long long* k1w_trace_last = nullptr;

template <typename T, bool SMF, int WPR, bool SYNC = false, bool G64 = false, bool PF = false>
int launch_k1w_t(const K1Params& k, int d_in, int device, cudaStream_t stream) {
  const int threads = WPR > 1 ? WPR * 32 : SYNC ? KW_THREADS_SYNC : KW_THREADS;
  // row groups stage the fp32 factors with the row for decode-sized calls
  // and rows up to 8192 channels; wide rows with many rows per CTA keep the
  // SMEM for co-resident row groups (SPLITQ_K1_STAGE_D=0|1 overrides)
  K1Params kk = k;
  const char* sde = getenv("SPLITQ_K1_STAGE_D");
  kk.kw_stage_d = sde ? atoi(sde) : (d_in <= 8192 || k.T <= 2 * sm_count(device));
  const size_t smem = k1w_smem(d_in, threads / 32, SMF, WPR, kk.kw_stage_d != 0);
  static int attr_dev[64] = {0};
  if (device >= 0 && device < 64 && !attr_dev[device]) {
    CUDA_TRY(cudaFuncSetAttribute(k1w_kernel<T, SMF, WPR, SYNC, G64, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    attr_dev[device] = 1;
  }
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1w_kernel<T, SMF, WPR, SYNC, G64, PF>, threads, smem));
  if (per_sm < 1) return SPLITQ_ERR_UNSUPPORTED;
  int64_t grid;
  if (WPR > 1) {  // one row per CTA
    grid = std::min<int64_t>(k.T, (int64_t)per_sm * sm_count(device));
  } else {
    const int64_t warps = (int64_t)per_sm * sm_count(device) * (threads / 32);
    grid = (std::min<int64_t>(k.T, warps) + threads / 32 - 1) / (threads / 32);
  }
#ifdef KW_TRACE
  static unsigned long long* kw_trace_buf = nullptr;
  if (!kw_trace_buf) cudaMalloc(&kw_trace_buf, 16 * 8);
  cudaMemsetAsync(kw_trace_buf, 0, 16 * 8, stream);
  kk.trace = kw_trace_buf;
  k1w_trace_last = kw_trace_buf;
#endif
  k1w_kernel<T, SMF, WPR, SYNC, G64, PF><<<(unsigned)grid, threads, smem, stream>>>(kk, d_in);
  CUDA_TRY(cudaGetLastError());
  return SPLITQ_OK;
}

template <typename T, bool G64>
int launch_k1w_g(const K1Params& k, int d_in, int device, cudaStream_t stream) {
  // 16-bit MAC fractions in SMEM (2 B per channel per warp): opt-in. It
  // removes the pass-G recompute but widens the MAC tie window; measured
  // 0.756 vs 0.696 ms on the 7B q-proj input, so the recompute stays default.
  static const char* env = getenv("SPLITQ_K1_SMF");
  const bool smf = k.use_mac && env && env[0] == '1' && d_in <= 8192;
  // Few rows (decode): a row per CTA of 8 warps, so one row's passes are not
  // one warp's serial latency chain (tools/k1_trace.py phase clocks;
  // 16 warps measured slower: the group barriers cost more than the passes
  // save). SPLITQ_K1_WPR=1|8|16 overrides.
  const char* wenv = getenv("SPLITQ_K1_WPR");  // read per call: tests switch it
  const int wpr_env = wenv ? atoi(wenv) : 0;
  // row groups also for wide rows (d_in > 8192) up to ~256 rows per SM: one
  // warp's serial passes over a wide row are the critical path when each
  // warp gets few rows, and row groups that keep only the row in SMEM (the
  // factors from the global table, launch_k1w_t) fit 5 per SM. 7B down
  // (d_in 18944): 4096 rows 0.53 (warp rows) -> 0.25 ms, 8192 rows 0.81 ->
  // 0.45 ms, 16384 1.16 -> 0.88 ms, 32768 1.82 -> 1.74 ms; at 65536 warp
  // rows win (3.04 vs 3.45 ms)
  const bool grouped = wpr_env ? wpr_env > 1
                               : k.T <= 2 * sm_count(device) || (d_in > 8192 && k.T <= 256 * sm_count(device));
  if (grouped && !smf)
    return wpr_env >= 16 ? launch_k1w_t<T, false, 16, false, G64>(k, d_in, device, stream)  // measured slower
                         : launch_k1w_t<T, false, 8, false, G64>(k, d_in, device, stream);
  if (smf) return launch_k1w_t<T, true, 1>(k, d_in, device, stream);
  // row rounds with a CTA barrier (k1w.cuh): faster at d_in <= 8192
  const char* senv = getenv("SPLITQ_K1_SYNC");
  const bool sync = senv ? senv[0] == '1' : d_in <= 8192;
  if (sync) return launch_k1w_t<T, false, 1, true, G64>(k, d_in, device, stream);
  // wide rows with a few rows per warp: loads one chunk ahead (k1w.cuh PF)
  const char* penv = getenv("SPLITQ_K1_PF");
  const bool pf = penv ? penv[0] == '1' : k.T <= 128 * sm_count(device);
  return pf ? launch_k1w_t<T, false, 1, false, G64, true>(k, d_in, device, stream)
            : launch_k1w_t<T, false, 1, false, G64>(k, d_in, device, stream);
}

template <typename T>
int launch_k1w(const K1Params& k, int d_in, int device, cudaStream_t stream) {
  // wide aux codes (S / S_e ~ aux levels > 32): the fp64 MAC pass (k1w.cuh)
  const bool g64 = k.use_mac && (k.aux.qmax - k.aux.qmin) > 32;
  return g64 ? launch_k1w_g<T, true>(k, d_in, device, stream) : launch_k1w_g<T, false>(k, d_in, device, stream);
}

bool k1v3_eligible(const K1Params& k, int d_in) {
  if (k.x_dtype != IN_F16 && k.x_dtype != IN_BF16) return false;
  if (d_in % 8 || (k.ldx % 8) || (reinterpret_cast<uintptr_t>(k.x) & 15)) return false;
  if (!k.d_main32 || !k.c_main || (k.ld_main % 8) || k.n_main != d_in) return false;
  return true;
}

// K1 dispatch: the SMEM-staged row-group kernel; the generic per-row CTA
// kernel (same arithmetic) covers code strides that are not 16-B multiples
// and rows too large to stage.
int launch_k1(const K1Params& k, int d_in, int device, cudaStream_t stream) {
  int rc = SPLITQ_ERR_UNSUPPORTED;
  if (k1v3_eligible(k, d_in) && !getenv("SPLITQ_K1_LEGACY")) {
    rc = k.x_dtype == IN_F16 ? launch_k1w<__half>(k, d_in, device, stream)
                             : launch_k1w<__nv_bfloat16>(k, d_in, device, stream);
    if (rc != SPLITQ_ERR_UNSUPPORTED) return rc;
  }
  if ((k.ld_main & 15) == 0) {
    rc = (k.c_main && k.d_main) ? launch_k1_dt<true>(k, d_in, stream)
                                : launch_k1_dt<false>(k, d_in, stream);
  }
  if (rc == SPLITQ_ERR_UNSUPPORTED) {
    k1_quantize_kernel<<<(unsigned)k.T, K1_THREADS, 0, stream>>>(k);
    CUDA_TRY(cudaGetLastError());
    return SPLITQ_OK;
  }
  return rc;
}

}  // namespace

namespace {
// int8 main codes (centred, in [-3, 3]) -> packed E2M1 codes for the
// kind::mxf4 GEMM: 16 code bytes per thread -> 8 bytes. Per 4 codes: the
// low 3 bits of each byte index an 8-entry byte table (PRMT), then nibble
// pairs are merged. Codes outside [-3, 3] (the don't-care bytes of outlier
// channels and row padding, which meet zero weights) map to finite values.
__global__ void fp4_pack_kernel(const int8_t* __restrict__ a, int64_t lda, uint8_t* __restrict__ o, int64_t ldo,
                                int rows, int chunks) {
  const int64_t n = (int64_t)rows * chunks;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / chunks, c = i - r * chunks;
    const uint4 w = *reinterpret_cast<const uint4*>(a + r * lda + 16 * c);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t t = ws[q] & 0x07070707u;
      const uint32_t x = t | (t >> 4);
      const uint32_t sel = (x & 0xFFu) | ((x >> 8) & 0xFF00u);
      const uint32_t nib = __byte_perm(0x05040200u, 0x0A0C0D00u, sel);  // E2M1 of 0,1,2,3 | -3,-2,-1
      const uint32_t y = nib | (nib >> 4);
      h[q] = (y & 0xFFu) | ((y >> 8) & 0xFF00u);
    }
    *reinterpret_cast<uint2*>(o + r * ldo + 8 * c) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
  }
}

int prof_record(splitq_layer_s* L, cudaStream_t stream) {
  if (L->ev_used == L->ev_pool.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    L->ev_pool.push_back(e);
  }
  CUDA_TRY(cudaEventRecord(L->ev_pool[L->ev_used++], stream));
  return SPLITQ_OK;
}
}  // namespace

extern "C" {

int splitq_forward(splitq_layer_t L, const void* x, int x_dtype, int64_t x_ld, const uint8_t* tags,
                   int64_t T, void* y, int y_dtype, int64_t y_ld, void* ws, size_t ws_bytes,
                   void* stream_, int flags) {
  if (!L || !x || !tags || !y || !ws) return fail(SPLITQ_ERR_INVALID, "null argument");
  if (T <= 0) return fail(SPLITQ_ERR_INVALID, "batch must contain at least one token");
  if (T > (int64_t)1 << 30) return fail(SPLITQ_ERR_INVALID, "too many tokens");
  if (x_dtype < 0 || x_dtype > 3) return fail(SPLITQ_ERR_INVALID, "bad x dtype");
  if (x_ld < L->d_in) return fail(SPLITQ_ERR_INVALID, "batch width does not match partition dim");
  const bool raw = (flags & SPLITQ_FWD_RAW) != 0;
  if (!raw && (y_dtype != SPLITQ_F32 && y_dtype != SPLITQ_F16 && y_dtype != SPLITQ_BF16))
    return fail(SPLITQ_ERR_INVALID, "bad y dtype");
  if (y_ld < L->d_out) return fail(SPLITQ_ERR_INVALID, "y leading dimension too small");
  // the layer's device is current for the call (its side stream, the
  // launches); the caller's is restored on return
  struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int d) {
      if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
      else prev = -1;
    }
    ~DeviceScope() {
      if (prev >= 0) cudaSetDevice(prev);
    }
  } device_scope(L->device);
  splitq_ws_layout_t W;
  int rc = splitq_workspace_layout(L, T, &W);
  if (rc) return rc;
  if ((int64_t)ws_bytes < W.total_bytes)
    return fail(SPLITQ_ERR_INVALID, "workspace too small (%zu < %lld)", ws_bytes,
                (long long)W.total_bytes);
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0)
    return fail(SPLITQ_ERR_INVALID, "workspace must be 256-byte aligned");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  auto at = [&](int64_t off) -> void* { return off < 0 ? nullptr : base + off; };
  int* err = (int*)at(W.status);
  int* n_text = (int*)at(W.n_text);
  int* text_idx = (int*)at(W.text_idx);
  int* text_rows = (int*)at(W.text_rows);

  const bool prof = (flags & SPLITQ_FWD_PROFILE) != 0;
  if (prof && (rc = prof_record(L, stream))) return rc;
  // decode-sized calls: CUDA-core / warp-MMA GEMV kernels (gemv_decode.cuh)
  const bool gv_packed = L->bp_main && !raw_unpacked(flags);
  const bool gv = T <= gemv_max_rows() &&
                  gv_fits(T, gv_packed, gv_packed ? L->ld_main / 2 : L->ld_main, (int)L->k_lr) &&
                  gv_fits(T, false, L->ld_main, 0);
  // status word + MAC row count (+ the GEMV LR1 split-K partials and counters)
  CUDA_TRY(cudaMemsetAsync(err, 0, 32 + (gv ? gv_scratch_bytes(L) : 0), stream));

  K1Params k{};
  k.x = x;
  k.x_dtype = x_dtype;
  k.ldx = x_ld;
  k.T = (int)T;
  k.c_main = L->c_main;
  k.d_main = L->d_main;
  k.d_main32 = L->k3_ok ? L->d_main32 : nullptr;
  k.d_main_lo32 = L->k3_ok && !getenv("SPLITQ_K1_NO_COMP") ? L->d_main_lo32 : nullptr;
  k.tags = tags;
  k.n_main = (int)L->k_nat;
  k.ld_main = (int)L->ld_main;
  k.act = L->act;
  k.aux = L->aux;
  k.a_main = (int8_t*)at(W.a_main);
  k.s_main = (double*)at(W.s_main);
  k.sf_main = (float*)at(W.sf_main);
  k.zp_main = (int*)at(W.zp_main);
  k.lrs_main = (float*)at(W.lrs_main);
  k.rho = (float*)at(W.rho);
  k.c_text = L->c_text;
  k.d_text = L->d_text;
  k.n_text = (int)L->n_text;
  k.ld_text = (int)L->ld_text;
  k.a_text = (int8_t*)at(W.a_text);
  k.s_text = (double*)at(W.s_text);
  k.sf_text = (float*)at(W.sf_text);
  k.zp_text = (int*)at(W.zp_text);
  k.c_vis = L->c_vis;
  k.d_vis = L->d_vis;
  k.n_vis = (int)L->n_vis;
  k.ld_vis = (int)L->ld_vis;
  k.a_vis = (int8_t*)at(W.a_vision);
  k.s_vis = (double*)at(W.s_vision);
  k.sf_vis = (float*)at(W.sf_vision);
  k.zp_vis = (int*)at(W.zp_vision);
  k.use_mac = L->use_mac;
  k.text_idx = text_idx;
  k.a_mac = (int8_t*)at(W.a_mac);
  k.s_mac = (double*)at(W.s_mac);
  k.zp_mac = (int*)at(W.zp_mac);
  k.lrs_mac = (float*)at(W.lrs_mac);
  k.lr_a = (__half*)at(W.lr_a);
  k.k_lr = (int)L->k_lr;
  k.lr_off_t = (int)L->off_t;
  k.lr_off_v = (int)L->off_v;
  k.lr_off_s = (int)L->off_s;
  k.kt16 = (int)L->kt16;
  k.kv16 = (int)L->kv16;
  k.err = err;
  if (k1v3_eligible(k, (int)L->d_in) && !getenv("SPLITQ_K1_LEGACY")) {
    // K1w claims the compact MAC rows itself (text_rows[slot] = row, order-free)
    k.mac_count = n_text;
    k.mac_rows = text_rows;
    k.text_idx = nullptr;
  } else {
    compact_text_rows_kernel<<<1, 1024, 0, stream>>>(tags, (int)T, text_idx, text_rows, n_text, err);
    CUDA_TRY(cudaGetLastError());
  }
  {
    NvtxRange r("splitq.K1");
    if ((rc = launch_k1(k, (int)L->d_in, L->device, stream))) return rc;
  }
  // A2 x W3 / W2 prefill: the main GEMM on kind::mxf4 from an E2M1 copy of the codes
  static const long packed_max_rows = getenv("SPLITQ_PACKED_MAX_ROWS")
                                          ? atol(getenv("SPLITQ_PACKED_MAX_ROWS")) : 2048;
  const bool mxf4 = L->bf4_main && W.a_main_fp4 >= 0 && !gv && !use_swap(T) && T > packed_max_rows &&
                    !getenv("SPLITQ_NO_MXF4");
  if (mxf4) {
    const int chunks = (int)(L->ld_main / 16);
    const int64_t n = T * chunks;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8L * sm_count(L->device));
    fp4_pack_kernel<<<blocks, 256, 0, stream>>>((const int8_t*)at(W.a_main), L->ld_main,
                                                (uint8_t*)at(W.a_main_fp4), L->ld_main / 2, (int)T, chunks);
    CUDA_TRY(cudaGetLastError());
  }
  if (prof && (rc = prof_record(L, stream))) return rc;

  __half* lr_a = (__half*)at(W.lr_a);

  // ---- low-rank first stages: fp16 columns of the auxiliary operand
  cudaStream_t lr_stream = stream;  // the LR1 launches' stream (the MAC one may fork)
  auto lr1 = [&](const void* a_codes, bool a_signed, const int8_t* bu, const float* su,
                 const int* csu, int64_t r, const float* row_s, const int* row_zp,
                 const int* m_count, const int* row_map, int64_t col_off, int64_t lo_off,
                 GvPlan* plan = nullptr) -> int {
    GemmLaunch g{};
    const bool sw = use_swap(T);
    g.p.M = (int)T;
    g.p.m_count = m_count;
    g.p.N = (int)r;
    g.p.swap = sw;
    g.p.bn = sw ? swap_bn(T) : tile_n(r, false);
    g.p.k_main = (int)L->k_nat;
    g.p.idesc_main = sw ? make_idesc(2, 1, a_signed ? 1u : 0u, G2_BM, g.p.bn) : idesc_i8(a_signed, g.p.bn);
    g.p.mode = G2_LR1;
    g.p.row_s = row_s;
    g.p.row_zp = row_zp;
    g.p.col_s = su;
    g.p.col_cs = csu;
    g.p.out = lr_a;
    g.p.ldo = L->k_lr;
    g.p.col_off = (int)col_off;
    g.p.lo_off = (int)lo_off;
    g.p.row_map = row_map;
    g.p.err = err;
    if (gv) {
      GvArgs a{};
      a.a = (const int8_t*)a_codes;
      a.lda = L->ld_main;
      a.a_bytes = L->ld_main;
      uint8_t* scr = base + W.status + 32;  // zeroed with the status block
      const bool mac = row_map != nullptr;
      a.red = reinterpret_cast<int*>(scr) + (mac ? GV_MAX_ROWS * L->r_s : 0);
      a.cnt = reinterpret_cast<unsigned*>(scr) + GV_MAX_ROWS * (L->r_s + L->r_c) +
              (mac ? 4 * ((L->r_s + 15) / 16) : 0);
      if (plan) return gv_plan(*plan, g.p, a, (int)T, bu, L->ld_main, nullptr, false, true, L->device);
      return launch_gv(g.p, a, (int)T, bu, L->ld_main, nullptr, false, a_signed, true, L->device, stream);
    }
    // swap-AB: the A slot (128 rows per CTA) takes the weights, B the token rows
    bool ok = map_i8(&g.maps.a, a_codes, T, L->k_nat, L->ld_main, sw ? g.p.bn / 2 : 128) &&
              map_i8(&g.maps.b, bu, r, L->k_nat, L->ld_main, sw ? 128 : g.p.bn / 2);
    g.maps.xa = g.maps.xb = g.maps.a;
    if (!ok) return fail(SPLITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (LR1)");
    // the CWS and MAC stages may run concurrently: each its own split-K slices
    const int64_t so = row_map ? lr1_scratch_off(L, T) : 0;
    const int64_t sb = row_map ? W.acc_scratch_bytes - so : std::min(W.acc_scratch_bytes, lr1_scratch_off(L, T));
    return launch_gemm(g, L->device, T, lr_stream, W.acc_scratch >= 0 && sb > 0 ? base + W.acc_scratch + so : nullptr,
                       sb);
  };
  NvtxRange nv_lr1("splitq.LR1");
  if (gv && L->r_s && L->r_c) {  // decode: both first stages in one launch
    GvPlan ps, pc;
    if ((rc = lr1(at(W.a_main), L->act.centered, L->b_us, L->s_us, L->cs_us, L->r_s,
                  (const float*)at(W.lrs_main), L->act.centered ? nullptr : (const int*)at(W.zp_main),
                  nullptr, nullptr, L->off_s, L->r_s8, &ps)) ||
        (rc = lr1(at(W.a_mac), L->aux.centered, L->b_uc, L->s_uc, L->cs_uc, L->r_c,
                  (const float*)at(W.lrs_mac), L->aux.centered ? nullptr : (const int*)at(W.zp_mac),
                  n_text, text_rows, L->off_c, 0, &pc)) ||
        (rc = launch_gv_pair(ps, L->act.centered, pc, L->aux.centered, (int)T, L->device, stream)))
      return rc;
  } else {
  // both first stages: the MAC one forks onto the layer's side stream (the
  // two are independent; with few tiles each they share the SMs)
  const bool fork = L->r_s && L->r_c && !getenv("SPLITQ_LR1_SERIAL");
  // the fork ... join enqueue sequence holds the layer's lock: host threads
  // sharing the layer must not interleave records of the shared events
  std::unique_lock<std::mutex> side_lock(L->side_mu, std::defer_lock);
  if (fork) {
    side_lock.lock();
    if (!L->side) {
      CUDA_TRY(cudaEventCreateWithFlags(&L->fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&L->join, cudaEventDisableTiming));
      CUDA_TRY(cudaStreamCreateWithFlags(&L->side, cudaStreamNonBlocking));
    }
    CUDA_TRY(cudaEventRecord(L->fork, stream));
    CUDA_TRY(cudaStreamWaitEvent(L->side, L->fork, 0));
  }
  if (L->r_s &&
      (rc = lr1(at(W.a_main), L->act.centered, L->b_us, L->s_us, L->cs_us, L->r_s,
                (const float*)at(W.lrs_main), L->act.centered ? nullptr : (const int*)at(W.zp_main),
                nullptr, nullptr, L->off_s, L->r_s8)))
    return rc;
  if (fork) lr_stream = L->side;
  if (L->r_c &&
      (rc = lr1(at(W.a_mac), L->aux.centered, L->b_uc, L->s_uc, L->cs_uc, L->r_c,
                (const float*)at(W.lrs_mac), L->aux.centered ? nullptr : (const int*)at(W.zp_mac),
                n_text, text_rows, L->off_c, 0)))
    return rc;
  if (fork) {
    lr_stream = stream;
    CUDA_TRY(cudaEventRecord(L->join, L->side));
    CUDA_TRY(cudaStreamWaitEvent(stream, L->join, 0));
    side_lock.unlock();
  }
  }
  if (prof && (rc = prof_record(L, stream))) return rc;

  // ---- split GEMM: int8 main GEMM + fp16 auxiliary GEMM + merge epilogue
  nv_lr1.next("splitq.K2");
  GemmLaunch g{};
  const bool sw = use_swap(T);  // decode-sized: 256-row tiles over output channels
  g.p.M = (int)T;
  g.p.N = (int)L->d_out;
  g.p.swap = sw;
  g.p.bn = sw ? swap_bn(T) : tile_n(L->d_out, L->k_lr > 0);
  g.p.k_main = (int)L->k_nat;
  g.p.k_aux = (int)L->k_lr;
  g.p.idesc_main = sw ? make_idesc(2, 1, L->act.centered ? 1u : 0u, G2_BM, g.p.bn)
                      : idesc_i8(L->act.centered, g.p.bn);
  g.p.idesc_aux = idesc_f16(g.p.bn);
  g.p.mode = raw ? G2_RAW : G2_SPLIT;
  g.p.out_dtype = y_dtype == SPLITQ_F32 ? G2_F32 : y_dtype == SPLITQ_F16 ? G2_F16 : G2_BF16;
  g.p.row_s = (const float*)at(W.sf_main);
  g.p.row_zp = L->act.centered ? nullptr : (const int*)at(W.zp_main);
  g.p.row_rho = (const float*)at(W.rho);
  g.p.col_s = L->s_main;
  g.p.col_cs = L->cs_main;
  g.p.col_kappa = L->kappa;
  g.p.out = y;
  g.p.ldo = y_ld;
  // the fast epilogue: centred codes (no zero-point term) and |acc| < 2^22,
  // bounded by K x (q_max - q_min) x max |w| (or exact fp32 sums from mxf4)
  g.p.epi_fast = !raw && L->act.centered && !getenv("SPLITQ_EPI_SLOW") &&
                 (mxf4 || (double)L->ld_main * (double)(L->act.qmax - L->act.qmin) * (double)L->wmax < 4194304.0);
  if (raw) g.p.raw_aux = reinterpret_cast<float*>(reinterpret_cast<int*>(y) + T * y_ld);
  if (gv) {
    GvArgs a{};
    a.a = (const int8_t*)at(W.a_main);
    a.lda = L->ld_main;
    a.a_bytes = L->ld_main;
    a.xa = lr_a;
    const bool pk = gv_packed;
    if ((rc = launch_gv(g.p, a, (int)T, pk ? (const void*)L->bp_main : (const void*)L->b_main,
                        pk ? L->ld_main / 2 : L->ld_main, L->b_lr, pk, L->act.centered, false, L->device,
                        stream)))
      return rc;
    if (prof && (rc = prof_record(L, stream))) return rc;
    return SPLITQ_OK;
  }
  // box rows per CTA: the A slot holds 128 rows, the B slot bn / 2; with
  // swap-AB the weights take the A slot and the token rows the B slot
  if (mxf4) {  // E2M1 operands: K counted in bytes (64 codes per MMA); 3 bn TMEM columns + scale factors
    g.p.bn = std::min(g.p.bn, G2_BN);
    g.p.k_main = (int)(L->ld_main / 2);
    g.p.mxf4 = 1;
    g.p.idesc_main = make_idesc_mxf4(G2_BM, g.p.bn);
  }
  const uint32_t act_box = sw ? g.p.bn / 2 : 128, w_box = sw ? 128 : g.p.bn / 2;
  bool ok = mxf4 ? map_i8(&g.maps.a, at(W.a_main_fp4), T, L->ld_main / 2, L->ld_main / 2, act_box)
                 : map_i8(&g.maps.a, at(W.a_main), T, L->k_nat, L->ld_main, act_box);
  // Packed 4-bit weights pay where the GEMM streams weights (few token rows:
  // decode); for large token counts the kernel is tensor / SMEM-bandwidth
  // bound and the SMEM unpack traffic (+50% over the UMMA operand reads at
  // 256 x 128 tiles) costs more than it saves, so the int8 expansion is used.
  if (mxf4) {
    ok = ok && map_i8(&g.maps.b, L->bf4_main, L->d_out, L->ld_main / 2, L->ld_main / 2, w_box);
  } else if (L->bp_main && !raw_unpacked(flags) && T <= packed_max_rows) {
    g.p.packed_b = 1;
    ok = ok && make_map_2d(&g.maps.b, L->bp_main, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, L->d_out,
                           L->ld_main / 2, L->ld_main / 2, w_box, 64, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    ok = ok && map_i8(&g.maps.b, L->b_main, L->d_out, L->k_nat, L->ld_main, w_box);
  }
  g.maps.xa = g.maps.xb = g.maps.a;
  if (ok && L->k_lr)
    ok = map_f16(&g.maps.xa, lr_a, T, L->k_lr, L->k_lr, act_box) &&
         map_f16(&g.maps.xb, L->b_lr, L->d_out, L->k_lr, L->k_lr, w_box);
  if (!ok) return fail(SPLITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (split GEMM)");
  if ((rc = launch_gemm(g, L->device, T, stream, at(W.acc_scratch), W.acc_scratch_bytes))) return rc;
  if (prof && (rc = prof_record(L, stream))) return rc;
  return SPLITQ_OK;
}

// G2_TRACE builds: copy the phase stamps of the last GEMM launch (host buffer
// of 148 * 8 u64); returns the number of CTAs. Not part of the public ABI.
// KW_TRACE builds: the 16 phase clocks of the last K1 launch's first row
int splitq_debug_k1_trace(unsigned long long* out) {
  if (!k1w_trace_last) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(out, k1w_trace_last, 16 * 8, cudaMemcpyDeviceToHost);
  return 16;
}

int splitq_debug_gemm_trace(unsigned long long* out) {
  if (!g2_trace_last) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g2_trace_last, 148 * 8 * 8, cudaMemcpyDeviceToHost);
  return g2_trace_ctas;
}

int splitq_profile_read(splitq_layer_t L, double* stage_ms, int32_t* calls) {
  if (!L || !stage_ms) return fail(SPLITQ_ERR_INVALID, "null argument");
  for (int i = 0; i < 3; ++i) stage_ms[i] = 0.0;
  const size_t n = L->ev_used / 4;
  for (size_t c = 0; c < n; ++c) {
    cudaEvent_t* e = &L->ev_pool[4 * c];
    CUDA_TRY(cudaEventSynchronize(e[3]));
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, e[i], e[i + 1]));
      stage_ms[i] += ms;
    }
  }
  if (calls) *calls = (int32_t)n;
  L->ev_used = 0;
  return SPLITQ_OK;
}

int splitq_read_status(void* ws, void* stream_, int32_t* status_out) {
  if (!ws) return fail(SPLITQ_ERR_INVALID, "null workspace");
  int32_t st = 0;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  CUDA_TRY(cudaMemcpyAsync(&st, ws, sizeof(st), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  if (status_out) *status_out = st;
  if (st & SPLITQ_STATUS_NONFINITE) return fail(SPLITQ_ERR_DATA, "non-finite value in matrix");
  if (st & SPLITQ_STATUS_SCALE) return fail(SPLITQ_ERR_DATA, "scales must be positive");
  if (st & SPLITQ_STATUS_TAG) return fail(SPLITQ_ERR_DATA, "tags must be 0 (text) or 1 (vision)");
  if (st & SPLITQ_STATUS_LR_RANGE)
    return fail(SPLITQ_ERR_DATA, "low-rank operand exceeded the fp16 range");
  return SPLITQ_OK;
}

int splitq_quantize_rows(const void* x, int x_dtype, int64_t x_ld, int64_t rows, int64_t cols,
                         splitq_qspec_t spec, int8_t* codes, int64_t codes_ld, double* scales,
                         int32_t* zero_points, int32_t* status, int32_t* centered_out,
                         void* stream_) {
  if (!x || !codes || !scales || !zero_points || !status)
    return fail(SPLITQ_ERR_INVALID, "null argument");
  if (rows <= 0 || cols <= 0) return fail(SPLITQ_ERR_INVALID, "empty matrix");
  if (codes_ld < cols || (codes_ld & 3)) return fail(SPLITQ_ERR_INVALID, "codes_ld must be >= cols and a multiple of 4");
  QSpecDev s;
  int rc = make_spec(spec, &s, "spec");
  if (rc) return rc;
  if (centered_out) *centered_out = s.centered;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), stream));
  K1Params k{};
  k.x = x;
  k.x_dtype = x_dtype;
  k.ldx = x_ld;
  k.T = (int)rows;
  k.n_main = (int)cols;
  k.ld_main = (int)codes_ld;
  k.act = s;
  k.aux = s;
  k.a_main = codes;
  k.s_main = scales;
  k.zp_main = zero_points;
  k.err = status;
  int device = 0;
  CUDA_TRY(cudaGetDevice(&device));
  return launch_k1(k, (int)cols, device, stream);
}

int splitq_gemm_i8(const int8_t* a, int64_t lda, int a_signed, const int8_t* b, int64_t ldb,
                   int32_t* c, int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream_) {
  if (!a || !b || !c) return fail(SPLITQ_ERR_INVALID, "null argument");
  if (m <= 0 || n <= 0 || k <= 0) return fail(SPLITQ_ERR_INVALID, "empty GEMM");
  if ((lda & 15) || (ldb & 15) || lda < k || ldb < k)
    return fail(SPLITQ_ERR_INVALID, "lda/ldb must be >= k and multiples of 16");
  int device = 0;
  CUDA_TRY(cudaGetDevice(&device));
  GemmLaunch g{};
  g.p.M = (int)m;
  g.p.N = (int)n;
  g.p.bn = tile_n(n, false);
  g.p.k_main = (int)k;
  g.p.idesc_main = idesc_i8(a_signed != 0, g.p.bn);
  g.p.mode = G2_RAW;
  g.p.out = c;
  g.p.ldo = ldc;
  bool ok = map_i8(&g.maps.a, a, m, k, lda, 128) && map_i8(&g.maps.b, b, n, k, ldb, g.p.bn / 2);
  g.maps.xa = g.maps.xb = g.maps.a;
  if (!ok) return fail(SPLITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return launch_gemm(g, device, m, reinterpret_cast<cudaStream_t>(stream_));
}

}  // extern "C"
