// Stage 1 of the split-linear forward: fused gather / smoothing / per-token
// quantization (K1) plus the text-row compaction that feeds the MAC branch.
//
// Bit-exactness contract with the reference (numpy float64):
//   z      = x[:, c_p] * d_p                    transform.py:94-103 (d_p = Transform.scale,
//                                               consumed as the host fp64 vector, F4b)
//   params = compute_params(z, PER_TOKEN spec)  quantizer.py:104-135
//   q      = clip(rha(z / S) + zp, qmin, qmax)  quantizer.py:146-155, rha = sign*floor(|v|+0.5)
//   x_hat  = (q - zp) * S ; e = (z - x_hat)[text rows]   layer.py:135-136, 157-160
// All of these are evaluated with explicitly-rounded fp64 intrinsics
// (__dmul_rn / __dsub_rn / __dadd_rn / __ddiv_rn) so the compiler cannot
// contract them into FMAs. The division z / S is replaced by z * (1 / S)
// except within a window around the rounding tie, where the exact IEEE
// quotient is recomputed; the two quotients differ by at most a couple of
// ulp, so the rounding decision is identical everywhere.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace splitq {

enum InDtype : int { IN_F16 = 0, IN_F32 = 1, IN_F64 = 2, IN_BF16 = 3 };

// error word bits (device), surfaced as ValueError by the host shim
enum ErrBits : int {
  ERR_NONFINITE = 1,    // "non-finite value in matrix" (tensor.py:39-40)
  ERR_SCALE_ZERO = 2,   // "scales must be positive" (quantizer.py:72-73)
  ERR_BAD_TAG = 4,      // "tags must be 0 (text) or 1 (vision)" (tensor.py:71-72)
  ERR_LR_RANGE = 8,     // low-rank fp16 operand out of range (build invariant broken)
};

struct QSpecDev {
  int qmin, qmax;
  int sym;
  int centered;  // 1: store (q - zp) as s8; 0: store q (u8, zero point applied in GEMM epilogue)
};

__device__ __forceinline__ double load_x(const void* x, int dt, int64_t idx) {
  switch (dt) {
    case IN_F16: return (double)__half2float(reinterpret_cast<const __half*>(x)[idx]);
    case IN_F32: return (double)reinterpret_cast<const float*>(x)[idx];
    case IN_BF16: return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[idx]);
    default: return reinterpret_cast<const double*>(x)[idx];
  }
}

// sign(v) * floor(|v| + 0.5)  (quantizer.py:76-77), evaluated for v = m / S.
__device__ __forceinline__ double rha_quotient(double m, double S, double rS) {
  double v = __dmul_rn(m, rS);
  double a = fabs(v);
  const double f = a - floor(a);
  if (fabs(f - 0.5) < 1e-6) {  // near a tie: use the exact IEEE quotient
    v = __ddiv_rn(m, S);
    a = fabs(v);
  }
  const double r = floor(__dadd_rn(a, 0.5));
  return v < 0.0 ? -r : r;
}

__device__ __forceinline__ int quant_code(double m, double S, double rS, double zp, int qmin,
                                          int qmax) {
  double q = rha_quotient(m, S, rS) + zp;
  q = fmin(fmax(q, (double)qmin), (double)qmax);
  return (int)q;
}

// compute_params for one group (quantizer.py:118-135). Returns false when the
// scale is not positive (the reference raises ValueError).
__device__ __forceinline__ bool group_params(double lo, double hi, const QSpecDev& s, double* S,
                                             double* zp) {
  if (s.sym) {
    const double amax = fmax(fabs(lo), fabs(hi));
    *S = amax > 0.0 ? __ddiv_rn(amax, (double)s.qmax) : 1.0;
    *zp = 0.0;
  } else {
    double span = __dsub_rn(hi, lo);
    if (span == 0.0) {
      lo = fmin(lo, 0.0);
      hi = fmax(hi, 0.0);
      span = __dsub_rn(hi, lo);
    }
    *S = span > 0.0 ? __ddiv_rn(span, (double)(s.qmax - s.qmin)) : 1.0;
    double z = rha_quotient(-lo, *S, __ddiv_rn(1.0, *S));
    z = fmin(fmax(z, (double)s.qmin), (double)s.qmax);
    *zp = z;
  }
  return *S > 0.0;
}

__device__ __forceinline__ int8_t store_code(int q, int zp, const QSpecDev& s) {
  return s.centered ? (int8_t)(q - zp) : (int8_t)(uint8_t)q;
}

// ---------------------------------------------------------------- compaction
// text_idx[i] = position of row i among text rows (or -1), text_rows[c] = i.
// One CTA of 1024 threads, each owning a contiguous run of rows.
static __global__ void compact_text_rows_kernel(const uint8_t* __restrict__ tags, int T,
                                         int* __restrict__ text_idx, int* __restrict__ text_rows,
                                         int* __restrict__ n_text, int* __restrict__ err) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  const int per = (T + 1024 * 64 - 1) / (1024 * 64) * 64;  // rows per thread per sweep
  for (int base = 0; base < T; base += per * 1024) {
    const int r0 = base + tid * per;
    int cnt = 0, bad = 0;
    for (int i = 0; i < per; ++i) {
      const int r = r0 + i;
      if (r < T) {
        const uint8_t t = tags[r];
        cnt += (t == 0);
        bad |= (t > 1);
      }
    }
    if (bad) atomicOr(err, ERR_BAD_TAG);
    // block exclusive scan of cnt
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = warp_sums[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += v;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    int pos = carry + (warp ? warp_sums[warp - 1] : 0) + incl - cnt;
    for (int i = 0; i < per; ++i) {
      const int r = r0 + i;
      if (r < T) {
        if (tags[r] == 0) {
          text_idx[r] = pos;
          text_rows[pos] = r;
          ++pos;
        } else {
          text_idx[r] = -1;
        }
      }
    }
    __syncthreads();
    if (tid == 1023) carry += warp_sums[31];
    __syncthreads();
  }
  if (tid == 0) *n_text = carry;
}

// ---------------------------------------------------------------- K1
struct K1Params {
  const void* x;
  int x_dtype;
  int64_t ldx;
  int T;
  // main path
  const int* c_main;
  const double* d_main;
  const float* d_main32;  // fp32 copy of d_main (K1 v3)
  const float* d_main_lo32;  // fl32(d_main - d_main32) (K1w compensated MAC pass; may be null)
  const uint8_t* tags;    // modality tags (K1 v3 validates them)
  int n_main;
  int ld_main;  // row stride (bytes) of the main / MAC code matrices
  QSpecDev act, aux;
  int8_t* a_main;
  double* s_main;
  float* sf_main;
  int* zp_main;
  float* lrs_main;  // S / rho
  float* rho;       // 2^floor(log2 S)
  // outliers
  const int* c_text;
  const double* d_text;
  int n_text, ld_text;
  int8_t* a_text;
  double* s_text;
  float* sf_text;
  int* zp_text;
  const int* c_vis;
  const double* d_vis;
  int n_vis, ld_vis;
  int8_t* a_vis;
  double* s_vis;
  float* sf_vis;
  int* zp_vis;
  // MAC residual (compact text rows)
  int use_mac;
  const int* text_idx;
  int* mac_count;  // K1w: MAC slots are claimed with an atomic (order-free; rows independent)
  int* mac_rows;   //      mac_rows[slot] = row
  unsigned long long* trace;  // KW_TRACE builds: phase clocks of the first row of CTA 0
  int kw_stage_d;  // K1w row groups: stage the fp32 smoothing factors in SMEM with the row
  int8_t* a_mac;
  double* s_mac;
  int* zp_mac;
  float* lrs_mac;  // S_e / rho(row)
  // fp16 auxiliary GEMM operand rows (k_lr per row): the outlier hi/lo
  // segments are written here, the low-rank columns [lr_off_s, k_lr) cleared
  __half* lr_a;
  int k_lr;
  int lr_off_t, lr_off_v, lr_off_s;  // segment offsets (elements)
  int kt16, kv16;                     // outlier K rounded to 16
  int* err;
};

constexpr int K1_THREADS = 256;

// z = x[row, c_main[k]] * d_main[k]; a null index table means identity
// columns and a null scale vector means no smoothing (plain quantize_rows).
__device__ __forceinline__ double main_z(const K1Params& p, int64_t xrow, int k) {
  const double x = load_x(p.x, p.x_dtype, xrow + (p.c_main ? p.c_main[k] : k));
  return p.d_main ? __dmul_rn(x, p.d_main[k]) : x;
}

__device__ __forceinline__ void block_minmax(double& lo, double& hi, double* red) {
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    red[warp] = lo;
    red[8 + warp] = hi;
  }
  __syncthreads();
  lo = red[0];
  hi = red[8];
#pragma unroll
  for (int w = 1; w < K1_THREADS / 32; ++w) {
    lo = fmin(lo, red[w]);
    hi = fmax(hi, red[8 + w]);
  }
}

// Quantize one outlier path (n <= a few hundred columns) with one warp.
static __device__ void outlier_row(const K1Params& p, int row, const int* cols, const double* d, int n,
                            int ld, int8_t* codes, double* s_out, float* sf_out, int* zp_out) {
  const int lane = threadIdx.x & 31;
  double lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  for (int k = lane; k < n; k += 32) {
    const double x = load_x(p.x, p.x_dtype, (int64_t)row * p.ldx + cols[k]);
    const double z = __dmul_rn(x, d[k]);
    bad |= !isfinite(z);
    lo = fmin(lo, z);
    hi = fmax(hi, z);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) atomicOr(p.err, ERR_NONFINITE);
    return;
  }
  double S, zp;
  const bool ok = group_params(lo, hi, p.aux, &S, &zp);
  if (!ok) {
    if (lane == 0) atomicOr(p.err, ERR_SCALE_ZERO);
    S = 1.0;
  }
  const double rS = __ddiv_rn(1.0, S);
  int8_t* out = codes + (int64_t)row * ld;
  for (int k = lane; k < ld; k += 32) {
    int8_t c = 0;
    if (k < n) {
      const double x = load_x(p.x, p.x_dtype, (int64_t)row * p.ldx + cols[k]);
      const double z = __dmul_rn(x, d[k]);
      c = store_code(quant_code(z, S, rS, zp, p.aux.qmin, p.aux.qmax), (int)zp, p.aux);
    }
    out[k] = c;
  }
  if (lane == 0) {
    s_out[row] = S;
    sf_out[row] = (float)S;
    zp_out[row] = (int)zp;
  }
}

static __global__ void __launch_bounds__(K1_THREADS) k1_quantize_kernel(const K1Params p) {
  __shared__ double red[16];
  __shared__ double sh_S, sh_zp;
  const int row = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t xrow = (int64_t)row * p.ldx;

  // ---- pass 1: z = x * d over the main channels, row min / max
  double lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  for (int k = tid; k < p.n_main; k += K1_THREADS) {
    const double z = main_z(p, xrow, k);
    bad |= !isfinite(z);
    lo = fmin(lo, z);
    hi = fmax(hi, z);
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) atomicOr(p.err, ERR_NONFINITE);
    return;
  }
  block_minmax(lo, hi, red);
  if (tid == 0) {
    double S, zp;
    if (!group_params(lo, hi, p.act, &S, &zp)) {
      atomicOr(p.err, ERR_SCALE_ZERO);
      S = 1.0;
    }
    sh_S = S;
    sh_zp = zp;
    p.s_main[row] = S;
    if (p.sf_main) p.sf_main[row] = (float)S;
    p.zp_main[row] = (int)zp;
    if (p.rho) {
      int e;
      frexp(S, &e);  // S = m * 2^e, m in [0.5, 1)
      const double rho = ldexp(1.0, e - 1);
      p.rho[row] = (float)rho;
      p.lrs_main[row] = (float)(S / rho);
    }
  }
  __syncthreads();
  const double S = sh_S, zp = sh_zp, rS = __ddiv_rn(1.0, S);
  const int cidx = p.use_mac ? p.text_idx[row] : -1;
  const bool mac = cidx >= 0;

  // ---- pass 2: main codes (+ MAC residual range on text rows)
  int8_t* arow = p.a_main + (int64_t)row * p.ld_main;
  double elo = INFINITY, ehi = -INFINITY;
  for (int k0 = tid * 4; k0 < p.ld_main; k0 += K1_THREADS * 4) {
    uint32_t packed = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u;
      if (k < p.n_main) {
        const double z = main_z(p, xrow, k);
        const int q = quant_code(z, S, rS, zp, p.act.qmin, p.act.qmax);
        packed |= (uint32_t)(uint8_t)store_code(q, (int)zp, p.act) << (8 * u);
        if (mac) {
          const double xh = __dmul_rn((double)q - zp, S);
          const double e = __dsub_rn(z, xh);
          elo = fmin(elo, e);
          ehi = fmax(ehi, e);
        }
      }
    }
    *reinterpret_cast<uint32_t*>(arow + k0) = packed;
  }

  // ---- outlier paths (one warp each), independent of the main path
  const int warp = tid >> 5;
  if (warp == 0 && p.n_text > 0)
    outlier_row(p, row, p.c_text, p.d_text, p.n_text, p.ld_text, p.a_text, p.s_text, p.sf_text,
                p.zp_text);
  if (warp == 1 && p.n_vis > 0)
    outlier_row(p, row, p.c_vis, p.d_vis, p.n_vis, p.ld_vis, p.a_vis, p.s_vis, p.sf_vis,
                p.zp_vis);
  // ---- clear this row of the low-rank operand (LR1 passes fill valid columns)
  if (p.k_lr > 0) {
    uint4* lr = reinterpret_cast<uint4*>(p.lr_a + (int64_t)row * p.k_lr);
    for (int i = tid; i < p.k_lr / 8; i += K1_THREADS) lr[i] = make_uint4(0, 0, 0, 0);
  }
  if (!mac) return;  // block-uniform

  // ---- pass 3 (text rows, MAC on): residual codes e = z - x_hat at aux bits
  block_minmax(elo, ehi, red);
  if (tid == 0) {
    double Se, zpe;
    if (!group_params(elo, ehi, p.aux, &Se, &zpe)) {
      atomicOr(p.err, ERR_SCALE_ZERO);
      Se = 1.0;
    }
    sh_S = Se;  // safe: every thread read S / zp before the barrier in block_minmax
    sh_zp = zpe;
    p.s_mac[cidx] = Se;
    p.zp_mac[cidx] = (int)zpe;
    int e;
    frexp(S, &e);
    p.lrs_mac[cidx] = (float)(Se / ldexp(1.0, e - 1));
  }
  __syncthreads();
  const double Se = sh_S, zpe = sh_zp, rSe = __ddiv_rn(1.0, Se);
  int8_t* erow = p.a_mac + (int64_t)cidx * p.ld_main;
  for (int k0 = tid * 4; k0 < p.ld_main; k0 += K1_THREADS * 4) {
    uint32_t packed = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u;
      if (k < p.n_main) {
        const double z = main_z(p, xrow, k);
        const int q = quant_code(z, S, rS, zp, p.act.qmin, p.act.qmax);
        const double e = __dsub_rn(z, __dmul_rn((double)q - zp, S));
        const int qe = quant_code(e, Se, rSe, zpe, p.aux.qmin, p.aux.qmax);
        packed |= (uint32_t)(uint8_t)store_code(qe, (int)zpe, p.aux) << (8 * u);
      }
    }
    *reinterpret_cast<uint32_t*>(erow + k0) = packed;
  }
}

}  // namespace splitq
