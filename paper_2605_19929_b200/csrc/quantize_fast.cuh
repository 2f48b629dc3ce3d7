// K1 (throughput version): fused gather / smoothing / per-token quantization
// and MAC residual codes, one CTA per block of rows.
//
// Same exactness contract as quantize.cuh (reference quantizer.py:104-155,
// transform.py:94-103, layer.py:135-136 / 157-160), restructured for HBM
// speed on sm_100a:
//   * the x row is staged in SMEM with double-buffered 16-B cp.async, so the
//     gather x[c_main[k]] is an SMEM read and HBM is read exactly once;
//   * z = x * d (fp64) stays in registers (EPT per thread) across the
//     min/max pass, the code pass and the MAC residual pass;
//   * rounding: v = z * (1/S) and RNE(|v|) via the 1.5*2^52 magic constant
//     (5 fp64 ops); within 1e-6 of a .5 tie the exact reference expression
//     floor(fl(|z / S| + 0.5)) is evaluated instead, so codes are identical;
//   * x_hat = (q - zp) * S comes from a per-row table of the <= 256 code
//     levels (one fp64 product per level, the reference's rounding).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "quantize.cuh"
#include "sm100_ptx.cuh"

namespace splitq {

constexpr double K1_MAGIC = 6755399441055744.0;  // 1.5 * 2^52

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<__half>(__half v) { return (double)__half2float(v); }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return (double)__bfloat162float(v);
}
template <>
__device__ __forceinline__ double to_f64<float>(float v) { return (double)v; }
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }

// Exact reference expression clip(rha(m / S) + zp) (quantizer.py:76-77,
// 152-154), kept out of line so the unrolled element loops stay small.
static __device__ __noinline__ int quant_exact(double m, double S, double zp_qmin_qmax_packed_unused,
                                        int zp, int qmin, int qmax) {
  const double ve = __ddiv_rn(m, S);
  const int n = (int)floor(__dadd_rn(fabs(ve), 0.5));
  return min(max((ve < 0.0 ? -n : n) + zp, qmin), qmax);
}

__device__ __forceinline__ void warp_minmax(double& lo, double& hi) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
}

constexpr int K1G_WARPS = 8;  // warps per CTA; a row group is G of them

// Round-to-nearest code with the zero point folded into the magic constant:
// t = v + (1.5 * 2^52 + zp) puts RN(v) + zp in the low word. Outside a 1e-6
// window around .5 ties RN equals the reference's half-away rounding
// (quantizer.py:76-77); inside it `tie` is set and the caller re-evaluates
// exactly. Valid for |v| < 2^29 (the caller guarantees it per row).
__device__ __forceinline__ int quant_rn(double m, double rS, double cz, bool& tie) {
  const double v = __dmul_rn(m, rS);
  const double t = __dadd_rn(v, cz);
  const double r = __dsub_rn(t, cz);  // RN(v), exact
  tie |= fabs(__dsub_rn(v, r)) > 0.499999;
  return __double2loint(t);
}

struct RowParams {
  double S, rS, cz;
  int zp, qmin, qmax;
  bool safe;  // |z / S| < 2^29 over the row: quant_rn is valid
};

__device__ __forceinline__ RowParams make_row_params(double lo, double hi, const QSpecDev& s,
                                                     bool* ok) {
  RowParams r;
  double zpd;
  *ok = group_params(lo, hi, s, &r.S, &zpd);
  if (!*ok) r.S = 1.0;
  r.rS = __ddiv_rn(1.0, r.S);
  r.zp = (int)zpd;
  r.cz = K1_MAGIC + zpd;
  r.qmin = s.qmin;
  r.qmax = s.qmax;
  r.safe = fmax(fabs(lo), fabs(hi)) * r.rS < 536870912.0;  // 2^29
  return r;
}

__device__ __forceinline__ int quant_row(double m, const RowParams& r, bool& tie) {
  int q;
  if (r.safe) {
    q = quant_rn(m, r.rS, r.cz, tie);
  } else {  // exact reference expression (rows with a huge offset relative to their span)
    q = quant_exact(m, r.S, 0.0, r.zp, r.qmin, r.qmax);
  }
  return min(max(q, r.qmin), r.qmax);
}

template <int G>
__device__ __forceinline__ void group_sync(int g) {
  if (G == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(32 * G) : "memory");
  }
}

// min / max over the row group (warp shuffles, then SMEM across its warps)
template <int G>
__device__ __forceinline__ void group_minmax(double& lo, double& hi, double* red, int g, int wg) {
  warp_minmax(lo, hi);
  if (G > 1) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
      red[2 * wg] = lo;
      red[2 * wg + 1] = hi;
    }
    group_sync<G>(g);
#pragma unroll
    for (int w = 0; w < G; ++w) {
      const double l2 = red[2 * w], h2 = red[2 * w + 1];
      lo = l2 < lo ? l2 : lo;
      hi = h2 > hi ? h2 : hi;
    }
    group_sync<G>(g);  // red is reused by the next reduction
  }
}

// ---- outlier paths in two steps: params (warp-level), then codes + the fp16
// hi/lo segments of the auxiliary GEMM operand. a = (q - zp) * (S_p / rho) is
// exact in fp64; a = a_hi + a_lo with a_hi = fp16(a), a_lo = fp16(a - a_hi).
template <typename T>
__device__ void outlier_params(const K1Params& p, const T* xs, const int* cols, const double* d,
                               int n, RowParams& rp, bool& ok, bool& bad) {
  const int lane = threadIdx.x & 31;
  double lo = INFINITY, hi = -INFINITY;
  bool nan = false;
  for (int k = lane; k < n; k += 32) {
    const double z = __dmul_rn(to_f64(xs[cols[k]]), d[k]);
    nan |= z != z;
    lo = z < lo ? z : lo;
    hi = z > hi ? z : hi;
  }
  warp_minmax(lo, hi);
  bad = __any_sync(0xffffffffu, nan) || !isfinite(lo) || !isfinite(hi);
  rp = make_row_params(bad ? 0.0 : lo, bad ? 0.0 : hi, p.aux, &ok);
}

template <typename T>
__device__ void outlier_codes(const K1Params& p, int row, const T* xs, const int* cols,
                              const double* d, int n, int ld, int8_t* codes, const RowParams& rp,
                              double fac, int seg_off, int k16, int k0 = -1, int step = 32,
                              const double* z0 = nullptr) {  // z of channel k0, if already formed
  int8_t* out = codes + (int64_t)row * ld;
  __half* seg = p.k_lr > 0 ? p.lr_a + (int64_t)row * p.k_lr + seg_off : nullptr;
  const int lim = max(ld, k16);
  for (int k = k0 < 0 ? (int)(threadIdx.x & 31) : k0; k < lim; k += step) {
    int c = 0;
    double a = 0.0;
    if (k < n) {
      const double z = z0 && k == k0 ? *z0 : __dmul_rn(to_f64(xs[cols[k]]), d[k]);
      bool tie = false;
      int q = quant_row(z, rp, tie);
      if (tie) q = quant_exact(z, rp.S, 0.0, rp.zp, rp.qmin, rp.qmax);
      c = p.aux.centered ? q - rp.zp : q;
      a = (double)(q - rp.zp) * fac;
    }
    if (k < ld) out[k] = (int8_t)c;
    if (seg && k < k16) {
      const __half hi = __double2half(a);
      const __half lo = __double2half(a - (double)__half2float(hi));
      seg[k] = hi;
      seg[k16 + k] = lo;
      seg[2 * k16 + k] = hi;
    }
  }
}

// raw-bit finiteness test per input type: max of |bits| >= inf pattern
template <typename T> struct InBits;
template <> struct InBits<__half> {
  static constexpr uint32_t inf = 0x7C00u;
  static __device__ __forceinline__ uint32_t absbits(__half v) { return __half_as_ushort(v) & 0x7FFFu; }
};
template <> struct InBits<__nv_bfloat16> {
  static constexpr uint32_t inf = 0x7F80u;
  static __device__ __forceinline__ uint32_t absbits(__nv_bfloat16 v) {
    return __bfloat16_as_ushort(v) & 0x7FFFu;
  }
};
template <> struct InBits<float> {
  static constexpr uint32_t inf = 0x7F800000u;
  static __device__ __forceinline__ uint32_t absbits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }
};
template <> struct InBits<double> {
  static constexpr uint32_t inf = 0x7FF00000u;
  static __device__ __forceinline__ uint32_t absbits(double v) {
    return (uint32_t)__double2hiint(v) & 0x7FFFFFFFu;
  }
};

// 4 main elements k0..k0+3 from the staged row; the gather tables are padded
// to ld_main with (index 0, scale NaN), so no bounds checks. Without a gather
// (quantize_rows) elements past n_main become NaN.
template <typename T, bool GATHER>
__device__ __forceinline__ void gather4_pad(const K1Params& p, const T* xs, int k0,
                                            double (&z)[4], uint32_t& xbits) {
  if (GATHER) {
    const int4 c4 = __ldg(reinterpret_cast<const int4*>(p.c_main + k0));
    const double2 d0 = __ldg(reinterpret_cast<const double2*>(p.d_main + k0));
    const double2 d1 = __ldg(reinterpret_cast<const double2*>(p.d_main + k0 + 2));
    const int c[4] = {c4.x, c4.y, c4.z, c4.w};
    const double d[4] = {d0.x, d0.y, d1.x, d1.y};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const T xv = xs[c[u]];
      xbits = max(xbits, InBits<T>::absbits(xv));
      z[u] = __dmul_rn(to_f64(xv), d[u]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = k0 + u < p.n_main;
      const T xv = xs[in ? k0 + u : 0];
      xbits = max(xbits, in ? InBits<T>::absbits(xv) : 0u);
      z[u] = in ? to_f64(xv) : __longlong_as_double(0x7ff8000000000000ll);
    }
  }
}

// One row per group of G warps (K1G_WARPS / G rows per CTA). The row is
// staged into SMEM with one TMA bulk copy (cp.async.bulk) when it is 16-B
// aligned, then every pass gathers from SMEM.
template <typename T, bool GATHER, int G>
__global__ void __launch_bounds__(K1G_WARPS * 32) k1_group_kernel(const K1Params p, int d_in) {
  constexpr int NG = K1G_WARPS / G;  // row groups per CTA
  extern __shared__ __align__(128) uint8_t k1g_smem[];
  const int row_bytes = (d_in * (int)sizeof(T) + 127) / 128 * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / G, wg = warp % G;  // group, warp within group
  const int tg = wg * 32 + lane;          // thread within group
  constexpr int NTG = 32 * G;
  uint8_t* base = k1g_smem + g * (row_bytes + 256 * 8 + 2 * G * 8 + 128);
  T* xs = reinterpret_cast<T*>(base);
  double* xh = reinterpret_cast<double*>(base + row_bytes);
  double* red = xh + 256;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 2 * G);
  double* oscale = reinterpret_cast<double*>(mbar + 1);  // [2]: S_text, S_vision of the row
  int* oflag = reinterpret_cast<int*>(oscale + 2);        // [2]: outlier path failed
  const int row = blockIdx.x * NG + g;
  if (row >= p.T) return;  // whole group exits together
  const T* xrow = reinterpret_cast<const T*>(p.x) + (int64_t)row * p.ldx;
  const int n_main = p.n_main, ld = p.ld_main;

  // ---- stage the row
  const uint32_t bytes = (uint32_t)(d_in * sizeof(T));
  const bool bulk = (bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(xrow) & 15) == 0);
  if (bulk) {
    if (tg == 0) {
      mbar_init(mbar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(mbar, bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(xs)),
          "l"(xrow), "r"(bytes), "r"(smem_u32(mbar))
          : "memory");
    }
    group_sync<G>(g);  // barrier initialised before anyone waits on it
    mbar_wait(mbar, 0);
  } else {
    for (int i = tg; i < d_in; i += NTG) xs[i] = xrow[i];
    group_sync<G>(g);
  }

  // ---- pass 1: row min / max of z = x * d. Padded table entries (scale NaN)
  // never win a comparison; finiteness is checked on the raw input bits.
  double lo = INFINITY, hi = -INFINITY;
  uint32_t xbits = 0;
  for (int k0 = 4 * tg; k0 < ld; k0 += 4 * NTG) {
    double z[4];
    gather4_pad<T, GATHER>(p, xs, k0, z, xbits);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      lo = z[u] < lo ? z[u] : lo;
      hi = z[u] > hi ? z[u] : hi;
    }
  }
  bool nan = __any_sync(0xffffffffu, xbits >= InBits<T>::inf);
  if (G > 1) {
    if (lane == 0) red[2 * wg] = nan ? 1.0 : 0.0;
    group_sync<G>(g);
    double any = 0.0;
    for (int w = 0; w < G; ++w) any += red[2 * w];
    nan = any != 0.0;
    group_sync<G>(g);
  }
  group_minmax<G>(lo, hi, red, g, wg);
  if (nan || !isfinite(lo) || !isfinite(hi)) {  // group-uniform
    if (tg == 0) atomicOr(p.err, ERR_NONFINITE);
    return;
  }
  bool ok;
  const RowParams rp = make_row_params(lo, hi, p.act, &ok);  // identical in every thread
  const int cix = p.use_mac ? p.text_idx[row] : -1;
  const bool mac = cix >= 0;
  const bool cen = p.act.centered != 0;

  // ---- outlier path parameters (warp 0: text, warp 1 or 0: vision)
  const int vw = G > 1 ? 1 : 0;
  RowParams rt, rv;
  bool okt = true, okv = true, badt = false, badv = false;
  if (wg == 0 && p.n_text > 0) {
    outlier_params(p, xs, p.c_text, p.d_text, p.n_text, rt, okt, badt);
    if (lane == 0) { oscale[0] = rt.S; oflag[0] = badt; }
  }
  if (wg == vw && p.n_vis > 0) {
    outlier_params(p, xs, p.c_vis, p.d_vis, p.n_vis, rv, okv, badv);
    if (lane == 0) { oscale[1] = rv.S; oflag[1] = badv; }
  }
  group_sync<G>(g);
  const double st = p.n_text > 0 ? oscale[0] : 0.0;
  const double sv = p.n_vis > 0 ? oscale[1] : 0.0;
  if ((p.n_text > 0 && oflag[0]) || (p.n_vis > 0 && oflag[1])) {  // group-uniform
    if (tg == 0) atomicOr(p.err, ERR_NONFINITE);
    return;
  }
  // rho: power of two with max(S_a, S_t, S_v) in [rho, 2 rho) -- the common row
  // normaliser of the fp32 auxiliary accumulator
  int rexp;
  frexp(fmax(rp.S, fmax(st, sv)), &rexp);
  const double rho = ldexp(1.0, rexp - 1);
  if (tg == 0) {
    if (!ok) atomicOr(p.err, ERR_SCALE_ZERO);
    p.s_main[row] = rp.S;
    if (p.sf_main) p.sf_main[row] = (float)rp.S;
    p.zp_main[row] = rp.zp;
    if (p.rho) {
      p.rho[row] = (float)rho;
      p.lrs_main[row] = (float)(rp.S / rho);
    }
  }
  if (wg == 0 && p.n_text > 0) {
    outlier_codes(p, row, xs, p.c_text, p.d_text, p.n_text, p.ld_text, p.a_text, rt,
                  rt.S / rho, p.lr_off_t, p.kt16);
    if (lane == 0) {
      if (!okt) atomicOr(p.err, ERR_SCALE_ZERO);
      p.s_text[row] = rt.S;
      p.sf_text[row] = (float)rt.S;
      p.zp_text[row] = rt.zp;
    }
  }
  if (wg == vw && p.n_vis > 0) {
    outlier_codes(p, row, xs, p.c_vis, p.d_vis, p.n_vis, p.ld_vis, p.a_vis, rv, rv.S / rho,
                  p.lr_off_v, p.kv16);
    if (lane == 0) {
      if (!okv) atomicOr(p.err, ERR_SCALE_ZERO);
      p.s_vis[row] = rv.S;
      p.sf_vis[row] = (float)rv.S;
      p.zp_vis[row] = rv.zp;
    }
  }
  if (mac) {
    for (int n = tg; n <= rp.qmax - rp.qmin; n += NTG)
      xh[n] = __dmul_rn((double)(n + rp.qmin - rp.zp), rp.S);  // fake_quantize's (q - z) * S
    group_sync<G>(g);
  }

  // ---- pass 2: main codes (4 per 32-bit store) + MAC residual range
  int8_t* arow = p.a_main + (int64_t)row * ld;
  double elo = INFINITY, ehi = -INFINITY;
  for (int k0 = 4 * tg; k0 < ld; k0 += 4 * NTG) {
    double z[4];
    uint32_t dummy = 0;
    gather4_pad<T, GATHER>(p, xs, k0, z, dummy);
    int qv[4];
    bool t4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      t4[u] = false;
      qv[u] = quant_row(z[u], rp, t4[u]);
    }
    if (t4[0] | t4[1] | t4[2] | t4[3]) {  // exact .5 ties are common with fp16 inputs
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (t4[u]) qv[u] = quant_exact(z[u], rp.S, 0.0, rp.zp, rp.qmin, rp.qmax);
    }
    uint32_t packed = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = qv[u];
      const bool in = k0 + u < n_main;
      packed |= (uint32_t)((in ? (cen ? q - rp.zp : q) : 0) & 0xFF) << (8 * u);
      if (mac) {  // padded elements give e = NaN, which never wins
        const double e = __dsub_rn(z[u], xh[q - rp.qmin]);
        elo = e < elo ? e : elo;
        ehi = e > ehi ? e : ehi;
      }
    }
    *reinterpret_cast<uint32_t*>(arow + k0) = packed;
  }
  // ---- clear the low-rank columns of the auxiliary operand row (LR1 fills them)
  if (p.k_lr > 0) {
    uint4* lr = reinterpret_cast<uint4*>(p.lr_a + (int64_t)row * p.k_lr + p.lr_off_s);
    for (int i = tg; i < (p.k_lr - p.lr_off_s) / 8; i += NTG) lr[i] = make_uint4(0, 0, 0, 0);
  }
  if (!mac) return;

  // ---- pass 3 (text rows): residual codes (layer.py:159-160); q is read back
  // from the code row this thread itself wrote (same addresses, program order)
  group_minmax<G>(elo, ehi, red, g, wg);
  bool oke;
  const RowParams re = make_row_params(elo, ehi, p.aux, &oke);
  const bool cena = p.aux.centered != 0;
  if (tg == 0) {
    if (!oke) atomicOr(p.err, ERR_SCALE_ZERO);
    p.s_mac[cix] = re.S;
    p.zp_mac[cix] = re.zp;
    p.lrs_mac[cix] = (float)(re.S / rho);
  }
  int8_t* erow = p.a_mac + (int64_t)cix * ld;
  for (int k0 = 4 * tg; k0 < ld; k0 += 4 * NTG) {
    double z[4];
    uint32_t dummy = 0;
    gather4_pad<T, GATHER>(p, xs, k0, z, dummy);
    const uint32_t codes = *reinterpret_cast<const uint32_t*>(arow + k0);
    double e[4];
    int qe[4];
    bool t4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = cen ? (int)(int8_t)(codes >> (8 * u)) : (int)((codes >> (8 * u)) & 0xFF);
      const int q = cen ? c + rp.zp : c;
      e[u] = __dsub_rn(z[u], xh[min(max(q, rp.qmin), rp.qmax) - rp.qmin]);
      t4[u] = false;
      qe[u] = quant_row(e[u], re, t4[u]);
    }
    if (t4[0] | t4[1] | t4[2] | t4[3]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (t4[u]) qe[u] = quant_exact(e[u], re.S, 0.0, re.zp, re.qmin, re.qmax);
    }
    uint32_t packed = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = k0 + u < n_main;
      packed |= (uint32_t)((in ? (cena ? qe[u] - re.zp : qe[u]) : 0) & 0xFF) << (8 * u);
    }
    *reinterpret_cast<uint32_t*>(erow + k0) = packed;
  }
}

inline size_t k1_group_smem(int d_in, int esz, int G) {
  const int row_bytes = (d_in * esz + 127) / 128 * 128;
  return (size_t)(K1G_WARPS / G) * (row_bytes + 256 * 8 + 2 * G * 8 + 128);
}

}  // namespace splitq
