// K1 (warp-per-row): the stage-1 quantizer whose common path runs in fp32
// with certified error bounds and an exact fp64 fallback, so codes stay
// bit-identical to the reference's float64 numpy (quantizer.py:104-155,
// transform.py:94-103, layer.py:128-136 / 157-160).
//
// Work split: one warp owns one token row at a time (persistent warps, row
// r -> warp r mod #warps), so there is no CTA barrier anywhere: reductions
// are warp shuffles and the per-row parameters of the main / text / vision
// groups are computed concurrently on lanes 0 / 1 / 2. Main-path codes are
// stored in natural channel order (column c = channel c; outlier channels
// carry don't-care codes against all-zero weight rows), so the row is read
// with coalesced 16-byte loads and no gather. The row is read three times
// (extremes, codes, MAC residual codes): once from HBM, then from L1 / L2.
//
// Exactness (per row; z = fl64(x d), v_ref = fl64(z / S)):
//  * extremes: z32 = fl32(x fl32(d)) has |z32 - z| <= |z| 2^-22.9. Each lane
//    tracks its best and second-best 8-element chunk extremes; only chunks
//    within a 2^-21 band of the warp's fp32 extreme can hold the exact one,
//    and those are recomputed in fp64.
//  * codes: t = fl32(fl32(z32 fl32(1/S)) + C), C = 1.5*2^k + 0.5 + W ulp
//    (+ zp for uncentred storage), puts floor(v + 0.5) in the integer bits
//    of t. |t - (v_ref + C)| <= vmax 2^-21 + ulp / 2 < W ulp, so unless the
//    fractional bits of t lie within 2W ulp of the tie point (then: exact
//    fp64 recompute), floor(t) matches the reference's sign(v)floor(|v|+.5)
//    (the fl64(|v| + 0.5) rounding only matters inside that window). The
//    code byte is (bits(t) >> (23 - k)) & 0xFF since 2^(k-1) = 0 mod 256.
//  * MAC residual (text rows): e = z - fl64(n S) is exact (Sterbenz) and
//    e / S = v - n, so f = fl32(v32 - n) has v32's absolute error bound and
//    e / S_e = f (S / S_e) is coded the same way; its exact extremes come
//    from the same band-and-recompute step.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "quantize.cuh"
#include "quantize_fast.cuh"

namespace splitq {

constexpr int KW_THREADS = 128;  // 4 row warps per CTA
constexpr float KW_BAND = 4.76837158e-7f;  // 2^-21
constexpr int KW_QCAP = 64;  // flagged-chunk queue entries per warp

template <typename T>
struct XW {};
template <>
struct XW<__half> {
  static __device__ __forceinline__ float2 to_f2(uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
  static __device__ __forceinline__ uint32_t nanmax(uint32_t a, uint32_t w) {
    __half2 r = __hmax2_nan(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&w));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  // NaN or +inf was seen by a max that started at +0
  static __device__ __forceinline__ bool nonfinite(uint32_t m) {
    return ((m & 0x7FFFu) >= 0x7C00u) || (((m >> 16) & 0x7FFFu) >= 0x7C00u);
  }
};
template <>
struct XW<__nv_bfloat16> {
  static __device__ __forceinline__ float2 to_f2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  }
  static __device__ __forceinline__ uint32_t nanmax(uint32_t a, uint32_t w) {
    __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<const __nv_bfloat162*>(&a),
                                   *reinterpret_cast<const __nv_bfloat162*>(&w));
    return *reinterpret_cast<uint32_t*>(&r);
  }
  static __device__ __forceinline__ bool nonfinite(uint32_t m) {
    return ((m & 0x7FFFu) >= 0x7F80u) || (((m >> 16) & 0x7FFFu) >= 0x7F80u);
  }
};

__device__ __forceinline__ uint64_t kw_pack64(float2 a) {
  return *reinterpret_cast<uint64_t*>(&a);
}
__device__ __forceinline__ float2 kw_unpack64(uint64_t a) {
  return *reinterpret_cast<float2*>(&a);
}
__device__ __forceinline__ float2 kw_mul2(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(kw_pack64(a)), "l"(kw_pack64(b)));
  return kw_unpack64(r);
}
__device__ __forceinline__ float2 kw_add2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(kw_pack64(a)), "l"(kw_pack64(b)));
  return kw_unpack64(r);
}
__device__ __forceinline__ float2 kw_fma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(kw_pack64(a)), "l"(kw_pack64(b)), "l"(kw_pack64(c)));
  return kw_unpack64(r);
}

__device__ __forceinline__ uint4 kw_ldg(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// exact reference code of m at scale S: clip(rha(fl64(m / S)) + zp, qmin, qmax)
__device__ __noinline__ int kw_exact_code(double m, double S, int zp, int qmin, int qmax) {
  const double v = __ddiv_rn(m, S);
  const double a = floor(__dadd_rn(fabs(v), 0.5));
  double q = (v < 0.0 ? -a : a) + (double)zp;
  q = fmin(fmax(q, (double)qmin), (double)qmax);
  return (int)q;
}

// Fixed-point rounding constants of one group (see the header comment).
struct KwConsts {
  float rs, C, base;
  uint32_t F, fm, W2;
  int safe;
};

// lo / hi exact, S / zp from group_params, qspec, extra error bound in units of v.
// The fast path has no clip: rows whose extreme codes would clip (never for
// the reference's own S / zp up to fp64 rounding at ties) run exactly.
__device__ __forceinline__ KwConsts kw_consts(double lo, double hi, double S, int zp,
                                          const QSpecDev& s, double err_scale_extra) {
  KwConsts c;
  const double rS = __ddiv_rn(1.0, S);
  const double vmax = fmax(fabs(lo), fabs(hi)) * rS;
  const double err = vmax * 4.76837158203125e-07 + err_scale_extra;  // 2^-21
  c.safe = vmax < 1048576.0;
  int k = 10;
  while (k < 22 && !((double)(1 << (k - 1)) > vmax + 2.0)) ++k;
  const double ulp = ldexp(1.0, k - 23);
  c.F = (uint32_t)(23 - k);
  c.fm = (1u << c.F) - 1u;
  const double Wd = floor((err + 0.5 * ulp) / ulp) + 1.0;
  if (!(Wd < (double)(1 << (c.F - 2)))) c.safe = 0;
  const double W = c.safe ? Wd : 1.0;
  c.W2 = (uint32_t)(2.0 * W);
  const int zq = s.centered ? 0 : zp;
  const double b = 1.5 * ldexp(1.0, k) + (double)zq;
  c.rs = (float)rS;
  c.base = (float)b;
  c.C = (float)(b + 0.5 + W * ulp);
  // The fast path does not clip. Elements that would clip lie beyond
  // qmax + 1/2 (or below qmin - 1/2) in units of code; while the row's
  // extremes overshoot those points by at most ulp / 2, every such element
  // is inside the flagged window (|t - tie| < W ulp + ulp / 2 rounds to
  // <= W ulp on the t grid) and takes the exact (clipping) path. Larger
  // overshoots (rows far from zero relative to their span) run exactly.
  const double vl = __ddiv_rn(lo, S), vh = __ddiv_rn(hi, S);
  const double over = vh + (double)zp - ((double)s.qmax + 0.5);
  const double under = ((double)s.qmin - 0.5) - (vl + (double)zp);
  if (over > 0.5 * ulp || under > 0.5 * ulp) c.safe = 0;
  return c;
}

__device__ __forceinline__ KwConsts kw_shfl(const KwConsts& c, int src) {
  KwConsts o;
  o.rs = __shfl_sync(0xffffffffu, c.rs, src);
  o.C = __shfl_sync(0xffffffffu, c.C, src);
  o.base = __shfl_sync(0xffffffffu, c.base, src);
  o.F = __shfl_sync(0xffffffffu, c.F, src);
  o.fm = __shfl_sync(0xffffffffu, c.fm, src);
  o.W2 = __shfl_sync(0xffffffffu, c.W2, src);
  o.safe = __shfl_sync(0xffffffffu, c.safe, src);
  return o;
}
__device__ __forceinline__ double kw_shfl_d(double v, int src) {
  return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(v), src),
                          __shfl_sync(0xffffffffu, __double2loint(v), src));
}

__device__ __forceinline__ float kw_min8(const float (&z)[8]) {
  return fminf(fminf(fminf(z[0], z[1]), fminf(z[2], z[3])), fminf(fminf(z[4], z[5]), fminf(z[6], z[7])));
}
__device__ __forceinline__ float kw_max8(const float (&z)[8]) {
  return fmaxf(fmaxf(fmaxf(z[0], z[1]), fmaxf(z[2], z[3])), fmaxf(fmaxf(z[4], z[5]), fmaxf(z[6], z[7])));
}

// best / second-best chunk extreme of a lane (min form; max uses negation)
struct KwExt {
  float m1, m2;
  int c1;
};
__device__ __forceinline__ void kw_ext_init(KwExt& e) {
  e.m1 = INFINITY;
  e.m2 = INFINITY;
  e.c1 = -1;
}
__device__ __forceinline__ void kw_ext_upd(KwExt& e, float cm, int j) {
  const bool better = cm < e.m1;
  e.m2 = better ? e.m1 : fminf(e.m2, cm);
  e.c1 = better ? j : e.c1;
  e.m1 = better ? cm : e.m1;
}

__device__ __forceinline__ double kw_warp_min_d(double v) {
  const unsigned m = __ballot_sync(0xffffffffu, v < INFINITY);
  if (m == 0) return INFINITY;
  if ((m & (m - 1)) == 0) return kw_shfl_d(v, __ffs(m) - 1);
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double kw_warp_max_d(double v) {
  const unsigned m = __ballot_sync(0xffffffffu, v > -INFINITY);
  if (m == 0) return -INFINITY;
  if ((m & (m - 1)) == 0) return kw_shfl_d(v, __ffs(m) - 1);
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ void kw_load(const K1Params& p, const uint4* xg, int j, float (&x)[8],
                                        float (&d)[8]) {
  const uint4 w = kw_ldg(xg + j);
  const float4 da = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j);
  const float4 db = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j + 1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 f2 = XW<T>::to_f2(ws[h]);
    x[2 * h] = f2.x;
    x[2 * h + 1] = f2.y;
  }
  d[0] = da.x; d[1] = da.y; d[2] = da.z; d[3] = da.w;
  d[4] = db.x; d[5] = db.y; d[6] = db.z; d[7] = db.w;
}

// z32, v32 and t bits of a chunk (bit-identical in every pass)
__device__ __forceinline__ void kw_codes(const float (&x)[8], const float (&d)[8], const KwConsts& c,
                                         float (&v)[8], uint32_t (&b)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 z = kw_mul2(make_float2(x[2 * h], x[2 * h + 1]), make_float2(d[2 * h], d[2 * h + 1]));
    const float2 vv = kw_mul2(z, make_float2(c.rs, c.rs));
    const float2 t = kw_add2(vv, make_float2(c.C, c.C));
    v[2 * h] = vv.x;
    v[2 * h + 1] = vv.y;
    b[2 * h] = __float_as_uint(t.x);
    b[2 * h + 1] = __float_as_uint(t.y);
  }
}

__device__ __forceinline__ uint32_t kw_minfrac(const uint32_t (&b)[8], uint32_t fm) {
  uint32_t m = b[0] & fm;
#pragma unroll
  for (int e = 1; e < 8; ++e) m = min(m, b[e] & fm);
  return m;
}

__device__ __forceinline__ uint2 kw_pack(const uint32_t (&bytes)[8]) {
  uint2 o;
  o.x = __byte_perm(__byte_perm(bytes[0], bytes[1], 0x0040), __byte_perm(bytes[2], bytes[3], 0x0040), 0x5410);
  o.y = __byte_perm(__byte_perm(bytes[4], bytes[5], 0x0040), __byte_perm(bytes[6], bytes[7], 0x0040), 0x5410);
  return o;
}

struct KwRow {  // exact main-group parameters needed by the fallbacks
  double S;
  int zp;
};

// exact MAC residual e64 of channel c (layer.py:135-136, 157-159)
__device__ __forceinline__ double kw_exact_e(const K1Params& p, float x, int c, const KwRow& r) {
  const double z64 = __dmul_rn((double)x, __ldg(p.d_main + c));
  const int q = kw_exact_code(z64, r.S, r.zp, p.act.qmin, p.act.qmax);
  return __dsub_rn(z64, __dmul_rn((double)(q - r.zp), r.S));
}

template <typename T>
__device__ __forceinline__ float kw_x(const T* xrow, int c) {
  const uint16_t h = reinterpret_cast<const uint16_t*>(xrow)[c];
  const float2 f = XW<T>::to_f2((uint32_t)h);
  return f.x;
}

// Warp-uniform append of chunk j to the warp's flagged queue (SMEM).
__device__ __forceinline__ void kw_enqueue(uint32_t* q, int& qn, bool flag, int j) {
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  if (bal) {
    const int lane = threadIdx.x & 31;
    const int pos = qn + __popc(bal & ((1u << lane) - 1u));
    if (flag && pos < KW_QCAP) q[pos] = (uint32_t)j;
    qn += __popc(bal);
  }
}

// Pass E: main codes (+ MAC fraction extremes of the unflagged chunks).
template <typename T, bool MAC>
__device__ __forceinline__ void kw_pass_codes(const K1Params& p, const uint4* xg, int nchunks,
                                              int8_t* arow, const KwConsts& c, KwExt& flo,
                                              KwExt& fhi, uint32_t* q, int& qn) {
  const int lane = threadIdx.x & 31;
  for (int j0 = 0; j0 < nchunks; j0 += 32) {
    const int j = j0 + lane;
    bool flag = false;
    if (j < nchunks) {
      float x[8], d[8], v[8];
      uint32_t b[8], bytes[8];
      kw_load<T>(p, xg, j, x, d);
      kw_codes(x, d, c, v, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) bytes[e] = b[e] >> c.F;
      *reinterpret_cast<uint2*>(arow + 8 * j) = kw_pack(bytes);
      flag = kw_minfrac(b, c.fm) <= c.W2;
      if (MAC && !flag) {
        float f[8], nf[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          f[e] = v[e] - (__uint_as_float(b[e] & ~c.fm) - c.base);
          nf[e] = -f[e];
        }
        kw_ext_upd(flo, kw_min8(f), j);
        kw_ext_upd(fhi, kw_min8(nf), j);
      }
    }
    kw_enqueue(q, qn, flag, j);
  }
}

// Pass G (text rows): MAC residual codes.
template <typename T>
__device__ __forceinline__ void kw_pass_mac(const K1Params& p, const uint4* xg, int nchunks,
                                            int8_t* erow, const KwConsts& c, const KwConsts& ce,
                                            float ratio, uint32_t* q, int& qn) {
  const int lane = threadIdx.x & 31;
  for (int j0 = 0; j0 < nchunks; j0 += 32) {
    const int j = j0 + lane;
    bool flag = false;
    if (j < nchunks) {
      float x[8], d[8], v[8];
      uint32_t b[8], be[8], bytes[8];
      kw_load<T>(p, xg, j, x, d);
      kw_codes(x, d, c, v, b);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float2 f = make_float2(v[2 * h] - (__uint_as_float(b[2 * h] & ~c.fm) - c.base),
                                     v[2 * h + 1] - (__uint_as_float(b[2 * h + 1] & ~c.fm) - c.base));
        const float2 t = kw_fma2(f, make_float2(ratio, ratio), make_float2(ce.C, ce.C));
        be[2 * h] = __float_as_uint(t.x);
        be[2 * h + 1] = __float_as_uint(t.y);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) bytes[e] = be[e] >> ce.F;
      *reinterpret_cast<uint2*>(erow + 8 * j) = kw_pack(bytes);
      flag = kw_minfrac(b, c.fm) <= c.W2 || kw_minfrac(be, ce.fm) <= ce.W2;
    }
    kw_enqueue(q, qn, flag, j);
  }
}

// exact extreme over the candidate chunks of one lane (main: z; band test on z32)
template <typename T>
__device__ __forceinline__ double kw_rescan_z(const K1Params& p, const T* xrow, int nchunks,
                                              const KwExt& e, float band, bool is_max) {
  const int lane = threadIdx.x & 31;
  double best = is_max ? -INFINITY : INFINITY;
  const bool all = e.m2 <= band;  // a second chunk is also within the band
  for (int j = all ? lane : e.c1; j < nchunks; j += 32) {
    for (int u = 0; u < 8; ++u) {
      const float x = kw_x<T>(xrow, 8 * j + u);
      const float z = __fmul_rn(x, __ldg(p.d_main32 + 8 * j + u));
      if ((is_max ? -z : z) <= band) {
        const double z64 = __dmul_rn((double)x, __ldg(p.d_main + 8 * j + u));
        best = is_max ? fmax(best, z64) : fmin(best, z64);
      }
    }
    if (!all) break;
  }
  return best;
}

// exact extreme of the MAC residual over a lane's candidate chunks (band test on f)
template <typename T>
__device__ __forceinline__ double kw_rescan_e(const K1Params& p, const T* xrow, int nchunks,
                                              const KwExt& e, float band, bool is_max,
                                              const KwConsts& c, const KwRow& r) {
  const int lane = threadIdx.x & 31;
  double best = is_max ? -INFINITY : INFINITY;
  const bool all = e.m2 <= band;
  for (int j = all ? lane : e.c1; j < nchunks; j += 32) {
    for (int u = 0; u < 8; ++u) {
      const float x = kw_x<T>(xrow, 8 * j + u);
      const float v = __fmul_rn(__fmul_rn(x, __ldg(p.d_main32 + 8 * j + u)), c.rs);
      const uint32_t b = __float_as_uint(__fadd_rn(v, c.C));
      const float f = v - (__uint_as_float(b & ~c.fm) - c.base);
      if ((is_max ? -f : f) <= band) {
        const double e64 = kw_exact_e(p, x, 8 * j + u, r);
        best = is_max ? fmax(best, e64) : fmin(best, e64);
      }
    }
    if (!all) break;
  }
  return best;
}

template <typename T>
__global__ void __launch_bounds__(KW_THREADS) k1w_kernel(const K1Params p, int d_in) {
  __shared__ uint32_t kw_q[KW_THREADS / 32][KW_QCAP];
  const int lane = threadIdx.x & 31;
  uint32_t* q = kw_q[threadIdx.x >> 5];
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int nchunks = d_in >> 3;
  const bool cen = p.act.centered != 0, cena = p.aux.centered != 0;
  for (int row = gw; row < p.T; row += nw) {
    const T* xrow = reinterpret_cast<const T*>(p.x) + (int64_t)row * p.ldx;
    const uint4* xg = reinterpret_cast<const uint4*>(xrow);

    // ------------------------------------------------ pass A: fp32 extremes
    KwExt elo, ehi;  // ehi tracks -max
    kw_ext_init(elo);
    kw_ext_init(ehi);
    uint32_t nm = 0u;
    for (int j = lane; j < nchunks; j += 32) {
      const uint4 w = kw_ldg(xg + j);
      const float4 da = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j);
      const float4 db = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j + 1);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      const float d[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
      float z[8], nz[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        nm = XW<T>::nanmax(nm, ws[h]);
        const float2 zz = kw_mul2(XW<T>::to_f2(ws[h]), make_float2(d[2 * h], d[2 * h + 1]));
        z[2 * h] = zz.x;
        z[2 * h + 1] = zz.y;
        nz[2 * h] = -zz.x;
        nz[2 * h + 1] = -zz.y;
      }
      kw_ext_upd(elo, kw_min8(z), j);
      kw_ext_upd(ehi, kw_min8(nz), j);
    }
    float L = elo.m1, H = ehi.m1;  // H = -max
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      L = fminf(L, __shfl_xor_sync(0xffffffffu, L, o));
      H = fminf(H, __shfl_xor_sync(0xffffffffu, H, o));
    }
    // row metadata (lane 0 loads, broadcast)
    int slot = -1;
    if (lane == 0) {
      const uint8_t tg = p.tags ? p.tags[row] : (uint8_t)1;
      if (tg > 1) atomicOr(p.err, ERR_BAD_TAG);
      slot = (p.use_mac && p.text_idx) ? p.text_idx[row] : -1;
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    bool bad = __any_sync(0xffffffffu, XW<T>::nonfinite(nm)) || !isfinite(L) || !isfinite(H);

    // outlier paths: exact fp64 params (warp-level; quantize_fast.cuh)
    RowParams rt, rv;
    bool okt = true, okv = true, badt = false, badv = false;
    rt.S = rv.S = 0.0;
    if (p.n_text > 0) outlier_params(p, xrow, p.c_text, p.d_text, p.n_text, rt, okt, badt);
    if (p.n_vis > 0) outlier_params(p, xrow, p.c_vis, p.d_vis, p.n_vis, rv, okv, badv);
    if (bad || badt || badv) {
      if (lane == 0) atomicOr(p.err, ERR_NONFINITE);
      continue;
    }

    // ------------------------------------------------ exact main extremes
    const float bl = L + fabsf(L) * KW_BAND + 1e-30f;
    const float bh = H + fabsf(H) * KW_BAND + 1e-30f;
    double lo64 = INFINITY, hi64 = -INFINITY;
    if (elo.m1 <= bl) lo64 = kw_rescan_z<T>(p, xrow, nchunks, elo, bl, false);
    if (ehi.m1 <= bh) hi64 = kw_rescan_z<T>(p, xrow, nchunks, ehi, bh, true);
    lo64 = kw_warp_min_d(lo64);
    hi64 = kw_warp_max_d(hi64);

    // ------------------------------------------------ main group parameters (lane 0)
    KwConsts c{};
    double S = 1.0;
    int zp = 0;
    if (lane == 0) {
      double zpd;
      if (!group_params(lo64, hi64, p.act, &S, &zpd)) {
        atomicOr(p.err, ERR_SCALE_ZERO);
        S = 1.0;
      }
      zp = (int)zpd;
      c = kw_consts(lo64, hi64, S, zp, p.act, 0.0);
    }
    c = kw_shfl(c, 0);
    S = kw_shfl_d(S, 0);
    zp = __shfl_sync(0xffffffffu, zp, 0);
    int rexp;
    frexp(fmax(S, fmax(rt.S, rv.S)), &rexp);
    const double rho = ldexp(1.0, rexp - 1);
    if (lane == 0) {
      p.s_main[row] = S;
      if (p.sf_main) p.sf_main[row] = (float)S;
      p.zp_main[row] = zp;
      if (p.rho) {
        p.rho[row] = (float)rho;
        p.lrs_main[row] = (float)(S / rho);
      }
    }
    const KwRow r{S, zp};

    // ------------------------------------------------ outlier codes + aux segments
    if (p.n_text > 0) {
      outlier_codes(p, row, xrow, p.c_text, p.d_text, p.n_text, p.ld_text, p.a_text, rt,
                    rt.S / rho, p.lr_off_t, p.kt16);
      if (lane == 0) {
        if (!okt) atomicOr(p.err, ERR_SCALE_ZERO);
        p.s_text[row] = rt.S;
        p.sf_text[row] = (float)rt.S;
        p.zp_text[row] = rt.zp;
      }
    }
    if (p.n_vis > 0) {
      outlier_codes(p, row, xrow, p.c_vis, p.d_vis, p.n_vis, p.ld_vis, p.a_vis, rv, rv.S / rho,
                    p.lr_off_v, p.kv16);
      if (lane == 0) {
        if (!okv) atomicOr(p.err, ERR_SCALE_ZERO);
        p.s_vis[row] = rv.S;
        p.sf_vis[row] = (float)rv.S;
        p.zp_vis[row] = rv.zp;
      }
    }
    if (p.k_lr > 0) {  // the low-rank columns of the aux operand row: LR1 fills them
      uint4* lr = reinterpret_cast<uint4*>(p.lr_a + (int64_t)row * p.k_lr + p.lr_off_s);
      for (int i = lane; i < (p.k_lr - p.lr_off_s) / 8; i += 32) lr[i] = make_uint4(0, 0, 0, 0);
    }

    // ------------------------------------------------ pass E: main codes
    int8_t* arow = p.a_main + (int64_t)row * p.ld_main;
    const bool mac = slot >= 0;
    KwExt flo, fhi;
    kw_ext_init(flo);
    kw_ext_init(fhi);
    int qn = 0;
    if (c.safe) {
      if (mac) kw_pass_codes<T, true>(p, xg, nchunks, arow, c, flo, fhi, q, qn);
      else kw_pass_codes<T, false>(p, xg, nchunks, arow, c, flo, fhi, q, qn);
    }
    // exact fallback: the flagged chunks (queue), or every chunk (unsafe row /
    // queue overflow); elements spread over the lanes. MAC: the exact residual
    // of every element of these chunks joins the extreme candidates.
    const bool allx = !c.safe || qn > KW_QCAP;
#ifdef KW_DEBUG
    if (lane == 0) {
      atomicAdd(p.err + 1, qn);
      if (allx) atomicAdd(p.err + 2, 1);
    }
#endif
    const int nfix = 8 * (allx ? nchunks : qn);
    __syncwarp();
    double xlo = INFINITY, xhi = -INFINITY;
    for (int i = lane; i < nfix; i += 32) {
      const int ch = 8 * (allx ? i >> 3 : (int)q[i >> 3]) + (i & 7);
      const float x = kw_x<T>(xrow, ch);
      const double z64 = __dmul_rn((double)x, __ldg(p.d_main + ch));
      const int qc = kw_exact_code(z64, S, zp, p.act.qmin, p.act.qmax);
      arow[ch] = (int8_t)(cen ? qc - zp : qc);
      if (mac) {
        const double e64 = __dsub_rn(z64, __dmul_rn((double)(qc - zp), S));
        xlo = fmin(xlo, e64);
        xhi = fmax(xhi, e64);
      }
    }
    if (!mac) continue;

    // ------------------------------------------------ MAC: exact residual extremes
    float FL = flo.m1, FH = fhi.m1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      FL = fminf(FL, __shfl_xor_sync(0xffffffffu, FL, o));
      FH = fminf(FH, __shfl_xor_sync(0xffffffffu, FH, o));
    }
    // |f - e / S| <= vmax 2^-22 (+ the fp32 rounding of f): an absolute band
    const float vmaxf = fmaxf(fabsf(L), fabsf(H)) * c.rs * 1.0001f + 1.0f;
    const float fband = 2.0f * vmaxf * KW_BAND + 1e-12f;
    const float bfl = FL + fband, bfh = FH + fband;
    double elo64 = xlo, ehi64 = xhi;
    if (!allx) {
      if (flo.m1 <= bfl) elo64 = fmin(elo64, kw_rescan_e<T>(p, xrow, nchunks, flo, bfl, false, c, r));
      if (fhi.m1 <= bfh) ehi64 = fmax(ehi64, kw_rescan_e<T>(p, xrow, nchunks, fhi, bfh, true, c, r));
    }
    elo64 = kw_warp_min_d(elo64);
    ehi64 = kw_warp_max_d(ehi64);
    KwConsts ce{};
    double Se = 1.0;
    int zpe = 0;
    if (lane == 0) {
      double zpd;
      if (!group_params(elo64, ehi64, p.aux, &Se, &zpd)) {
        atomicOr(p.err, ERR_SCALE_ZERO);
        Se = 1.0;
      }
      zpe = (int)zpd;
      // f carries |err| <= vmax 2^-22 in units of S: times S / Se in units of e / Se
      ce = kw_consts(elo64, ehi64, Se, zpe, p.aux, (double)vmaxf * 2.384185791015625e-07 * (S / Se) * 1.01);
      p.s_mac[slot] = Se;
      p.zp_mac[slot] = zpe;
      p.lrs_mac[slot] = (float)(Se / rho);
    }
    ce = kw_shfl(ce, 0);
    Se = kw_shfl_d(Se, 0);
    zpe = __shfl_sync(0xffffffffu, zpe, 0);
    const float ratio = (float)(S / Se);

    // ------------------------------------------------ pass G: MAC residual codes
    int8_t* erow = p.a_mac + (int64_t)slot * p.ld_main;
    qn = 0;
    const bool allg = allx || !ce.safe;
    __syncwarp();
    if (!allg) kw_pass_mac<T>(p, xg, nchunks, erow, c, ce, ratio, q, qn);
    const bool allg2 = allg || qn > KW_QCAP;
#ifdef KW_DEBUG
    if (lane == 0) {
      atomicAdd(p.err + 3, qn);
      if (allg2) atomicAdd(p.err + 2, 1 << 16);
    }
#endif
    const int ngix = 8 * (allg2 ? nchunks : qn);
    __syncwarp();
    for (int i = lane; i < ngix; i += 32) {
      const int ch = 8 * (allg2 ? i >> 3 : (int)q[i >> 3]) + (i & 7);
      const double e64 = kw_exact_e(p, kw_x<T>(xrow, ch), ch, r);
      const int qe = kw_exact_code(e64, Se, zpe, p.aux.qmin, p.aux.qmax);
      erow[ch] = (int8_t)(cena ? qe - zpe : qe);
    }
    __syncwarp();
  }
}

}  // namespace splitq
