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
//  * codes: t = fl32(z32 fl32(1/S) + C) (one fused rounding), C = 1.5*2^k +
//    0.5 + W ulp (+ zp for uncentred storage), puts floor(v + 0.5) in the
//    integer bits of t. |t - (v_ref + C)| <= vmax 2^-21 + ulp / 2 < W ulp
//    (the bound holds for the two-rounding form too), so unless the
//    fractional bits of t lie within 2W ulp of the tie point (then: exact
//    fp64 recompute), floor(t) matches the reference's sign(v)floor(|v|+.5)
//    (the fl64(|v| + 0.5) rounding only matters inside that window). The
//    code byte is (bits(t) >> (23 - k)) & 0xFF since 2^(k-1) = 0 mod 256.
//  * MAC residual (text rows): e = z - fl64(n S) is exact (Sterbenz) and
//    e / S = v - n, so f = fl32(z32 fl32(1/S) - n) has v32's absolute error
//    bound (plus one rounding of |f| <= 1/2) and
//    e / S_e = f (S / S_e) is coded the same way; its exact extremes come
//    from the same band-and-recompute step.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "quantize.cuh"
#include "quantize_fast.cuh"

namespace splitq {

constexpr int KW_THREADS = 128;       // warp-per-row CTAs: 4 row warps
constexpr int KW_THREADS_SYNC = 512;  // ... with a barrier per row round: 16 row warps

#ifdef KW_TRACE  // phase clocks of CTA 0's first row (tools/k1_trace.py)
#define KW_STAMP(i) \
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && row == gw) p.trace[i] = clock64();
#else
#define KW_STAMP(i)
#endif
constexpr float KW_BAND = 4.76837158e-7f;  // 2^-21
constexpr int KW_QCAP = 128;  // flagged-chunk queue entries per warp

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
static __device__ __noinline__ int kw_exact_code(double m, double S, int zp, int qmin, int qmax) {
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

// one chunk's raw operands, loaded a loop iteration ahead (PF)
struct KwRaw {
  uint4 w;
  float4 da, db;
};
__device__ __forceinline__ KwRaw kw_ldraw(const K1Params& p, const uint4* xg, int j) {
  KwRaw r;
  r.w = kw_ldg(xg + j);
  r.da = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j);
  r.db = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j + 1);
  return r;
}
template <typename T>
__device__ __forceinline__ void kw_cvt(const KwRaw& r, float (&x)[8], float (&d)[8]) {
  const uint32_t ws[4] = {r.w.x, r.w.y, r.w.z, r.w.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 f2 = XW<T>::to_f2(ws[h]);
    x[2 * h] = f2.x;
    x[2 * h + 1] = f2.y;
  }
  d[0] = r.da.x; d[1] = r.da.y; d[2] = r.da.z; d[3] = r.da.w;
  d[4] = r.db.x; d[5] = r.db.y; d[6] = r.db.z; d[7] = r.db.w;
}

// x from the row group's SMEM copy, the factors from the global fp32 table
template <typename T>
__device__ __forceinline__ void kw_load_xs(const K1Params& p, const uint4* xs, int j, float (&x)[8],
                                           float (&d)[8]) {
  const uint4 w = xs[j];
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

// the same from the row group's SMEM copy (x plane + two d planes)
template <typename T>
__device__ __forceinline__ void kw_load_s(const uint4* xs, const float4* ds, int nch, int j,
                                          float (&x)[8], float (&d)[8]) {
  const uint4 w = xs[j];
  const float4 da = ds[j], db = ds[nch + j];
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

__device__ __forceinline__ void kw_mulz(const float (&x)[8], const float (&d)[8], float (&z)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 zz = kw_mul2(make_float2(x[2 * h], x[2 * h + 1]), make_float2(d[2 * h], d[2 * h + 1]));
    z[2 * h] = zz.x;
    z[2 * h + 1] = zz.y;
  }
}

// the t bits of a chunk from its z32: t = fl32(z32 rs + C), one rounding
// (bit-identical in every pass). The window of kw_consts2 was derived for
// fl32(fl32(z32 rs) + C); the fused form's error is no larger.
__device__ __forceinline__ void kw_vt(const float (&z)[8], const KwConsts& c, uint32_t (&b)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 t = kw_fma2(make_float2(z[2 * h], z[2 * h + 1]), make_float2(c.rs, c.rs), make_float2(c.C, c.C));
    b[2 * h] = __float_as_uint(t.x);
    b[2 * h + 1] = __float_as_uint(t.y);
  }
}

// f = fl32(z32 rs - n) for the chunk (n from the integer bits of t; the
// product is not rounded before the subtraction, so f carries only z32's
// error, |f - (v - n)| <= |v| 2^-22.4 + 2^-25)
__device__ __forceinline__ void kw_frac(const float (&z)[8], const uint32_t (&b)[8], const KwConsts& c,
                                        float (&f)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 nf = kw_add2(make_float2(__uint_as_float(b[2 * h] & ~c.fm), __uint_as_float(b[2 * h + 1] & ~c.fm)),
                              make_float2(-c.base, -c.base));
    const float2 ff = kw_fma2(make_float2(z[2 * h], z[2 * h + 1]), make_float2(c.rs, c.rs), make_float2(-nf.x, -nf.y));
    f[2 * h] = ff.x;
    f[2 * h + 1] = ff.y;
  }
}

// f = v - n, compensated: z = x d as fl32(x d_hi) + (its exact error + x d_lo),
// v = z (rs + rs_lo) with the exact error of the leading product, so
// |f - (fl64(x d) / S - n)| <= 2^-23 + |v| 2^-40 (two fp32 roundings of
// quantities below 0.52, then terms of relative size 2^-44)
__device__ __forceinline__ void kw_frac_comp(const K1Params& p, int j, const float (&x)[8], const float (&d)[8],
                                             const float (&z)[8], const uint32_t (&b)[8], const KwConsts& c,
                                             float rs_lo, float (&f)[8]) {
  const float4 la = __ldg(reinterpret_cast<const float4*>(p.d_main_lo32) + 2 * j);
  const float4 lb = __ldg(reinterpret_cast<const float4*>(p.d_main_lo32) + 2 * j + 1);
  const float dl[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
  const float2 rs2 = make_float2(c.rs, c.rs), rl2 = make_float2(rs_lo, rs_lo);
#pragma unroll
  for (int h = 0; h < 4; ++h) {  // two elements per packed op (each lane rounds as the scalar op)
    const float2 x2 = make_float2(x[2 * h], x[2 * h + 1]), z2 = make_float2(z[2 * h], z[2 * h + 1]);
    const float2 plo = kw_fma2(x2, make_float2(d[2 * h], d[2 * h + 1]), make_float2(-z2.x, -z2.y));  // exact
    const float2 zl = kw_fma2(x2, make_float2(dl[2 * h], dl[2 * h + 1]), plo);                     // + x d_lo
    const float2 vh = kw_mul2(z2, rs2);
    float2 vl = kw_fma2(z2, rs2, make_float2(-vh.x, -vh.y));  // exact error of vh
    vl = kw_fma2(z2, rl2, vl);
    vl = kw_fma2(zl, rs2, vl);
    const float2 n2 = kw_add2(make_float2(__uint_as_float(b[2 * h] & ~c.fm), __uint_as_float(b[2 * h + 1] & ~c.fm)),
                              make_float2(-c.base, -c.base));
    const float2 ff = kw_add2(kw_add2(vh, make_float2(-n2.x, -n2.y)), vl);
    f[2 * h] = ff.x;
    f[2 * h + 1] = ff.y;
  }
}

__device__ __forceinline__ uint32_t kw_minfrac(const uint32_t (&b)[8], uint32_t fm) {
  uint32_t m = b[0] & fm;
#pragma unroll
  for (int e = 1; e < 8; ++e) m = min(m, b[e] & fm);
  return m;
}

__device__ __forceinline__ uint2 kw_pack_shift(const uint32_t (&b)[8], uint32_t F) {
  uint32_t by[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) by[e] = b[e] >> F;
  uint2 o;
  o.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040), __byte_perm(by[2], by[3], 0x0040), 0x5410);
  o.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040), __byte_perm(by[6], by[7], 0x0040), 0x5410);
  return o;
}

__device__ __forceinline__ unsigned long long okey_d(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ounkey_d(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

struct KwRow {  // exact main-group parameters needed by the fallbacks
  double S;
  int zp;
};

template <typename T>
__device__ __forceinline__ float kw_x(const T* xrow, int c) {
  const uint16_t h = reinterpret_cast<const uint16_t*>(xrow)[c];
  return XW<T>::to_f2((uint32_t)h).x;
}

// fp64 smoothing factor of channel c: from the global table, or from the
// row group's SMEM copy (KwD::smem)
struct KwD {
  const double* d;
  bool smem;
  __device__ __forceinline__ double operator[](int c) const { return smem ? d[c] : __ldg(d + c); }
};

// exact main code of channel c: returns q, writes z64
__device__ __forceinline__ int kw_exact_main(const K1Params& p, const KwD& dm, float x, int c, const KwRow& r,
                                             double& z64) {
  z64 = __dmul_rn((double)x, dm[c]);
  return kw_exact_code(z64, r.S, r.zp, p.act.qmin, p.act.qmax);
}
// exact MAC residual e64 of channel c (layer.py:135-136, 157-159)
__device__ __forceinline__ double kw_exact_e(const K1Params& p, const KwD& dm, float x, int c, const KwRow& r) {
  double z64;
  const int q = kw_exact_main(p, dm, x, c, r, z64);
  return __dsub_rn(z64, __dmul_rn((double)(q - r.zp), r.S));
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

// warp reductions through REDUX on order-preserving integer keys
__device__ __forceinline__ int kw_fkey(float f) {
  const int b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float kw_warp_minf(float v) {
  const int k = __reduce_min_sync(0xffffffffu, kw_fkey(v));
  return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF));
}
// fp64 min / max of non-NaN values (+-inf allowed) in two 32-bit REDUX steps
__device__ __forceinline__ double kw_warp_mind(double v) {
  const unsigned long long k = okey_d(v);
  const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)(k >> 32));
  const unsigned lo = __reduce_min_sync(0xffffffffu, (unsigned)(k >> 32) == hi ? (unsigned)k : 0xFFFFFFFFu);
  return ounkey_d(((unsigned long long)hi << 32) | lo);
}
__device__ __forceinline__ double kw_warp_maxd(double v) {
  const unsigned long long k = okey_d(v);
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
  return ounkey_d(((unsigned long long)hi << 32) | lo);
}

// Row groups of WPR > 1 warps (decode-sized calls: one CTA per row): the
// warp-uniform values of NV order-preserving u64 keys meet in SMEM (one slot
// block per call site, so consecutive sites need one barrier each); min.
template <int WPR, int NV>
__device__ __forceinline__ void kw_gmin(uint64_t* red, uint64_t (&k)[NV]) {
  if constexpr (WPR > 1) {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int v = 0; v < NV; ++v) red[w * NV + v] = k[v];
    __syncthreads();
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      uint64_t m = red[v];
      for (int i = 1; i < WPR; ++i) m = min(m, red[i * NV + v]);
      k[v] = m;
    }
  }
}
__device__ __forceinline__ uint64_t kw_fkey64(float f) { return (uint64_t)((uint32_t)kw_fkey(f) ^ 0x80000000u); }
__device__ __forceinline__ float kw_unfkey64(uint64_t k) {
  const int i = (int)((uint32_t)k ^ 0x80000000u);
  return __int_as_float(i ^ ((i >> 31) & 0x7FFFFFFF));
}
// row groups stage the fp64 smoothing factors in SMEM for rows up to 8192
// channels (14 B per channel with the x row and the fp32 factors)
__host__ __device__ constexpr bool kw_stage64(int d_in) { return d_in <= 8192; }
constexpr int KW_RED_SITES = 6;  // SMEM key blocks per row group: sites x WPR x 8 keys

// compute_params (quantizer.py:118-135) returning 1 / S as well
__device__ __forceinline__ bool kw_params(double lo, double hi, const QSpecDev& s, double* S,
                                          int* zp, double* rS) {
  bool ok;
  if (s.sym) {
    const double amax = fmax(fabs(lo), fabs(hi));
    *S = amax > 0.0 ? __ddiv_rn(amax, (double)s.qmax) : 1.0;
    *zp = 0;
    ok = *S > 0.0;
    if (!ok) *S = 1.0;
    *rS = __ddiv_rn(1.0, *S);
  } else {
    double span = __dsub_rn(hi, lo);
    if (span == 0.0) {
      lo = fmin(lo, 0.0);
      hi = fmax(hi, 0.0);
      span = __dsub_rn(hi, lo);
    }
    *S = span > 0.0 ? __ddiv_rn(span, (double)(s.qmax - s.qmin)) : 1.0;
    ok = *S > 0.0;
    if (!ok) *S = 1.0;
    *rS = __ddiv_rn(1.0, *S);
    const double z = fmin(fmax(rha_quotient(-lo, *S, *rS), (double)s.qmin), (double)s.qmax);
    *zp = (int)z;
  }
  return ok;
}

// Fast-path constants of a group from its exact parameters (see the header).
// The fast path does not clip: elements that would clip lie beyond qmax +
// 1/2 (or below qmin - 1/2) in code units; while the extremes overshoot those
// points by at most ulp / 4, every such element is inside the flagged window
// and takes the exact (clipping) path. Larger overshoots (rows far from zero
// relative to their span) run exactly.
__device__ __forceinline__ KwConsts kw_consts2(double lo, double hi, double S, double rS, int zp,
                                              const QSpecDev& s, double err_extra) {
  KwConsts c;
  const double vl = lo * rS, vh = hi * rS;  // within 2 ulp of lo / S, hi / S
  const double vmax = fmax(fabs(vl), fabs(vh));
  const double err = vmax * 4.76837158203125e-07 + err_extra;  // 2^-21
  c.safe = vmax < 1048576.0;
  // k: the smallest k in [10, 22] with 2^(k-1) > vmax + 2, from the exponent
  // of vmax + 2 (2^e <= vmax + 2 < 2^(e+1) -> k = e + 2); powers of two by
  // their bit patterns (no loop, no ldexp / division on the row's critical path)
  const double vm2 = vmax + 2.0;
  int k = 22;
  if (vm2 < 4194304.0) k = min(22, max(10, ((__double2hiint(vm2) >> 20) & 0x7FF) - 1023 + 2));
  const double ulp = __hiloint2double((k - 23 + 1023) << 20, 0);
  const double rulp = __hiloint2double((23 - k + 1023) << 20, 0);
  c.F = (uint32_t)(23 - k);
  c.fm = (1u << c.F) - 1u;
  const double Wd = floor((err + 0.5 * ulp) * rulp) + 1.0;  // exact: rulp = 1 / ulp is a power of two
  if (!(Wd < (double)(1 << (c.F - 2)))) c.safe = 0;
  const double W = c.safe ? Wd : 1.0;
  c.W2 = (uint32_t)(2.0 * W);
  const int zq = s.centered ? 0 : zp;
  const double b = 1.5 * __hiloint2double((k + 1023) << 20, 0) + (double)zq;
  c.rs = (float)rS;
  c.base = (float)b;
  c.C = (float)(b + 0.5 + W * ulp);
  const double over = vh + (double)zp - ((double)s.qmax + 0.5);
  const double under = ((double)s.qmin - 0.5) - (vl + (double)zp);
  if (over > 0.25 * ulp || under > 0.25 * ulp) c.safe = 0;
  return c;
}

struct KwOut {  // outlier group parameters broadcast to the warp
  double S, rS;
  int zp, safe;
};
__device__ __forceinline__ RowParams kw_rowparams(double S, double rS, int zp, int safe,
                                                  const QSpecDev& s) {
  RowParams r;
  r.S = S;
  r.rS = rS;
  r.zp = zp;
  r.cz = K1_MAGIC + (double)zp;
  r.qmin = s.qmin;
  r.qmax = s.qmax;
  r.safe = safe != 0;
  return r;
}

// per-lane fp64 extremes of one outlier path (channels lane, lane + 32, ...)
template <typename T>
__device__ __forceinline__ void kw_outlier_ext(const T* xrow, const int* cols, const double* d, int n,
                                               double& lo, double& hi, bool& nan, int k0 = -1,
                                               int step = 32) {
  lo = INFINITY;
  hi = -INFINITY;
  for (int k = k0 < 0 ? (int)(threadIdx.x & 31) : k0; k < n; k += step) {
    const double z = __dmul_rn((double)kw_x<T>(xrow, __ldg(cols + k)), __ldg(d + k));
    nan |= z != z;
    lo = fmin(lo, z);
    hi = fmax(hi, z);
  }
}

// power of two rho with max(S, St, Sv) in [rho, 2 rho), and 1 / rho
__device__ __forceinline__ void kw_rho(double m, double& rho, double& rrho) {
  const int hi = __double2hiint(m) & 0x7FF00000;
  rho = __hiloint2double(hi, 0);
  rrho = __hiloint2double(0x7FE00000 - hi, 0);
}

// The z (then f) row of a warp in SMEM: two float4 planes, so lane-strided
// 16-byte accesses are bank-conflict free.
struct KwZ {
  float4* a;
  float4* b;
  __device__ __forceinline__ void put(int j, const float (&z)[8]) const {
    a[j] = make_float4(z[0], z[1], z[2], z[3]);
    b[j] = make_float4(z[4], z[5], z[6], z[7]);
  }
  __device__ __forceinline__ void get(int j, float (&z)[8]) const {
    const float4 u = a[j], w = b[j];
    z[0] = u.x; z[1] = u.y; z[2] = u.z; z[3] = u.w;
    z[4] = w.x; z[5] = w.y; z[6] = w.z; z[7] = w.w;
  }
};

// SMF: the MAC fractions f of a text row are kept in SMEM between pass E and
// pass G as 16-bit fixed point (f * 2^15, offset-binary), so pass G does not
// recompute the row: the extra rounding (<= 2^-16) enters the MAC tie window
// (kw_consts2 err_extra); rows whose window would get too wide recompute.
//
// WPR > 1 (decode-sized calls, few rows): the CTA's WPR warps share one row,
// chunks strided over all WPR x 32 threads; warp reductions are completed
// across the group through SMEM (kw_gmin), the per-row parameters are
// computed redundantly by every warp (deterministic) and stored by warp 0.
// PF (warp rows only): each pass issues the next chunk's loads one iteration
// ahead. For few rows per warp on wide rows, where a warp's serial passes
// are the critical path; it costs registers (occupancy) at full load.
template <typename T, bool SMF, int WPR, bool SYNC = false, bool G64 = false, bool PF = false>
__global__ void __launch_bounds__(WPR > 1 ? WPR * 32 : SYNC ? KW_THREADS_SYNC : KW_THREADS,
                                  WPR > 1 ? 1 : SYNC ? 2 : 8)  // warp rows: 64 registers, 32 warps per SM
    k1w_kernel(const K1Params p, int d_in) {
  static_assert(!(SMF && WPR > 1), "SMEM MAC fractions are per-warp rows");
  extern __shared__ __align__(16) uint8_t kw_smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nwc = blockDim.x >> 5;
  const int gl = WPR > 1 ? (int)threadIdx.x : lane;  // thread within the row group
  constexpr int GT = WPR > 1 ? WPR * 32 : 32;          // threads per row group
  const bool w0 = WPR == 1 || wl == 0;                 // the group's storing warp
  const int nchunks = d_in >> 3;
  uint32_t* q = reinterpret_cast<uint32_t*>(kw_smem) + wl * KW_QCAP;
  uint4* fs = SMF ? reinterpret_cast<uint4*>(kw_smem + nwc * KW_QCAP * 4) + (size_t)wl * nchunks
                  : nullptr;
  uint64_t* red = reinterpret_cast<uint64_t*>(kw_smem + nwc * KW_QCAP * 4);  // WPR > 1
  int* s_slot = reinterpret_cast<int*>(red + KW_RED_SITES * WPR * 8);
  // WPR > 1: the row (x) and its fp32 smoothing factors staged in SMEM by
  // pass A; the later passes read them there
  uint4* xs = reinterpret_cast<uint4*>(red + KW_RED_SITES * WPR * 8 + 2);
  float4* ds = reinterpret_cast<float4*>(xs + nchunks);
  // (the fp32 factors are staged only when the launch asks: for wide rows
  // with several rows per CTA the SMEM buys more co-resident rows instead)
  const bool sd = WPR > 1 && p.kw_stage_d;
  // ... and, for rows up to 8192 channels, the fp64 smoothing factors too, so
  // the exact paths (band candidates, flagged chunks, MAC residuals) read
  // SMEM instead of making global round trips on the row's critical path
  // (one bulk copy per CTA, issued before the first row and awaited just
  // before the first exact path)
  double* d64s = reinterpret_cast<double*>(ds + 2 * nchunks);
  uint64_t* d64bar = red + KW_RED_SITES * WPR * 8 + 1;
  const bool st64 = sd && kw_stage64(d_in) && ((reinterpret_cast<uintptr_t>(p.d_main) & 15) == 0);
  const KwD dm{st64 ? d64s : p.d_main, st64};
  if (st64 && threadIdx.x == 0) {
    mbar_init(d64bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(d64bar, (uint32_t)d_in * 8u);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(d64s)),
                 "l"(p.d_main), "r"((uint32_t)d_in * 8u), "r"(smem_u32(d64bar))
                 : "memory");
  }
  [[maybe_unused]] const int gw = WPR > 1 ? (int)blockIdx.x : (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = WPR > 1 ? (int)gridDim.x : (int)((gridDim.x * blockDim.x) >> 5);
  const bool cen = p.act.centered != 0, cena = p.aux.centered != 0;
  // dependents (the decode GEMVs) may launch now and prefetch their weights
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // rows: warp w of the grid takes rows w, w + #warps, ... (row groups: CTA b
  // takes rows b, b + #CTAs, ...). The body is a do-while(0): `continue`
  // ends the row. SYNC: a barrier per row round keeps the CTA's 16 warps in
  // the same code region, so they share instruction-cache lines (the
  // kernel is i-cache bound: `no_instruction` is its top stall). Measured
  // at d_in = 3584: 0.695 -> 0.61 ms; at 18944 rows vary more and the
  // barrier costs more than it saves (3.31 -> 4.6 ms), so it is not used.
  const int rstep = WPR > 1 ? (int)gridDim.x : nw;
  // the tag of the storing lane's next row, loaded a row ahead (its value
  // decides the MAC slot claim at the row's start)
  const int rb0 = WPR > 1 ? (int)blockIdx.x : (int)(blockIdx.x * nwc);
  uint8_t tg_next = 1;
  if (lane == 0 && w0 && p.tags && rb0 + (WPR > 1 ? 0 : wl) < p.T) tg_next = p.tags[rb0 + (WPR > 1 ? 0 : wl)];
  for (int rb = rb0; rb < p.T; rb += rstep) {
    const int row = WPR > 1 ? rb : rb + wl;
    const uint8_t tg_row = tg_next;
    if (lane == 0 && w0 && p.tags && row + rstep < p.T) tg_next = p.tags[row + rstep];
    if constexpr (WPR > 1) __syncthreads();  // the previous row's SMEM reads are done
    if (row < p.T) do {
    KW_STAMP(0)
    const T* xrow = reinterpret_cast<const T*>(p.x) + (int64_t)row * p.ldx;
    const uint4* xg = reinterpret_cast<const uint4*>(xrow);
    const T* xr = WPR > 1 ? reinterpret_cast<const T*>(xs) : xrow;  // element reads after pass A
    auto kwl = [&](int j, float (&x)[8], float (&d)[8]) {
      if constexpr (WPR > 1) {
        if (sd) kw_load_s<T>(xs, ds, nchunks, j, x, d);
        else kw_load_xs<T>(p, xs, j, x, d);
      }
      else kw_load<T>(p, xg, j, x, d);
    };

    // the row's tag and MAC slot (an atomic with return: an L2 round trip)
    // are requested before pass A, so their latency hides under it
    int slot = -1;
    if (lane == 0 && w0) {
      const uint8_t tg = tg_row;
      if (tg > 1) atomicOr(p.err, ERR_BAD_TAG);
      if (p.use_mac && tg == 0) {
        if (p.mac_count) {
          slot = atomicAdd(p.mac_count, 1);  // consumed after pass A (in-order issue)
        } else if (p.text_idx) {
          slot = p.text_idx[row];
        }
      }
    }
    // row groups: the outlier channel indices and scales of this thread are
    // fetched before pass A, so only the x gather follows it
    int pc_t = -1, pc_v = -1;
    double pd_t = 0.0, pd_v = 0.0;
    if constexpr (WPR > 1) {
      if (gl < p.n_text) pc_t = __ldg(p.c_text + gl), pd_t = __ldg(p.d_text + gl);
      if (gl < p.n_vis) pc_v = __ldg(p.c_vis + gl), pd_v = __ldg(p.d_vis + gl);
    }
    // ------------------------------------------------ pass A: fp32 z and its extremes
    KwExt elo, ehi;  // ehi tracks -max
    kw_ext_init(elo);
    kw_ext_init(ehi);
    uint32_t nm = 0u;
    KwRaw pa{};
    if (PF && gl < nchunks) pa = kw_ldraw(p, xg, gl);
    // row groups: the outlier channels' x is gathered with the first chunk's
    // loads (its latency hides under pass A, not after it)
    uint16_t hx_t = 0, hx_v = 0;
    bool gathered = false;
    for (int j = gl; j < nchunks; j += GT) {
      uint4 w;
      float4 da, db;
      if constexpr (PF) {
        w = pa.w, da = pa.da, db = pa.db;
        if (j + GT < nchunks) pa = kw_ldraw(p, xg, j + GT);
      } else {
        w = kw_ldg(xg + j);
        da = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j);
        db = __ldg(reinterpret_cast<const float4*>(p.d_main32) + 2 * j + 1);
      }
      if constexpr (WPR > 1) {
        if (!gathered) {
          gathered = true;
          if (pc_t >= 0) hx_t = __ldg(reinterpret_cast<const uint16_t*>(xrow) + pc_t);
          if (pc_v >= 0) hx_v = __ldg(reinterpret_cast<const uint16_t*>(xrow) + pc_v);
        }
        xs[j] = w;
        if (sd) {
          ds[j] = da;
          ds[nchunks + j] = db;
        }
      }
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
    KW_STAMP(1)
    float L = kw_warp_minf(elo.m1), H = kw_warp_minf(ehi.m1);  // H = -max
    if (lane == 0 && w0 && slot >= 0 && p.mac_count) p.mac_rows[slot] = row;
    slot = __shfl_sync(0xffffffffu, slot, 0);

    // outlier paths: exact fp64 extremes (every warp of a group: few channels)
    double tlo, thi, vlo, vhi;
    double z_t = 0.0, z_v = 0.0;  // row groups: this thread's outlier z (reused for its code)
    bool nan = XW<T>::nonfinite(nm);
    // (a row group spreads the outlier channels over all its threads)
    if constexpr (WPR > 1) {
      kw_outlier_ext<T>(xrow, p.c_text, p.d_text, p.n_text, tlo, thi, nan, gl + GT, GT);
      kw_outlier_ext<T>(xrow, p.c_vis, p.d_vis, p.n_vis, vlo, vhi, nan, gl + GT, GT);
      if (!gathered) {
        if (pc_t >= 0) hx_t = __ldg(reinterpret_cast<const uint16_t*>(xrow) + pc_t);
        if (pc_v >= 0) hx_v = __ldg(reinterpret_cast<const uint16_t*>(xrow) + pc_v);
      }
      if (pc_t >= 0) {
        z_t = __dmul_rn((double)XW<T>::to_f2((uint32_t)hx_t).x, pd_t);
        nan |= z_t != z_t;
        tlo = fmin(tlo, z_t);
        thi = fmax(thi, z_t);
      }
      if (pc_v >= 0) {
        z_v = __dmul_rn((double)XW<T>::to_f2((uint32_t)hx_v).x, pd_v);
        nan |= z_v != z_v;
        vlo = fmin(vlo, z_v);
        vhi = fmax(vhi, z_v);
      }
    } else {
      kw_outlier_ext<T>(xrow, p.c_text, p.d_text, p.n_text, tlo, thi, nan);
      kw_outlier_ext<T>(xrow, p.c_vis, p.d_vis, p.n_vis, vlo, vhi, nan);
    }
    nan = __any_sync(0xffffffffu, nan);
    if constexpr (WPR > 1) {
      tlo = kw_warp_mind(tlo);
      thi = kw_warp_maxd(thi);
      vlo = kw_warp_mind(vlo);
      vhi = kw_warp_maxd(vhi);
      if (lane == 0 && wl == 0) *s_slot = slot;
      uint64_t k[7] = {kw_fkey64(L), kw_fkey64(H), nan ? 0ull : 1ull, okey_d(tlo), ~okey_d(thi),
                       okey_d(vlo), ~okey_d(vhi)};
      kw_gmin<WPR, 7>(red, k);
      L = kw_unfkey64(k[0]);
      H = kw_unfkey64(k[1]);
      nan = k[2] == 0;
      tlo = ounkey_d(k[3]);
      thi = ounkey_d(~k[4]);
      vlo = ounkey_d(k[5]);
      vhi = ounkey_d(~k[6]);
      slot = *s_slot;
    }
    KW_STAMP(2)
    if (nan || !isfinite(L) || !isfinite(H)) {
      if (lane == 0 && w0) atomicOr(p.err, ERR_NONFINITE);
      continue;
    }
    if constexpr (WPR == 1) {
      tlo = kw_warp_mind(tlo);
      thi = kw_warp_maxd(thi);
      vlo = kw_warp_mind(vlo);
      vhi = kw_warp_maxd(vhi);
    }
    if ((p.n_text > 0 && !(isfinite(tlo) && isfinite(thi))) ||
        (p.n_vis > 0 && !(isfinite(vlo) && isfinite(vhi)))) {
      if (lane == 0 && w0) atomicOr(p.err, ERR_NONFINITE);
      continue;
    }

    if (dm.smem) mbar_wait(d64bar, 0);  // the staged fp64 factors (first row of the CTA)
    // ------------------------------------------------ exact main extremes: candidates
    // are the elements within 2^-21 of the fp32 extremes (one chunk per lane, or all
    // of the lane's chunks when its second-best chunk is also in the band)
    const float bl = L + fabsf(L) * KW_BAND + 1e-30f;
    const float bh = H + fabsf(H) * KW_BAND + 1e-30f;
    double lo64 = INFINITY, hi64 = -INFINITY;
    if (elo.m1 <= bl || ehi.m1 <= bh) {
      const bool all = elo.m2 <= bl || ehi.m2 <= bh || (elo.m1 <= bl && ehi.m1 <= bh && elo.c1 != ehi.c1);
      for (int j = all ? gl : (elo.m1 <= bl ? elo.c1 : ehi.c1); j < nchunks; j += GT) {
        float z[8], x[8], d[8];
        kwl(j, x, d);
        kw_mulz(x, d, z);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (z[u] <= bl || -z[u] <= bh) {
            double z64;
            z64 = __dmul_rn((double)kw_x<T>(xr, 8 * j + u), dm[8 * j + u]);
            if (z[u] <= bl) lo64 = fmin(lo64, z64);
            if (-z[u] <= bh) hi64 = fmax(hi64, z64);
          }
        }
        if (!all) break;
      }
    }
    lo64 = kw_warp_mind(lo64);
    hi64 = kw_warp_maxd(hi64);
    if constexpr (WPR > 1) {
      uint64_t k[2] = {okey_d(lo64), ~okey_d(hi64)};
      kw_gmin<WPR, 2>(red + 1 * WPR * 8, k);
      lo64 = ounkey_d(k[0]);
      hi64 = ounkey_d(~k[1]);
    }

    KW_STAMP(3)
    // ------------------------------------------------ group parameters, lane-parallel:
    // lane 0 main (act spec), lane 1 text, lane 2 vision (aux spec)
    KwConsts c{};
    double gS = 1.0, grS = 1.0;
    int gzp = 0, gsafe = 0;
    {
      const bool g_main = lane == 0, g_vis = lane == 2;
      const double glo = g_main ? lo64 : g_vis ? vlo : tlo;
      const double ghi = g_main ? hi64 : g_vis ? vhi : thi;
      const QSpecDev gs = g_main ? p.act : p.aux;
      if (lane < 3 && (lane == 0 || (lane == 1 ? p.n_text : p.n_vis) > 0)) {
        if (!kw_params(glo, ghi, gs, &gS, &gzp, &grS) && w0) atomicOr(p.err, ERR_SCALE_ZERO);
        c = kw_consts2(glo, ghi, gS, grS, gzp, gs, 0.0);
        gsafe = fmax(fabs(glo), fabs(ghi)) * grS < 536870912.0;  // 2^29 (quant_rn range)
      }
    }
    c = kw_shfl(c, 0);
    const double S = kw_shfl_d(gS, 0);
    [[maybe_unused]] double rSm = 0.0;  // the main group's 1 / S (compensated MAC pass)
    if constexpr (G64) rSm = kw_shfl_d(grS, 0);
    const int zp = __shfl_sync(0xffffffffu, gzp, 0);
    const RowParams rt = kw_rowparams(kw_shfl_d(gS, 1), kw_shfl_d(grS, 1),
                                      __shfl_sync(0xffffffffu, gzp, 1),
                                      __shfl_sync(0xffffffffu, gsafe, 1), p.aux);
    const RowParams rv = kw_rowparams(kw_shfl_d(gS, 2), kw_shfl_d(grS, 2),
                                      __shfl_sync(0xffffffffu, gzp, 2),
                                      __shfl_sync(0xffffffffu, gsafe, 2), p.aux);
    double rho, rrho;
    kw_rho(fmax(S, fmax(p.n_text > 0 ? rt.S : 0.0, p.n_vis > 0 ? rv.S : 0.0)), rho, rrho);
    if (!w0) {
    } else if (lane == 0) {
      p.s_main[row] = S;
      if (p.sf_main) p.sf_main[row] = (float)S;
      p.zp_main[row] = zp;
      if (p.rho) {
        p.rho[row] = (float)rho;
        p.lrs_main[row] = (float)(S * rrho);
      }
    } else if (lane == 1 && p.n_text > 0) {
      p.s_text[row] = rt.S;
      p.sf_text[row] = (float)rt.S;
      p.zp_text[row] = rt.zp;
    } else if (lane == 2 && p.n_vis > 0) {
      p.s_vis[row] = rv.S;
      p.sf_vis[row] = (float)rv.S;
      p.zp_vis[row] = rv.zp;
    }
    const KwRow r{S, zp};

    KW_STAMP(4)
    // ------------------------------------------------ outlier codes + aux segments
    // (a row group spreads both outlier paths over all its threads)
    if (p.n_text > 0)
      outlier_codes(p, row, xr, p.c_text, p.d_text, p.n_text, p.ld_text, p.a_text, rt,
                    rt.S * rrho, p.lr_off_t, p.kt16, WPR > 1 ? gl : -1, GT, pc_t >= 0 ? &z_t : nullptr);
    if (p.n_vis > 0)
      outlier_codes(p, row, xr, p.c_vis, p.d_vis, p.n_vis, p.ld_vis, p.a_vis, rv, rv.S * rrho,
                    p.lr_off_v, p.kv16, WPR > 1 ? gl : -1, GT, pc_v >= 0 ? &z_v : nullptr);
    if (p.k_lr > 0) {  // the low-rank columns of the aux operand row: LR1 fills them
      uint4* lr = reinterpret_cast<uint4*>(p.lr_a + (int64_t)row * p.k_lr + p.lr_off_s);
      for (int i = gl; i < (p.k_lr - p.lr_off_s) / 8; i += GT) lr[i] = make_uint4(0, 0, 0, 0);
    }

    KW_STAMP(5)
    // ------------------------------------------------ pass E: main codes (+ f = v - n)
    int8_t* arow = p.a_main + (int64_t)row * p.ld_main;
    const bool mac = slot >= 0;
    KwExt flo, fhi;
    kw_ext_init(flo);
    kw_ext_init(fhi);
    int qn = 0;
    if (c.safe) {
      KwRaw pe{};
      if (PF && gl < nchunks) pe = kw_ldraw(p, xg, gl);
      for (int j0 = 0; j0 < nchunks; j0 += GT) {
        const int j = j0 + gl;
        bool flag = false;
        KwRaw cur = pe;
        if (PF && j + GT < nchunks) pe = kw_ldraw(p, xg, j + GT);
        if (j < nchunks) {
          float z[8], x[8], d[8];
          uint32_t b[8];
          if constexpr (PF) kw_cvt<T>(cur, x, d);
          else kwl(j, x, d);
          kw_mulz(x, d, z);
          kw_vt(z, c, b);
          *reinterpret_cast<uint2*>(arow + 8 * j) = kw_pack_shift(b, c.F);
          flag = kw_minfrac(b, c.fm) <= c.W2;
          if (mac) {
            float f[8], nf[8];
            kw_frac(z, b, c, f);
            if (SMF) {  // f * 2^15 rounded, offset-binary u16 (|f| < 1 off the flagged window)
              uint32_t u[8];
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float2 t = kw_fma2(make_float2(f[2 * h], f[2 * h + 1]), make_float2(32768.f, 32768.f),
                                         make_float2(12582912.f, 12582912.f));
                u[2 * h] = __float_as_uint(t.x);
                u[2 * h + 1] = __float_as_uint(t.y);
              }
              fs[j] = make_uint4(__byte_perm(u[0], u[1], 0x5410) ^ 0x80008000u,
                                 __byte_perm(u[2], u[3], 0x5410) ^ 0x80008000u,
                                 __byte_perm(u[4], u[5], 0x5410) ^ 0x80008000u,
                                 __byte_perm(u[6], u[7], 0x5410) ^ 0x80008000u);
            }
            if (!flag) {
#pragma unroll
              for (int e = 0; e < 8; ++e) nf[e] = -f[e];
              kw_ext_upd(flo, kw_min8(f), j);
              kw_ext_upd(fhi, kw_min8(nf), j);
            }
          }
        }
        kw_enqueue(q, qn, flag, j);
      }
    }
    // exact fallback: the flagged chunks (queue), or every chunk (unsafe row /
    // queue overflow), elements spread over the lanes. MAC: the exact residual
    // of every element of these chunks joins the extreme candidates.
    KW_STAMP(6)
    bool allx = !c.safe || qn > KW_QCAP;
    if constexpr (WPR > 1) {  // any warp's queue overflow: the whole row runs exactly
      uint64_t k[1] = {allx ? 0ull : 1ull};
      kw_gmin<WPR, 1>(red + 2 * WPR * 8, k);
      allx = k[0] == 0;
    }
    KW_STAMP(7)
#ifdef KW_DEBUG  // fallback counters in the status block (tools/k1_debug.py)
    if (lane == 0) {
      atomicAdd(p.err + 1, qn);
      if (allx) atomicAdd(p.err + 2, 1);
      if (!c.safe) atomicAdd(p.err + 5, 1);
    }
#endif
    const int qnE = allx ? 0 : qn;
    const int nfix = 8 * (allx ? nchunks : qn);
    __syncwarp();
    double xlo = INFINITY, xhi = -INFINITY;
    for (int i = allx ? gl : lane; i < nfix; i += allx ? GT : 32) {
      const int ch = 8 * (allx ? i >> 3 : (int)q[i >> 3]) + (i & 7);
      double z64;
      const int qc = kw_exact_main(p, dm, kw_x<T>(xr, ch), ch, r, z64);
      arow[ch] = (int8_t)(cen ? qc - zp : qc);
      if (mac) {
        const double e64 = __dsub_rn(z64, __dmul_rn((double)(qc - zp), S));
        xlo = fmin(xlo, e64);
        xhi = fmax(xhi, e64);
      }
    }
    KW_STAMP(8)
    if (!mac) continue;

    // ------------------------------------------------ MAC: exact residual extremes
    float FL = kw_warp_minf(flo.m1), FH = kw_warp_minf(fhi.m1);
    if constexpr (WPR > 1) {
      uint64_t k[2] = {kw_fkey64(FL), kw_fkey64(FH)};
      kw_gmin<WPR, 2>(red + 3 * WPR * 8, k);
      FL = kw_unfkey64(k[0]);
      FH = kw_unfkey64(k[1]);
    }
    // |f - e / S| <= vmax 2^-22 (+ the fp32 rounding of f): an absolute band
    KW_STAMP(9)
    const float vmaxf = fmaxf(fabsf(L), fabsf(H)) * c.rs * 1.0001f + 1.0f;
    const float fband = 2.0f * vmaxf * KW_BAND + 1e-12f;
    const float bfl = FL + fband, bfh = FH + fband;
    double elo64 = xlo, ehi64 = xhi;
    if (!allx && (flo.m1 <= bfl || fhi.m1 <= bfh)) {
      const bool all = flo.m2 <= bfl || fhi.m2 <= bfh || (flo.m1 <= bfl && fhi.m1 <= bfh && flo.c1 != fhi.c1);
      for (int j = all ? gl : (flo.m1 <= bfl ? flo.c1 : fhi.c1); j < nchunks; j += GT) {
        float f[8], x[8], d[8], z[8];
        uint32_t b[8];
        kwl(j, x, d);
        kw_mulz(x, d, z);
        kw_vt(z, c, b);
        kw_frac(z, b, c, f);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (f[u] <= bfl || -f[u] <= bfh) {
            // off the tie window the fast path's n is the exact code (safe
            // row: no clipping), so e = z - n S needs no division
            const int ch = 8 * j + u;
            double e64;
            if ((b[u] & c.fm) > c.W2) {
              const float n = __uint_as_float(b[u] & ~c.fm) - c.base;
              e64 = __dsub_rn(__dmul_rn((double)kw_x<T>(xr, ch), dm[ch]), __dmul_rn((double)n, S));
            } else {
              e64 = kw_exact_e(p, dm, kw_x<T>(xr, ch), ch, r);
            }
            if (f[u] <= bfl) elo64 = fmin(elo64, e64);
            if (-f[u] <= bfh) ehi64 = fmax(ehi64, e64);
          }
        }
        if (!all) break;
      }
    }
    KW_STAMP(10)
    elo64 = kw_warp_mind(elo64);
    ehi64 = kw_warp_maxd(ehi64);
    if constexpr (WPR > 1) {
      uint64_t k[2] = {okey_d(elo64), ~okey_d(ehi64)};
      kw_gmin<WPR, 2>(red + 4 * WPR * 8, k);
      elo64 = ounkey_d(k[0]);
      ehi64 = ounkey_d(~k[1]);
    }
    KW_STAMP(11)
    KwConsts ce{};
    double Se = 1.0;
    int zpe = 0;
    float ratio = 1.f;
    int use_smf = 0, comp = 0;
    double rSe = 1.0;
    if (lane == 0) {
      if (!kw_params(elo64, ehi64, p.aux, &Se, &zpe, &rSe) && w0) atomicOr(p.err, ERR_SCALE_ZERO);
      // f carries |err| <= vmax 2^-22 in units of S (+ 2^-16 when read back from
      // the 16-bit SMEM copy): times S / Se in units of e / Se
      const double ef = (double)vmaxf * 2.384185791015625e-07;
      if (SMF) {
        ce = kw_consts2(elo64, ehi64, Se, rSe, zpe, p.aux, (ef + 1.52587890625e-05) * (S * rSe) * 1.01);
        use_smf = ce.safe && ce.W2 <= 16;
      }
      if (G64 && !SMF && p.d_main_lo32 && S * rSe > 64.0) {
        // wide aux codes: pass G forms f compensated (kw_frac_comp), |err| <=
        // 2^-23 + vmax 2^-40 in units of S, so the fp32 code pass keeps a
        // narrow window where the plain f would flag most chunks
        ce = kw_consts2(elo64, ehi64, Se, rSe, zpe, p.aux,
                        (1.1920928955078125e-07 + (double)vmaxf * 9.094947017729282e-13) * (S * rSe) * 1.01);
        comp = 1;
      } else if (!use_smf) {
        ce = kw_consts2(elo64, ehi64, Se, rSe, zpe, p.aux, ef * (S * rSe) * 1.01);
      }
      if (w0) {
        p.s_mac[slot] = Se;
        p.zp_mac[slot] = zpe;
        p.lrs_mac[slot] = (float)(Se * rrho);
      }
      ratio = (float)(S * rSe);
    }
    ce = kw_shfl(ce, 0);
    Se = kw_shfl_d(Se, 0);
    if constexpr (G64) rSe = kw_shfl_d(rSe, 0);
    zpe = __shfl_sync(0xffffffffu, zpe, 0);
    ratio = __shfl_sync(0xffffffffu, ratio, 0);
    use_smf = __shfl_sync(0xffffffffu, use_smf, 0);
    comp = __shfl_sync(0xffffffffu, comp, 0);

    KW_STAMP(12)
    // ------------------------------------------------ pass G: MAC residual codes
    int8_t* erow = p.a_mac + (int64_t)slot * p.ld_main;
    qn = qnE;  // the chunks flagged in pass E are exact-coded here as well
    [[maybe_unused]] const float rs_lo = G64 ? (float)(rSm - (double)c.rs) : 0.f;  // 1 / S = rs + rs_lo
    // fp64 pass G: when S / S_e is large (8-bit aux codes: ~255) the fp32
    // residual f = v - n carries too few bits for the MAC code (measured: 14 %
    // of chunks flagged, queue overflow on nearly every 18944-wide row). The
    // residual is then formed as the reference does -- e = fl64(z - fl64(m S))
    // with the exact main code m already in the row -- and e / S_e taken as
    // e * (1 / S_e) (<= 2 fp64 roundings from the reference's quotient): only
    // fractions within 2^-30 of one half are flagged for the exact division.
    // (a separate instantiation, chosen on the host for wide aux codes: its
    // registers would cost the 4-bit configurations occupancy)
    const bool g64 = G64 && !SMF && !allx && (!ce.safe || (ratio > 64.f && !comp));
    const bool allg = allx || (!ce.safe && !g64);
    if (g64) {
      for (int j0 = 0; j0 < nchunks; j0 += GT) {
        const int j = j0 + gl;
        bool flag = false;
        if (j < nchunks) {
          float x[8], d[8];
          kwl(j, x, d);
          const uint2 cm = *reinterpret_cast<const uint2*>(arow + 8 * j);  // exact main codes (pass E + fixups)
          const uint32_t cw[2] = {cm.x, cm.y};
          const double2* d64 = reinterpret_cast<const double2*>((dm.smem ? d64s : p.d_main) + 8 * j);
          uint32_t by[2] = {0u, 0u};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 dd = dm.smem ? d64[h] : __ldg(d64 + h);
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
              const int u = 2 * h + u2;
              const uint32_t byte = (cw[u >> 2] >> (8 * (u & 3))) & 0xFFu;
              const int m = cen ? (int)(int8_t)byte : (int)byte - zp;  // q - zp
              const double z64 = __dmul_rn((double)x[u], u2 ? dd.y : dd.x);
              const double e64 = __dsub_rn(z64, __dmul_rn((double)m, S));
              const double t = __dmul_rn(e64, rSe);
              const double a = fabs(t);
              const double fr = a - floor(a);
              flag |= !(fabs(fr - 0.5) > 9.313225746154785e-10);  // 2^-30 (also catches NaN)
              double qa = floor(a + 0.5);
              int qe = (int)(t < 0.0 ? -qa : qa) + zpe;
              qe = min(max(qe, p.aux.qmin), p.aux.qmax);
              by[u >> 2] |= ((uint32_t)(cena ? qe - zpe : qe) & 0xFFu) << (8 * (u & 3));
            }
          }
          *reinterpret_cast<uint2*>(erow + 8 * j) = make_uint2(by[0], by[1]);
        }
        kw_enqueue(q, qn, flag, j);
      }
    } else if (!allg) {
      constexpr bool PG = PF && !SMF;
      KwRaw pg{};
      if (PG && gl < nchunks) pg = kw_ldraw(p, xg, gl);
      for (int j0 = 0; j0 < nchunks; j0 += GT) {
        const int j = j0 + gl;
        bool flag = false;
        KwRaw cur = pg;
        if (PG && j + GT < nchunks) pg = kw_ldraw(p, xg, j + GT);
        if (j < nchunks) {
          uint32_t be[8];
          if (SMF && use_smf) {  // f from the 16-bit SMEM copy (pass-E-flagged chunks are queued)
            const uint4 w = fs[j];
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            const float r15 = ratio * 3.0517578125e-05f;  // ratio * 2^-15 (exact)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 n2 = kw_add2(make_float2(__uint_as_float(__byte_perm(ws[h], 0x4B40u, 0x5410)),
                                                    __uint_as_float(__byte_perm(ws[h], 0x4B40u, 0x5432))),
                                        make_float2(-12615680.f, -12615680.f));  // - (1.5 2^23 + 2^15)
              const float2 t = kw_fma2(n2, make_float2(r15, r15), make_float2(ce.C, ce.C));
              be[2 * h] = __float_as_uint(t.x);
              be[2 * h + 1] = __float_as_uint(t.y);
            }
          } else {
            // (chunks whose main codes were flagged in pass E are still in the
            // queue: qn starts at qnE, so their MAC codes are exact-coded too)
            float f[8], x[8], d[8], z[8];
            uint32_t b[8];
            if constexpr (PG) kw_cvt<T>(cur, x, d);
            else kwl(j, x, d);
            kw_mulz(x, d, z);
            kw_vt(z, c, b);
            if (G64 && comp) kw_frac_comp(p, j, x, d, z, b, c, rs_lo, f);
            else kw_frac(z, b, c, f);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 t = kw_fma2(make_float2(f[2 * h], f[2 * h + 1]), make_float2(ratio, ratio),
                                       make_float2(ce.C, ce.C));
              be[2 * h] = __float_as_uint(t.x);
              be[2 * h + 1] = __float_as_uint(t.y);
            }
          }
          *reinterpret_cast<uint2*>(erow + 8 * j) = kw_pack_shift(be, ce.F);
          flag = kw_minfrac(be, ce.fm) <= ce.W2;
        }
        kw_enqueue(q, qn, flag, j);
      }
    }
    KW_STAMP(13)
    bool allg2 = allg || qn > KW_QCAP;
    if constexpr (WPR > 1) {
      uint64_t k[1] = {allg2 ? 0ull : 1ull};
      kw_gmin<WPR, 1>(red + 5 * WPR * 8, k);
      allg2 = k[0] == 0;
    }
    KW_STAMP(14)
#ifdef KW_DEBUG
    if (lane == 0) {
      atomicAdd(p.err + 3, qn);
      if (allg2) atomicAdd(p.err + 2, 1 << 16);
      if (!ce.safe) atomicAdd(p.err + 6, 1);
    }
#endif
    const int ngix = 8 * (allg2 ? nchunks : qn);
    __syncwarp();
    for (int i = allg2 ? gl : lane; i < ngix; i += allg2 ? GT : 32) {
      const int ch = 8 * (allg2 ? i >> 3 : (int)q[i >> 3]) + (i & 7);
      const double e64 = kw_exact_e(p, dm, kw_x<T>(xr, ch), ch, r);
      const int qe = kw_exact_code(e64, Se, zpe, p.aux.qmin, p.aux.qmax);
      erow[ch] = (int8_t)(cena ? qe - zpe : qe);
    }
    __syncwarp();
    KW_STAMP(15)
    } while (0);
    if constexpr (WPR == 1 && SYNC) __syncthreads();
  }
}

inline size_t k1w_smem(int d_in, int warps, bool smf, int wpr = 1, bool stage_d = true) {
  const size_t per_ch = 2 + (stage_d ? 4 + (kw_stage64(d_in) ? 8 : 0) : 0);  // x [+ fp32 [+ fp64] factors]
  return (size_t)warps * (KW_QCAP * 4 + (smf ? (size_t)d_in * 2 : 0)) +
         (wpr > 1 ? (size_t)KW_RED_SITES * wpr * 8 * 8 + 16 + (size_t)d_in * per_ch : 0);
}

}  // namespace splitq
