// MOCD calibration statistics on sm_100a (reference: pkg/src/modquant/mocd.py).
//
//   absmax      per-channel max |x| over vision rows (vision_score, mocd.py:72-77)
//               and over all rows (init_transform statistic, transform.py:89)
//   rank_counts percentile_rank numerators (mocd.py:92-111): per text row, the
//               keys |x[row, cand]| are radix-sorted in SMEM and every count is
//               the upper bound of its own key (ties via <=)
//   text_score  _kmeans_1d per channel (mocd.py:114-150) evaluated exactly as
//               numpy does: order statistics from the channel's level histogram,
//               numpy 'linear' quantile init, per-level nearest-centre
//               assignment (ties to the lower index), centre means and the final
//               variance as numpy pairwise sums over the members in token order
//               (one subtree of the pairwise tree per thread, ts_pairwise_pass
//               below), so scores are bit-identical
//   topk        select_topk (mocd.py:80-89): k largest, ties to the lower index
// Multi-GPU (mocd_gpu.py): absmax is MAX-all-reduced, the integer rank counts
// are all-gathered in token order and channels are sharded for text_score.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <algorithm>
#include <mutex>
#include <cub/block/block_radix_sort.cuh>
#include <string>

#include "../../include/splitq.h"

namespace {

}  // namespace
#include "nvtx.cuh"

extern "C" int splitq_internal_fail(int code, const char* msg);  // splitq_capi.cu
namespace {

int mfail(int code, const char* msg) { return splitq_internal_fail(code, msg); }

template <typename T>
__device__ __forceinline__ double absval(const void* x, int64_t idx) {
  return fabs((double)reinterpret_cast<const T*>(x)[idx]);
}
template <>
__device__ __forceinline__ double absval<__half>(const void* x, int64_t idx) {
  return fabs((double)__half2float(reinterpret_cast<const __half*>(x)[idx]));
}
template <>
__device__ __forceinline__ double absval<__nv_bfloat16>(const void* x, int64_t idx) {
  return fabs((double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[idx]));
}

// ---------------------------------------------------------------- absmax
// max over non-negative doubles == max over their bit patterns
template <typename T>
__global__ void mocd_absmax_kernel(const void* x, int64_t ld, const uint8_t* tags, int64_t T_,
                                   int64_t D, int64_t rows_per_block, unsigned long long* vmax,
                                   unsigned long long* amax, int* status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(T_, r0 + rows_per_block);
  double mv = 0.0, ma = 0.0;
  bool bad = false;
  for (int64_t r = r0; r < r1; ++r) {
    const double a = absval<T>(x, r * ld + c);
    bad |= !(a <= 1.7976931348623157e308);
    ma = fmax(ma, a);
    if (tags[r] == 1) mv = fmax(mv, a);
  }
  if (bad) atomicOr(status, SPLITQ_STATUS_NONFINITE);
  atomicMax(&amax[c], (unsigned long long)__double_as_longlong(ma));
  atomicMax(&vmax[c], (unsigned long long)__double_as_longlong(mv));
}

// fp16 / bf16 rows, 8 channels per thread with 16-byte loads: |x| of a 16-bit
// float is its bit pattern with the sign cleared, and those patterns order
// like the values (NaN / inf patterns are the largest), so the maxima are
// SIMD u16 maxima; each thread converts its 8 maxima to fp64 once at the end.
template <typename T>
__global__ void __launch_bounds__(256) mocd_absmax16_kernel(const void* x, int64_t ld,
                                                            const uint8_t* tags, int64_t T_,
                                                            int64_t D, int64_t rows_per_block,
                                                            unsigned long long* vmax,
                                                            unsigned long long* amax, int* status) {
  const int64_t c8 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (8 * c8 >= D) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(T_, r0 + rows_per_block);
  uint32_t va[4] = {0u, 0u, 0u, 0u}, vv[4] = {0u, 0u, 0u, 0u};
  const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(x) + 8 * c8);
  const int64_t ldv = ld / 8;
#pragma unroll 4
  for (int64_t r = r0; r < r1; ++r) {
    const uint4 w = __ldg(base + r * ldv);
    const uint32_t ws[4] = {w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu, w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu};
    const bool vis = __ldg(tags + r) == 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      va[i] = __vmaxu2(va[i], ws[i]);
      vv[i] = __vmaxu2(vv[i], vis ? ws[i] : 0u);
    }
  }
  const uint32_t inf = sizeof(T) == 2 && std::is_same<T, __half>::value ? 0x7C00u : 0x7F80u;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ha = (va[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
    const uint32_t hv = (vv[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
    bad |= ha >= inf;
    const int64_t c = 8 * c8 + i;
    if (c < D) {
      const double da = std::is_same<T, __half>::value
                            ? (double)__half2float(__ushort_as_half((unsigned short)ha))
                            : (double)__uint_as_float(ha << 16);
      const double dv = std::is_same<T, __half>::value
                            ? (double)__half2float(__ushort_as_half((unsigned short)hv))
                            : (double)__uint_as_float(hv << 16);
      atomicMax(&amax[c], (unsigned long long)__double_as_longlong(da));
      atomicMax(&vmax[c], (unsigned long long)__double_as_longlong(dv));
    }
  }
  if (bad) atomicOr(status, SPLITQ_STATUS_NONFINITE);
}

__global__ void mocd_tag_check_kernel(const uint8_t* tags, int64_t T_, int* status) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T_;
       i += (int64_t)gridDim.x * blockDim.x)
    if (tags[i] > 1) atomicOr(status, SPLITQ_STATUS_TAG);
}

// ---------------------------------------------------------------- rank counts
template <typename T>
struct KeyOf {
  using type = uint32_t;
  static __device__ __forceinline__ uint32_t get(const void* x, int64_t i) {
    return __float_as_uint((float)absval<T>(x, i));  // exact for f16 / bf16 / f32
  }
};
template <>
struct KeyOf<double> {
  using type = unsigned long long;
  static __device__ __forceinline__ unsigned long long get(const void* x, int64_t i) {
    return (unsigned long long)__double_as_longlong(absval<double>(x, i));
  }
};

constexpr int RC_THREADS = 256;

template <typename T, int ITEMS>
__global__ void __launch_bounds__(RC_THREADS) mocd_rank_counts_kernel(
    const void* x, int64_t ld, const int* text_rows, const int* n_text, const int* cand,
    int n_cand, uint16_t* counts) {
  using Key = typename KeyOf<T>::type;
  using Sort = cub::BlockRadixSort<Key, RC_THREADS, ITEMS>;
  extern __shared__ __align__(16) uint8_t rc_smem[];
  typename Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(rc_smem);
  Key* sorted = reinterpret_cast<Key*>(rc_smem + (sizeof(typename Sort::TempStorage) + 15) / 16 * 16);
  const int i = blockIdx.x;
  if (i >= *n_text) return;
  const int64_t xrow = (int64_t)text_rows[i] * ld;
  Key keys[ITEMS];
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const int j = threadIdx.x * ITEMS + u;
    keys[u] = j < n_cand ? KeyOf<T>::get(x, xrow + cand[j]) : (Key)~(Key)0;
  }
  Sort(tmp).Sort(keys);
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) sorted[threadIdx.x * ITEMS + u] = keys[u];
  __syncthreads();
  uint16_t* out = counts + (int64_t)i * n_cand;
  for (int j = threadIdx.x; j < n_cand; j += RC_THREADS) {
    const Key v = KeyOf<T>::get(x, xrow + cand[j]);
    int lo = 0, hi = n_cand;  // first position with sorted > v
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sorted[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    out[j] = (uint16_t)lo;
  }
}

template <typename T, int ITEMS>
size_t rc_smem_bytes() {
  using Key = typename KeyOf<T>::type;
  using Sort = cub::BlockRadixSort<Key, RC_THREADS, ITEMS>;
  return (sizeof(typename Sort::TempStorage) + 15) / 16 * 16 + sizeof(Key) * RC_THREADS * ITEMS;
}

template <typename T, int ITEMS>
int launch_rc(const void* x, int64_t ld, const int* rows, const int* n_text, int64_t max_text,
              const int* cand, int n_cand, uint16_t* counts, cudaStream_t s) {
  const size_t smem = rc_smem_bytes<T, ITEMS>();
  if (smem > 220 * 1024) return mfail(SPLITQ_ERR_UNSUPPORTED, "too many candidate channels");
  static bool attr[64] = {};  // per device (the attribute is per context)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return mfail(SPLITQ_ERR_CUDA, "cudaGetDevice");
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    if (cudaFuncSetAttribute(mocd_rank_counts_kernel<T, ITEMS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return mfail(SPLITQ_ERR_CUDA, "cudaFuncSetAttribute (rank counts)");
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  mocd_rank_counts_kernel<T, ITEMS><<<(unsigned)max_text, RC_THREADS, smem, s>>>(
      x, ld, rows, n_text, cand, n_cand, counts);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK
                                           : mfail(SPLITQ_ERR_CUDA, "rank counts launch failed");
}

template <typename T>
int launch_rc_items(const void* x, int64_t ld, const int* rows, const int* n_text,
                    int64_t max_text, const int* cand, int n_cand, uint16_t* counts,
                    cudaStream_t s) {
  const int need = (n_cand + RC_THREADS - 1) / RC_THREADS;
  if (need <= 2) return launch_rc<T, 2>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 4) return launch_rc<T, 4>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 8) return launch_rc<T, 8>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 16) return launch_rc<T, 16>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 32) return launch_rc<T, 32>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 48) return launch_rc<T, 48>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  if (need <= 80) return launch_rc<T, 80>(x, ld, rows, n_text, max_text, cand, n_cand, counts, s);
  return mfail(SPLITQ_ERR_UNSUPPORTED, "at most 20480 candidate channels");
}

// 16-bit inputs (fp16 / bf16): |x| is the bit pattern with the sign cleared,
// and those 15-bit keys order like the values, so a row's counts come from a
// histogram over all 32768 keys (two 16-bit bins per word, 64 KB of SMEM),
// its inclusive prefix sum, and one lookup per candidate: the count of keys
// <= the candidate's own key (searchsorted side='right', mocd.py:109-110).
// No sort and no binary search per element.
constexpr int RC16_THREADS = 512;
constexpr int RC16_WORDS = 16384;  // 32768 bins
size_t rc16_smem_bytes() { return (size_t)RC16_WORDS * 4 + 64 * 4; }

__global__ void __launch_bounds__(RC16_THREADS) mocd_rank_counts16_kernel(
    const void* x, int64_t ld, const int* text_rows, const int* n_text, const int* cand, int n_cand,
    uint16_t* counts) {
  extern __shared__ __align__(16) uint32_t rc16_smem[];
  uint32_t* h = rc16_smem;                   // [RC16_WORDS]: bins 2w (low half), 2w + 1 (high half)
  uint32_t* wsum = rc16_smem + RC16_WORDS;   // [RC16_THREADS / 32]
  const int i = blockIdx.x;
  if (i >= *n_text) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* xr = reinterpret_cast<const uint16_t*>(x) + (int64_t)text_rows[i] * ld;
  for (int w = tid; w < RC16_WORDS; w += RC16_THREADS) h[w] = 0u;
  __syncthreads();
  for (int j = tid; j < n_cand; j += RC16_THREADS) {
    const uint32_t k = (uint32_t)__ldg(xr + __ldg(cand + j)) & 0x7FFFu;
    atomicAdd(h + (k >> 1), 1u << (16 * (k & 1)));
  }
  __syncthreads();
  // inclusive prefix over the 32768 bins: thread t owns words [32 t, 32 t + 32)
  constexpr int PER = RC16_WORDS / RC16_THREADS;
  uint32_t* mine = h + tid * PER;
  uint32_t tot = 0;
#pragma unroll 8
  for (int q = 0; q < PER; ++q) {
    const uint32_t w = mine[q];
    tot += (w & 0xFFFFu) + (w >> 16);
  }
  uint32_t inc = tot;  // block exclusive scan of the per-thread totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < RC16_THREADS / 32 ? wsum[lane] : 0u, iv = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += y;
    }
    if (lane < RC16_THREADS / 32) wsum[lane] = iv - v;
  }
  __syncthreads();
  uint32_t run = wsum[warp] + inc - tot;  // keys in the bins before this thread's
#pragma unroll 8
  for (int q = 0; q < PER; ++q) {
    const uint32_t w = mine[q];
    const uint32_t lo = run + (w & 0xFFFFu), hi = lo + (w >> 16);
    mine[q] = lo | (hi << 16);  // cumulative counts <= n_cand < 65536
    run = hi;
  }
  __syncthreads();
  uint16_t* out = counts + (int64_t)i * n_cand;
  for (int j = tid; j < n_cand; j += RC16_THREADS) {
    const uint32_t k = (uint32_t)__ldg(xr + __ldg(cand + j)) & 0x7FFFu;
    out[j] = (uint16_t)((h[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);
  }
}

int launch_rc16(const void* x, int64_t ld, const int* rows, const int* n_text, int64_t max_text,
                const int* cand, int n_cand, uint16_t* counts, cudaStream_t s) {
  const size_t smem = rc16_smem_bytes();
  static bool attr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return mfail(SPLITQ_ERR_CUDA, "cudaGetDevice");
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    if (cudaFuncSetAttribute(mocd_rank_counts16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return mfail(SPLITQ_ERR_CUDA, "cudaFuncSetAttribute (rank counts)");
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  mocd_rank_counts16_kernel<<<(unsigned)max_text, RC16_THREADS, smem, s>>>(x, ld, rows, n_text, cand,
                                                                          n_cand, counts);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK
                                           : mfail(SPLITQ_ERR_CUDA, "rank counts launch failed");
}

// ---------------------------------------------------------------- transpose
__global__ void transpose_u16_kernel(const uint16_t* in, int64_t rows, int64_t cols,
                                     uint16_t* out, int64_t ld_out) {
  __shared__ uint16_t tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ld_out + r] = tile[threadIdx.x][dy];
  }
}

// ---------------------------------------------------------------- exact k-means
// numpy float64 pairwise summation (oracle/mocd_oracle.py pairwise_sum /
// PairwiseStream are the reference-checked models).
// numpy's 8-accumulator combine of a pairwise-sum leaf
__device__ __forceinline__ double ts_combine8(const double* r) {
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

constexpr int TS_THREADS = 512;
constexpr int TS_KMAX = 8;

// Parallel exact pairwise sums of member sequences in token order.
//
// The reference sums cluster members (and the final squared deviations) with
// numpy's pairwise algorithm over the members in token order. Its tree
// depends only on the member count m: a node of more than 128 terms splits
// into n2 = (m/2) & ~7 and m - n2; a node of at most 128 is a leaf (8
// accumulators, then the remainder). With T = 2^D threads, thread t takes the
// subtree reached from the root by the D bits of t (or nothing, when a leaf
// is reached early and t's remaining bits are not zero), sums it sequentially
// with the same recursion (ts_subtree), and the D top levels are folded
// in SMEM level by level, left + right -- bit-identical to the serial sum.
// A pass first counts each cluster's members in every thread's contiguous
// token segment; the scanned counts locate a subtree's first member.
#ifdef TS_TRACE  // cycles per pass step, printed by channel 0 (debug builds)
__device__ unsigned long long ts_trace[8];
#define TS_T0() long long _t = clock64();
#define TS_T(i) if (threadIdx.x == 0 && blockIdx.x == 0) { long long _n = clock64(); ts_trace[i] += _n - _t; _t = _n; }
#else
#define TS_T0()
#define TS_T(i)
#endif
constexpr int TS_DEPTH = 9;  // log2(TS_THREADS)
static_assert((1 << TS_DEPTH) == TS_THREADS, "one subtree per thread");

struct TsShared {
  int* seg;          // [TS_THREADS][TS_KMAX] member counts -> exclusive bases
  double* val;       // [TS_THREADS] subtree sums
  uint16_t* cmp;     // this CTA's member slots: cluster j, segment t at cmp[j * cs + t * S]
  uint16_t* sbuf;    // SMEM store buffers: 8 members per (cluster, thread), written out 16 B at a time
  int64_t cs;        // per-cluster region (elements): TS_THREADS * S, S <= cs / TS_THREADS
  int nj[TS_KMAX];
  double tot[TS_KMAX];
  int dirty;  // MODE 0: bit j set -> cluster j's member set changed since its last sum
};

// Member test and value of token value v for pass `mode`:
//   0: cluster j members (asg[v] == j), value v / nc
//   1: every token, value (v / nc - cen[asg[v]])^2           (final variance)
//   2: every token, value v / nc                             (np.var: sum)
//   3: every token, value (v / nc - cen[0])^2                (np.var: deviations)
template <int MODE>
__device__ __forceinline__ bool ts_member(int v, const int8_t* asg, int j) {
  return MODE != 0 || asg[v] == j;
}
// A rank count's value fl64(v / nc) (mocd.py:111). With fast set, the host
// has checked, for every v in [0, nc], that the division-free form
// q = fl(v rnc), x = fma(fma(-q, nc, v), rnc, q) (rnc = fl(1 / nc)) equals
// the IEEE quotient, so the per-token division goes away bit-identically.
__device__ __forceinline__ double ts_x(int v, double nc, double rnc, bool fast) {
  const double dv = (double)v;
  if (!fast) return dv / nc;
  const double q = __dmul_rn(dv, rnc);
  return __fma_rn(__fma_rn(-q, nc, dv), rnc, q);
}
template <int MODE>
__device__ __forceinline__ double ts_value(int v, double nc, double rnc, bool fast, const int8_t* asg,
                                           const double* cen) {
  const double x = ts_x(v, nc, rnc, fast);
  if (MODE == 0 || MODE == 2) return x;
  const double d = x - (MODE == 1 ? cen[asg[v]] : cen[0]);
  return __dmul_rn(d, d);  // numpy squares first, then sums: no FMA contraction
}

// Sequential token reader: 16-byte loads (8 tokens) when the row is aligned.
struct TokReader {
  const uint16_t* col;
  int pos;
  bool vec;
  uint4 buf;
  __device__ void start(const uint16_t* c, int p, bool v) {
    col = c;
    pos = p;
    vec = v;
    if (vec && (pos & 7)) buf = __ldg(reinterpret_cast<const uint4*>(col) + (pos >> 3));
  }
  __device__ __forceinline__ int next() {
    if (!vec) return col[pos++];
    if ((pos & 7) == 0) buf = __ldg(reinterpret_cast<const uint4*>(col) + (pos >> 3));
    const int q = pos & 7;
    const uint32_t w = q < 2 ? buf.x : q < 4 ? buf.y : q < 6 ? buf.z : buf.w;
    ++pos;
    return (int)((q & 1) ? (w >> 16) : (w & 0xFFFFu));
  }
};

// Cluster j's members in token order from the compacted slots: segment s
// holds its members contiguously at base + s * S (16-byte aligned), and the
// scanned bases give each segment's count.
struct GapReader {
  const uint16_t* base;
  const int* seg;  // exclusive bases, [TS_THREADS][TS_KMAX]
  int j, m, S, s, i, cnt;
  TokReader rd;
  __device__ __forceinline__ int count(int t) const {
    const int b = seg[t * TS_KMAX + j];
    return (t + 1 < TS_THREADS ? seg[(t + 1) * TS_KMAX + j] : m) - b;
  }
  // member index st lies in segment t0 (the last whose base <= st)
  __device__ void start(const uint16_t* b, const int* sg, int jj, int mm, int SS, int t0, int st) {
    base = b, seg = sg, j = jj, m = mm, S = SS, s = t0;
    i = st - seg[t0 * TS_KMAX + j];
    cnt = count(s);
    rd.start(base + (int64_t)s * S, i, true);
  }
  bool stale = false;  // rd not positioned at i (after a next8)
  __device__ __forceinline__ int next() {
    while (i == cnt) {
      ++s;
      i = 0;
      cnt = count(s);
      rd.start(base + (int64_t)s * S, 0, true);
      stale = false;
    }
    if (stale) {
      rd.start(base + (int64_t)s * S, i, true);
      stale = false;
    }
    ++i;
    return rd.next();
  }
  // the next 8 members at once when they lie in the current segment: two
  // aligned 16-byte loads and a funnel shift by the offset (the scratch is
  // padded past its end for the second load); false -> use next()
  __device__ __forceinline__ bool next8(int (&v)[8]) {
    if (i + 8 > cnt) return false;
    const uint4* p4 = reinterpret_cast<const uint4*>(base + (int64_t)s * S) + (i >> 3);
    const uint4 a = __ldg(p4), b = __ldg(p4 + 1);
    const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const int k = (i & 7) >> 1, sh = 16 * (i & 1);
    uint32_t y[5];  // y[q] = x[k + q]
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const uint32_t x0 = x[q], x1 = x[q + 1], x2 = x[q + 2], x3 = x[min(q + 3, 7)];
      y[q] = k == 0 ? x0 : k == 1 ? x1 : k == 2 ? x2 : x3;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t w = __funnelshift_r(y[q], y[q + 1], sh);
      v[2 * q] = (int)(w & 0xFFFFu);
      v[2 * q + 1] = (int)(w >> 16);
    }
    i += 8;
    stale = true;
    return true;
  }
};

// Pairwise sum of the next m member values from the reader (numpy recursion);
// SKIP: the reader yields every token and non-members are skipped here.
template <int MODE, bool SKIP, class R>
__device__ double ts_subtree(R& rd, int m, int j, double nc, double rnc, bool fast, const int8_t* asg,
                            const double* cen) {
  auto next = [&]() -> double {
    int v = rd.next();
    if (SKIP)
      while (!ts_member<MODE>(v, asg, j)) v = rd.next();
    return ts_value<MODE>(v, nc, rnc, fast, asg, cen);
  };
  auto leaf = [&](int len) -> double {
    double res = 0.0;
    if (len < 8) {
      for (int q = 0; q < len; ++q) res += next();
      return res;
    }
    double r[8];
    const int body = len - len % 8;
    if constexpr (std::is_same<R, GapReader>::value) {  // compacted members: 8 at a time
      int v8[8];
      if (rd.next8(v8)) {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = ts_value<MODE>(v8[u], nc, rnc, fast, asg, cen);
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = next();
      }
      for (int q = 8; q < body; q += 8) {
        if (rd.next8(v8)) {
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] += ts_value<MODE>(v8[u], nc, rnc, fast, asg, cen);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] += next();
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = next();
      for (int q = 8; q < body; q += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] += next();
      }
    }
    res = ts_combine8(r);
    for (int q = body; q < len; ++q) res += next();
    return res;
  };
  if (m <= 128) return leaf(m);
  // explicit recursion: pending right-subtree lengths and left sums
  int len_[24], n2_[24], ph_[24];
  double left_[24];
  int d = 0, cur = m;
  double s;
  for (;;) {
    while (cur > 128) {
      int n2 = cur / 2;
      n2 -= n2 % 8;
      len_[d] = cur, n2_[d] = n2, ph_[d] = 0;
      ++d;
      cur = n2;
    }
    s = leaf(cur);
    while (d > 0 && ph_[d - 1] == 1) {
      --d;
      s = left_[d] + s;
    }
    if (d == 0) return s;
    ph_[d - 1] = 1;
    left_[d - 1] = s;
    cur = len_[d - 1] - n2_[d - 1];
  }
}

// Exact pairwise sums for clusters 0..nk-1 (MODE 0) or the single all-token
// sequence (MODE 1-3, nk = 1): results in sh.tot[j] and sh.nj[j].
template <int MODE>
__device__ void ts_pairwise_pass(const uint16_t* col, int n, int nk, double nc, double rnc, bool fast,
                                 const int8_t* asg, const double* cen, TsShared& sh, bool vec) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = ((n + TS_THREADS - 1) / TS_THREADS + 7) & ~7;  // segments of whole 16-byte vectors
  const int t0 = min(n, tid * S), t1 = min(n, t0 + S);
  TS_T0()
  if (MODE == 0) {
    // one read of the segment: each member's value goes to its cluster's
    // slot for this segment, in token order (16-bit counters packed in two
    // words: no indexed local array); the counts are then scanned per
    // cluster over the segments
    uint64_t c_lo = 0, c_hi = 0;
    uint16_t* my = sh.cmp + (int64_t)tid * S;
    // members collect 8 at a time in this thread's SMEM buffer of their
    // cluster and leave as one 16-byte store (2-byte stores scattered over
    // 32 slots per warp instruction were the pass's bound)
    uint16_t* sb = sh.sbuf + tid * 8;  // cluster a: sb + a * TS_THREADS * 8
    auto emit = [&](int a, int idx, int v) {
      uint16_t* b = sb + a * (TS_THREADS * 8);
      b[idx & 7] = (uint16_t)v;
      if ((idx & 7) == 7)
        *reinterpret_cast<uint4*>(my + a * sh.cs + (idx & ~7)) = *reinterpret_cast<const uint4*>(b);
    };
    auto put = [&](int v) {
      const int a = asg[v];
      const int sh16 = 16 * (a & 3);
      const int idx = (int)(((a < 4 ? c_lo : c_hi) >> sh16) & 0xFFFFu);
      emit(a, idx, v);
      if (a < 4) c_lo += 1ull << sh16;
      else c_hi += 1ull << sh16;
    };
    if (vec) {  // t0 is a multiple of 8: whole 16-byte vectors, 8 tokens each
      const uint4* c4 = reinterpret_cast<const uint4*>(col);
      for (int p = t0; p < t1; p += 8) {
        const uint4 w = __ldg(c4 + (p >> 3));
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
        if (p + 8 <= t1) {
          // the 8 level -> cluster lookups first (independent), then the
          // counter chain and the stores
          int vv[8], aa[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) vv[u] = (int)((ww[u >> 1] >> (16 * (u & 1))) & 0xFFFFu);
#pragma unroll
          for (int u = 0; u < 8; ++u) aa[u] = asg[vv[u]];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int a = aa[u], sh16 = 16 * (a & 3);
            const int idx = (int)(((a < 4 ? c_lo : c_hi) >> sh16) & 0xFFFFu);
            emit(a, idx, vv[u]);
            if (a < 4) c_lo += 1ull << sh16;
            else c_hi += 1ull << sh16;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p + u < t1) put((int)((ww[u >> 1] >> (16 * (u & 1))) & 0xFFFFu));
        }
      }
    } else {
      for (int i = t0; i < t1; ++i) put(col[i]);
    }
    for (int j = 0; j < nk; ++j) {  // the partial buffers (< 8 members each)
      const int cnt = (int)(((j < 4 ? c_lo : c_hi) >> (16 * (j & 3))) & 0xFFFFu);
      const uint16_t* b = sb + j * (TS_THREADS * 8);
      for (int q = cnt & ~7; q < cnt; ++q) my[j * sh.cs + q] = b[q & 7];
    }
#pragma unroll
    for (int j = 0; j < TS_KMAX; ++j)
      sh.seg[tid * TS_KMAX + j] = (int)(((j < 4 ? c_lo : c_hi) >> (16 * (j & 3))) & 0xFFFFu);
    __syncthreads();
    if (warp < nk) {  // warp j: exclusive scan of cluster j's counts
      const int j = warp;
      constexpr int PER = TS_THREADS / 32;
      int v[PER], run = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] = sh.seg[(lane * PER + q) * TS_KMAX + j], run += v[q];
      int inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int base = inc - run;
#pragma unroll
      for (int q = 0; q < PER; ++q) sh.seg[(lane * PER + q) * TS_KMAX + j] = base, base += v[q];
      if (lane == 31) sh.nj[j] = inc;
    }
  } else if (tid == 0) {
    sh.nj[0] = n;
  }
  __syncthreads();
  TS_T(0)
  for (int j = 0; j < nk; ++j) {
    // a cluster whose members did not change keeps its sum (and its mean):
    // the same members in the same token order give the same pairwise sum
    if (MODE == 0 && !((sh.dirty >> j) & 1)) continue;
    const int m = sh.nj[j];
    // this thread's subtree: the D bits of tid from the root
    int st = 0, len = m;
    bool own = m > 0;
    for (int l = 0; l < TS_DEPTH && own; ++l) {
      if (len <= 128) {  // a leaf above the thread level: its leftmost thread owns it
        own = (tid & ((1 << (TS_DEPTH - l)) - 1)) == 0;
        break;
      }
      int n2 = len / 2;
      n2 -= n2 % 8;
      if ((tid >> (TS_DEPTH - 1 - l)) & 1) st += n2, len -= n2;
      else len = n2;
    }
    double v = 0.0;
    if (own) {
      if (MODE == 0) {  // member st through the segment bases, then the compacted slots
        int lo = 0, hi = TS_THREADS - 1;  // last segment whose base <= st and with members
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sh.seg[mid * TS_KMAX + j] <= st) lo = mid;
          else hi = mid - 1;
        }
        GapReader gr;
        gr.start(sh.cmp + (int64_t)j * sh.cs, sh.seg, j, m, S, lo, st);
        v = ts_subtree<MODE, false>(gr, len, j, nc, rnc, fast, asg, cen);
      } else {
        TokReader rd;
        rd.start(col, st, vec);
        v = ts_subtree<MODE, true>(rd, len, j, nc, rnc, fast, asg, cen);
      }
    }
    sh.val[tid] = v;
    __syncthreads();
    TS_T(1)
    // fold the top D levels: node (l, p) = left slot p << (D - l) + right slot
    for (int l = TS_DEPTH - 1; l >= 0; --l) {
      if (tid < (1 << l)) {
        int nl = m;  // node (l, tid) length: descend l levels
        bool split = m > 0;
        for (int q = 0; q < l && split; ++q) {
          if (nl <= 128) {
            split = false;
            break;
          }
          int n2 = nl / 2;
          n2 -= n2 % 8;
          nl = ((tid >> (l - 1 - q)) & 1) ? nl - n2 : n2;
        }
        if (split && nl > 128)
          sh.val[tid << (TS_DEPTH - l)] = sh.val[tid << (TS_DEPTH - l)] + sh.val[(2 * tid + 1) << (TS_DEPTH - l - 1)];
      }
      __syncthreads();
    }
    if (tid == 0) sh.tot[j] = sh.val[0];
    __syncthreads();
    TS_T(2)
  }
#ifdef TS_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) ts_trace[4] += 1;
#endif
}

// One CTA per candidate channel c (c0 + blockIdx.x). counts_t: [n_cand x ld] uint16.
__global__ void __launch_bounds__(TS_THREADS, 2) mocd_text_score_kernel(
    const uint16_t* counts_t, int64_t ld, int n_cand, int n_text, int k_req, int max_iter, int c0,
    int c1, double* scores, double rnc, int fast_div, uint16_t* scratch, int64_t scratch_cta) {
  // SMEM: a bitmask of the levels present, then one region used twice: the
  // (cumulative) level histogram while the centres are initialised, then the
  // level -> cluster map, the segment counts and the subtree sums. The peak
  // is the histogram alone, so D = 18944 fits two CTAs per SM.
  extern __shared__ __align__(16) uint8_t ts_smem[];
  uint32_t* present = reinterpret_cast<uint32_t*>(ts_smem);               // [(n_cand + 32) / 32]
  uint8_t* region = ts_smem + (((n_cand + 32) / 32 * 4 + 15) & ~15);
  int* hist = reinterpret_cast<int*>(region);                              // [n_cand + 1] -> cumulative
  double* val = reinterpret_cast<double*>(region);                         // [TS_THREADS]        (after)
  int* seg = reinterpret_cast<int*>(val + TS_THREADS);                     // [TS_THREADS x KMAX] (after)
  int8_t* asg = reinterpret_cast<int8_t*>(seg + TS_THREADS * TS_KMAX);     // [n_cand + 1]        (after)
  uint16_t* sbuf = reinterpret_cast<uint16_t*>(
      (reinterpret_cast<uintptr_t>(asg + n_cand + 1) + 15) & ~uintptr_t(15));  // [k][TS_THREADS][8] (after)
  __shared__ TsShared sh;
  __shared__ double centers[TS_KMAX], new_centers[TS_KMAX];
  __shared__ int distinct, changed, dirty_next;
  // persistent CTAs (each owns one scratch slot of compacted member values)
  // take the channels c0 + blockIdx.x, + gridDim.x, ...
  for (int c = c0 + (int)blockIdx.x; c < c1; c += (int)gridDim.x) {
  __syncthreads();  // the previous channel's SMEM reads are done
  const uint16_t* col = counts_t + (int64_t)c * ld;
  const bool vec = (reinterpret_cast<uintptr_t>(col) & 15) == 0;  // 16-byte token loads
  const int tid = threadIdx.x;
  const double nc = (double)n_cand;
  const bool fast = fast_div != 0;
  if (tid == 0) {
    sh.seg = seg;
    sh.val = val;
    sh.cmp = scratch + (int64_t)blockIdx.x * scratch_cta;
    sh.sbuf = sbuf;
    sh.cs = (int64_t)TS_THREADS * ((((n_text + TS_THREADS - 1) / TS_THREADS) + 7) & ~7);
  }

  for (int v = tid; v <= n_cand; v += TS_THREADS) hist[v] = 0;
  for (int w = tid; w < (n_cand + 32) / 32; w += TS_THREADS) present[w] = 0;
  if (tid == 0) distinct = 0;
  __syncthreads();
  for (int i = tid; i < n_text; i += TS_THREADS) atomicAdd(&hist[col[i]], 1);
  __syncthreads();
  for (int v = tid; v <= n_cand; v += TS_THREADS)
    if (hist[v]) {
      atomicAdd(&distinct, 1);
      atomicOr(&present[v >> 5], 1u << (v & 31));
    }
  __syncthreads();
  // cumulative histogram (one thread; n_cand <= ~20k)
  if (tid == 0) {
    int acc = 0;
    for (int v = 0; v <= n_cand; ++v) {
      acc += hist[v];
      hist[v] = acc;
    }
  }
  __syncthreads();
  const int k = min(k_req, distinct);
  const int n = n_text;
  // from here on the region holds asg / seg / val (the histogram is only
  // read by the centre initialisation, before the switch below)
  auto release_hist = [&]() {
    __syncthreads();
    for (int v = tid; v <= n_cand; v += TS_THREADS) asg[v] = 0;
    __syncthreads();
  };

  if (k <= 1) {
    release_hist();
    // np.var(values): mean = sum / n, then mean((v - mean)^2) (pairwise sums)
    ts_pairwise_pass<2>(col, n, 1, nc, rnc, fast, asg, centers, sh, vec);
    if (tid == 0) centers[0] = sh.tot[0] / (double)n;
    __syncthreads();
    ts_pairwise_pass<3>(col, n, 1, nc, rnc, fast, asg, centers, sh, vec);
    if (tid == 0) scores[c] = sh.tot[0] / (double)n;
    continue;
  }

  // order statistic: value of the idx-th element of the sorted values
  auto order_stat = [&](int idx) -> double {
    int lo = 0, hi = n_cand;  // first level with cum > idx
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (hist[mid] > idx) hi = mid;
      else lo = mid + 1;
    }
    return ts_x(lo, nc, rnc, fast);
  };
  if (tid < k) {  // np.quantile(values, (2j - 1) / (2k)), method 'linear'
    const double q = (double)(2 * (tid + 1) - 1) / (double)(2 * k);
    const double vi = (double)(n - 1) * q;
    int lo, hi;
    if (vi >= (double)(n - 1)) {
      lo = hi = n - 1;
    } else {
      lo = (int)floor(vi);
      hi = lo + 1;
    }
    const double t = vi - floor(vi);
    const double a = order_stat(lo), b = order_stat(hi);
    const double diff = b - a;
    centers[tid] = t >= 0.5 ? b - diff * (1.0 - t) : a + diff * t;
  }
  release_hist();
  // level assignment: argmin |v - c_j|, ties to the lower index (np.argmin)
  auto assign_levels = [&](const double* cen, bool track) {
    for (int v = tid; v <= n_cand; v += TS_THREADS) {
      if (!((present[v >> 5] >> (v & 31)) & 1u)) continue;
      const double x = ts_x(v, nc, rnc, fast);
      int best = 0;
      double bd = fabs(x - cen[0]);
      for (int j = 1; j < k; ++j) {
        const double d = fabs(x - cen[j]);
        if (d < bd) {
          bd = d;
          best = j;
        }
      }
      if (track && asg[v] != (int8_t)best) {
        changed = 1;
        atomicOr(&dirty_next, (1 << asg[v]) | (1 << best));
      }
      asg[v] = (int8_t)best;
    }
  };
  assign_levels(centers, false);
  __syncthreads();
  if (tid == 0) sh.dirty = (1 << k) - 1;  // the first means come from the quantile centres
  for (int it = 0; it < max_iter; ++it) {
    if (tid == 0) changed = 0, dirty_next = 0;
    // members.mean() per cluster in token order (numpy pairwise), in parallel;
    // clusters whose members did not change keep their centre (the mean of
    // the same members, computed last iteration)
    ts_pairwise_pass<0>(col, n, k, nc, rnc, fast, asg, centers, sh, vec);
    if (tid < k)
      new_centers[tid] = !((sh.dirty >> tid) & 1) ? centers[tid]
                         : sh.nj[tid] > 0 ? sh.tot[tid] / (double)sh.nj[tid] : centers[tid];
    __syncthreads();
    assign_levels(new_centers, true);
    if (tid < k) centers[tid] = new_centers[tid];
    __syncthreads();
    const int ch = changed;
    if (tid == 0) sh.dirty = dirty_next;
    __syncthreads();  // every thread has read the flag before thread 0 resets it
    if (!ch) break;
  }
  // mean((values - centers[assign])^2)
  ts_pairwise_pass<1>(col, n, 1, nc, rnc, fast, asg, centers, sh, vec);
  if (tid == 0) scores[c] = sh.tot[0] / (double)n;
  }  // channels
#ifdef TS_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("TS_TRACE passes=%llu count+scan=%llu subtrees=%llu fold=%llu\n", ts_trace[4], ts_trace[0],
           ts_trace[1], ts_trace[2]);
#endif
}

// ---------------------------------------------------------------- top-k
// rank_i = #{j: s_j > s_i} + #{j < i: s_j == s_i}; selected iff rank_i < k.
__global__ void mocd_topk_mark_kernel(const double* s, int n, int k, int* flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double si = s[i];
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const double sj = s[j];
    rank += (sj > si) || (sj == si && j < i);
  }
  flags[i] = rank < k;
}
__global__ void mocd_topk_compact_kernel(const int* flags, int n, int64_t* out) {
  // single block: ascending indices of the selected entries
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const int f = i < n ? flags[i] : 0;
    const unsigned ballot = __ballot_sync(0xffffffffu, f);
    __shared__ int warp_tot[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_tot[warp] = __popc(ballot);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    if (f) out[off + __popc(ballot & ((1u << lane) - 1))] = i;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) base += warp_tot[w];
    __syncthreads();
  }
}

}  // namespace

extern "C" {

int splitq_mocd_absmax(const void* x, int x_dtype, int64_t x_ld, const uint8_t* tags,
                       int64_t tokens, int64_t dim, double* vision_max, double* all_max,
                       int32_t* status, void* stream_) {
  splitq::NvtxRange nv("splitq.mocd_absmax");
  if (!x || !tags || !vision_max || !all_max || !status)
    return mfail(SPLITQ_ERR_INVALID, "null argument");
  if (tokens <= 0 || dim <= 0) return mfail(SPLITQ_ERR_INVALID, "empty batch");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
  if (cudaMemsetAsync(vision_max, 0, dim * 8, s) != cudaSuccess ||
      cudaMemsetAsync(all_max, 0, dim * 8, s) != cudaSuccess ||
      cudaMemsetAsync(status, 0, 4, s) != cudaSuccess)
    return mfail(SPLITQ_ERR_CUDA, "cudaMemsetAsync failed");
  const int64_t rows_per_block = 256;
  dim3 grid((unsigned)((dim + 255) / 256), (unsigned)((tokens + rows_per_block - 1) / rows_per_block));
  auto vm = reinterpret_cast<unsigned long long*>(vision_max);
  auto am = reinterpret_cast<unsigned long long*>(all_max);
  const bool vec16 = (x_dtype == SPLITQ_F16 || x_dtype == SPLITQ_BF16) && dim % 8 == 0 &&
                     x_ld % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (vec16) {
    // 8 channels per thread; rows split so the grid covers ~8 waves of 148 SMs
    const int64_t cblocks = (dim / 8 + 255) / 256;
    int64_t rpb = std::max<int64_t>(64, (tokens * cblocks + 8 * 148 - 1) / (8 * 148));
    rpb = std::min<int64_t>(rpb, tokens);
    dim3 g2((unsigned)cblocks, (unsigned)((tokens + rpb - 1) / rpb));
    if (x_dtype == SPLITQ_F16)
      mocd_absmax16_kernel<__half><<<g2, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rpb, vm, am, status);
    else
      mocd_absmax16_kernel<__nv_bfloat16><<<g2, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rpb, vm, am, status);
    mocd_tag_check_kernel<<<64, 256, 0, s>>>(tags, tokens, status);
    return cudaGetLastError() == cudaSuccess ? SPLITQ_OK : mfail(SPLITQ_ERR_CUDA, "absmax launch failed");
  }
  switch (x_dtype) {
    case SPLITQ_F16:
      mocd_absmax_kernel<__half><<<grid, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rows_per_block, vm, am, status);
      break;
    case SPLITQ_BF16:
      mocd_absmax_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rows_per_block, vm, am, status);
      break;
    case SPLITQ_F32:
      mocd_absmax_kernel<float><<<grid, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rows_per_block, vm, am, status);
      break;
    case SPLITQ_F64:
      mocd_absmax_kernel<double><<<grid, 256, 0, s>>>(x, x_ld, tags, tokens, dim, rows_per_block, vm, am, status);
      break;
    default:
      return mfail(SPLITQ_ERR_INVALID, "bad x dtype");
  }
  mocd_tag_check_kernel<<<64, 256, 0, s>>>(tags, tokens, status);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK : mfail(SPLITQ_ERR_CUDA, "absmax launch failed");
}

int splitq_mocd_rank_counts(const void* x, int x_dtype, int64_t x_ld, const int32_t* text_rows,
                            const int32_t* n_text, int64_t max_text, const int32_t* cand,
                            int64_t n_cand, uint16_t* counts, void* stream_) {
  splitq::NvtxRange nv("splitq.mocd_rank_counts");
  if (!x || !text_rows || !n_text || !cand || !counts) return mfail(SPLITQ_ERR_INVALID, "null argument");
  if (n_cand <= 0) return mfail(SPLITQ_ERR_INVALID, "candidate channel set is empty");
  if (n_cand > 65535) return mfail(SPLITQ_ERR_UNSUPPORTED, "at most 65535 candidate channels");
  if (max_text <= 0) return SPLITQ_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
  const int nc = (int)n_cand;
  switch (x_dtype) {
    case SPLITQ_F16:  // 16-bit keys: histogram counts (SPLITQ_MOCD_RC_SORT=1: the sort path)
    case SPLITQ_BF16:
      if (!getenv("SPLITQ_MOCD_RC_SORT") && nc < 65536)
        return launch_rc16(x, x_ld, text_rows, n_text, max_text, cand, nc, counts, s);
      return x_dtype == SPLITQ_F16
                 ? launch_rc_items<__half>(x, x_ld, text_rows, n_text, max_text, cand, nc, counts, s)
                 : launch_rc_items<__nv_bfloat16>(x, x_ld, text_rows, n_text, max_text, cand, nc, counts, s);
    case SPLITQ_F32: return launch_rc_items<float>(x, x_ld, text_rows, n_text, max_text, cand, nc, counts, s);
    case SPLITQ_F64: return launch_rc_items<double>(x, x_ld, text_rows, n_text, max_text, cand, nc, counts, s);
    default: return mfail(SPLITQ_ERR_INVALID, "bad x dtype");
  }
}

int splitq_mocd_transpose_u16(const uint16_t* in, int64_t rows, int64_t cols, uint16_t* out,
                              int64_t ld_out, void* stream_) {
  if (!in || !out) return mfail(SPLITQ_ERR_INVALID, "null argument");
  if (rows <= 0 || cols <= 0) return SPLITQ_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_u16_kernel<<<grid, dim3(32, 8), 0, reinterpret_cast<cudaStream_t>(stream_)>>>(
      in, rows, cols, out, ld_out);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK : mfail(SPLITQ_ERR_CUDA, "transpose launch failed");
}

}  // extern "C"

// The text score's per-device scratch (compacted member values), grown on
// demand. The caller holds ts_mu from the request through the launch, so a
// larger request (which drains the device before freeing the old buffer)
// cannot free a buffer whose kernel has not been enqueued yet.
static std::mutex ts_mu;
static uint16_t* ts_scratch(int dev, size_t bytes) {
  static uint16_t* buf[64] = {};
  static size_t cap[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  if (cap[dev] < bytes) {
    if (buf[dev]) {
      cudaDeviceSynchronize();
      cudaFree(buf[dev]);
      buf[dev] = nullptr;
      cap[dev] = 0;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    buf[dev] = static_cast<uint16_t*>(p);
    cap[dev] = bytes;
  }
  return buf[dev];
}

extern "C" {

int splitq_mocd_text_score(const uint16_t* counts_t, int64_t ld, int64_t n_cand, int64_t n_text,
                           int k, int max_iter, int64_t c0, int64_t c1, double* scores,
                           void* stream_) {
  splitq::NvtxRange nv("splitq.mocd_text_score");
  if (!counts_t || !scores) return mfail(SPLITQ_ERR_INVALID, "null argument");
  if (k < 1) return mfail(SPLITQ_ERR_INVALID, "cluster count must be positive");
  if (k > n_text) return mfail(SPLITQ_ERR_INVALID, "cluster count exceeds number of text tokens");
  if (k > TS_KMAX) return mfail(SPLITQ_ERR_UNSUPPORTED, "at most 8 clusters on the GPU path");
  if (c1 <= c0) return SPLITQ_OK;
  const size_t bits = (size_t)(((n_cand + 32) / 32 * 4 + 15) & ~15);
  const size_t after = (size_t)TS_THREADS * 8 + (size_t)TS_THREADS * TS_KMAX * 4 + (size_t)(n_cand + 1) + 16 +
                       (size_t)k * TS_THREADS * 16;  // + the compaction store buffers
  const size_t smem = bits + std::max((size_t)(n_cand + 1) * 4, after) + 16;
  static bool attr[64] = {};  // per device (the attribute is per context)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return mfail(SPLITQ_ERR_CUDA, "cudaGetDevice");
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    if (cudaFuncSetAttribute(mocd_text_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024) != cudaSuccess)
      return mfail(SPLITQ_ERR_CUDA, "cudaFuncSetAttribute (text score)");
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  if (smem > 200 * 1024) return mfail(SPLITQ_ERR_UNSUPPORTED, "too many candidate channels");
  // the division-free rank values (ts_x) where they match the IEEE quotient
  // for every level of this denominator (checked here, host fma = device fma)
  const double nc = (double)n_cand, rnc = 1.0 / nc;
  int fast = 1;
  for (int64_t v = 0; v <= n_cand && fast; ++v) {
    const double dv = (double)v, q = dv * rnc;
    fast = std::fma(std::fma(-q, nc, dv), rnc, q) == dv / nc;
  }
  // persistent grid: the resident CTAs, each with a scratch slot for the
  // compacted member values of its channel (k regions of TS_THREADS
  // segments), kept per device and grown on demand
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mocd_text_score_kernel, TS_THREADS, smem) !=
          cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || per_sm < 1)
    return mfail(SPLITQ_ERR_CUDA, "text score occupancy");
  const int64_t grid = std::min<int64_t>(c1 - c0, (int64_t)per_sm * sms);
  const int64_t seg = (((n_text + TS_THREADS - 1) / TS_THREADS) + 7) & ~7;
  const int64_t per_cta = (int64_t)k * TS_THREADS * seg;
  std::lock_guard<std::mutex> lk(ts_mu);
  uint16_t* scratch = ts_scratch(dev, (size_t)(grid * per_cta + 16) * sizeof(uint16_t));  // + next8 read pad
  if (!scratch) return mfail(SPLITQ_ERR_CUDA, "text score scratch allocation");
  mocd_text_score_kernel<<<(unsigned)grid, TS_THREADS, smem, reinterpret_cast<cudaStream_t>(stream_)>>>(
      counts_t, ld, (int)n_cand, (int)n_text, k, max_iter, (int)c0, (int)c1, scores, rnc, fast, scratch,
      per_cta);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK : mfail(SPLITQ_ERR_CUDA, "text score launch failed");
}

int splitq_mocd_topk(const double* scores, int64_t n, int64_t k, int32_t* flags, int64_t* out,
                     void* stream_) {
  splitq::NvtxRange nv("splitq.mocd_topk");
  if (!scores || !flags || !out) return mfail(SPLITQ_ERR_INVALID, "null argument");
  if (k > n) return mfail(SPLITQ_ERR_INVALID, "k exceeds score vector length");
  if (k <= 0 || n <= 0) return SPLITQ_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
  mocd_topk_mark_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scores, (int)n, (int)k, flags);
  mocd_topk_compact_kernel<<<1, 1024, 0, s>>>(flags, (int)n, out);
  return cudaGetLastError() == cudaSuccess ? SPLITQ_OK : mfail(SPLITQ_ERR_CUDA, "topk launch failed");
}

}  // extern "C"
