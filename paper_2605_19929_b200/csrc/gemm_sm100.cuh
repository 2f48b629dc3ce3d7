// Split-linear GEMM for sm_100a: tcgen05 kind::i8 main GEMM with the
// text/vision outlier GEMMs and the low-rank (CWS + MAC) second stage fused
// into the same tile, accumulators in TMEM, dequantize-and-merge epilogue.
//
// Reference semantics (numpy float64, /root/reference/pkg/src/modquant):
//   y_m = x_hat @ b_m [+ (x_hat @ u_q) @ v_q]            layer.py:141-155
//   y_m[text] += (e_q @ uc_q) @ vc_q                      layer.py:157-166
//   y_t, y_v = Q(X_p d_p) @ Q(W_p / d_p) over all rows     layer.py:106-115,132-133
//   y = y_m + y_t + y_v                                    layer.py:171
// Every fake-quantized operand is (q - z) * S, so each integer GEMM is exact
// in int32 and the scales are applied per row / per column in the epilogue.
//
// One persistent CTA per SM, 6 warps:
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue (one TMEM lane = one output row per thread)
// Every tile is a sequence of "virtual k-stages" that share one SMEM ring:
//   [text chunks][vision chunks][low-rank chunks][main chunks]
// Each stage holds an A box (128 rows x 128 B) and a B box (BN rows x 128 B),
// both K-major in the 128-byte swizzle layout written by TMA.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100_ptx.cuh"

namespace splitq {

constexpr int GEMM_BM = 128;
constexpr int GEMM_STAGE_A_BYTES = GEMM_BM * 128;  // 16 KB
constexpr int GEMM_MAX_BN = 128;
constexpr int GEMM_STAGE_BYTES = GEMM_STAGE_A_BYTES + GEMM_MAX_BN * 128;  // 32 KB
constexpr int GEMM_STAGES = 6;
constexpr int GEMM_THREADS = 192;
constexpr int GEMM_TMEM_COLS = 512;
constexpr int GEMM_SMEM_BYTES = GEMM_STAGES * GEMM_STAGE_BYTES + 1024 /*align*/ + 256 /*bars*/;

enum EpiMode : int {
  EPI_SPLIT = 0,  // y = full split-linear merge (fp32 / fp16 / bf16 store)
  EPI_RAW = 1,    // raw accumulators: int32 main / text / vision, fp32 low-rank
  EPI_LR1 = 2,    // low-rank first stage: fp16 (row_scale * col_scale * acc) into the LR operand
};

enum OutDtype : int { OUT_F32 = 0, OUT_F16 = 1, OUT_BF16 = 2 };

enum StageKind : int { SK_TEXT = 0, SK_VIS = 1, SK_LR = 2, SK_MAIN = 3 };

struct GemmMaps {
  CUtensorMap a, b;    // main operands (int8)
  CUtensorMap at, bt;  // text outlier operands (int8)
  CUtensorMap av, bv;  // vision outlier operands (int8)
  CUtensorMap la, lb;  // low-rank second-stage operands (fp16)
};

struct GemmParams {
  int M;                   // rows; overridden by *m_count when m_count != nullptr
  const int* m_count;
  int N;                   // output columns
  int bn;                  // tile N (multiple of 16, <= GEMM_MAX_BN)
  int k_main;              // main K (int8 elements)
  int k_text, k_vis;       // outlier K (int8 elements, 0 = path absent)
  int k_lr;                // low-rank K (fp16 elements, multiple of 64, 0 = absent)
  uint32_t idesc_main, idesc_text, idesc_vis, idesc_lr;
  int mode;
  int out_dtype;
  // per-row epilogue operands (index = tile row)
  const float* row_s;      // main activation scale (EPI_SPLIT) / lr row scale (EPI_LR1)
  const int* row_zp;       // zero point when the A codes are u8 (else nullptr)
  const float* row_st;
  const int* row_zpt;
  const float* row_sv;
  const int* row_zpv;
  const float* row_rho;    // low-rank row normaliser
  // per-column epilogue operands
  const float* col_s;      // main weight scale / lr first-stage column scale
  const int* col_cs;       // column code sums (for u8 zero-point correction)
  const float* col_st;
  const int* col_cst;
  const float* col_sv;
  const int* col_csv;
  const float* col_kappa;  // low-rank column normaliser
  // outputs
  void* out;               // EPI_SPLIT: y [M x ldo]; EPI_LR1: fp16 LR operand; EPI_RAW: int32 main
  int64_t ldo;
  const int* row_map;      // EPI_LR1: output row = row_map[r] (nullptr = identity)
  int col_off;             // EPI_LR1: first output column
  int* raw_t;              // EPI_RAW extra outputs (nullable)
  int* raw_v;
  float* raw_f;
  int* err;                // device error word (EPI_LR1 range check)
};

__device__ __forceinline__ int num_chunks(int k_bytes) { return (k_bytes + 127) / 128; }

template <typename F>
__device__ __forceinline__ void for_each_stage(const GemmParams& p, F&& f) {
  // text / vision int8 chunks of 128 B, low-rank fp16 chunks of 64 elements,
  // main int8 chunks of 128 B.
  const int nt = num_chunks(p.k_text), nv = num_chunks(p.k_vis);
  const int nl = p.k_lr / 64, nm = num_chunks(p.k_main);
  for (int c = 0; c < nt; ++c) f(SK_TEXT, c, p.k_text - c * 128);
  for (int c = 0; c < nv; ++c) f(SK_VIS, c, p.k_vis - c * 128);
  for (int c = 0; c < nl; ++c) f(SK_LR, c, 128);
  for (int c = 0; c < nm; ++c) f(SK_MAIN, c, p.k_main - c * 128);
}

__device__ __forceinline__ float to_f32(uint32_t u) { return __uint_as_float(u); }

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    splitq_gemm_kernel(const __grid_constant__ GemmMaps maps, const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GEMM_STAGES * GEMM_STAGE_BYTES);
  uint64_t* empty = full + GEMM_STAGES;
  uint64_t* tmem_full = empty + GEMM_STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  const int M = p.m_count ? *p.m_count : p.M;
  const int m_tiles = (M + GEMM_BM - 1) / GEMM_BM;
  const int n_tiles = (p.N + p.bn - 1) / p.bn;
  const int num_tiles = m_tiles * n_tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < GEMM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 4);
    fence_mbar_init();
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
  }
  if (warp == 1) tmem_alloc(tmem_base_slot, GEMM_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (num_tiles == 0) {
    // nothing to do (e.g. no text rows for the MAC pass)
  } else if (warp == 0) {
    // ============================ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tx = GEMM_STAGE_A_BYTES + p.bn * 128;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles) * GEMM_BM;
        const int n0 = (tile % n_tiles) * p.bn;
        for_each_stage(p, [&](int kind, int c, int) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * GEMM_STAGE_BYTES;
          uint8_t* sb = sa + GEMM_STAGE_A_BYTES;
          mbar_arrive_expect_tx(&full[stage], tx);
          const CUtensorMap* ma = kind == SK_TEXT ? &maps.at
                                  : kind == SK_VIS ? &maps.av
                                  : kind == SK_LR  ? &maps.la
                                                   : &maps.a;
          const CUtensorMap* mb = kind == SK_TEXT ? &maps.bt
                                  : kind == SK_VIS ? &maps.bv
                                  : kind == SK_LR  ? &maps.lb
                                                   : &maps.b;
          const int kc = kind == SK_LR ? c * 64 : c * 128;  // element coordinate
          tma_load_2d(sa, ma, &full[stage], kc, m0);
          tma_load_2d(sb, mb, &full[stage], kc, n0);
          if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
        });
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tphase = 0;
      const uint32_t d_main = tmem_base;
      const uint32_t d_text = tmem_base + p.bn;
      const uint32_t d_vis = tmem_base + 2 * p.bn;
      const uint32_t d_lr = tmem_base + 3 * p.bn;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(tmem_empty, tphase ^ 1);
        tc_fence_after();
        for_each_stage(p, [&](int kind, int c, int krem) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * GEMM_STAGE_BYTES);
          const uint32_t b_addr = a_addr + GEMM_STAGE_A_BYTES;
          const uint64_t ad = sw128_kmajor_desc(a_addr);
          const uint64_t bd = sw128_kmajor_desc(b_addr);
          if (kind == SK_LR) {
            // 4 x (K = 16 fp16 = 32 B) per 128-B chunk
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_f16(d_lr, ad + 2 * k, bd + 2 * k, p.idesc_lr, (c | k) != 0);
          } else {
            const int nk = min(4, (krem + 31) / 32);  // K = 32 int8 per MMA
            const uint32_t d = kind == SK_TEXT ? d_text : kind == SK_VIS ? d_vis : d_main;
            const uint32_t id = kind == SK_TEXT ? p.idesc_text
                                : kind == SK_VIS ? p.idesc_vis
                                                 : p.idesc_main;
            for (int k = 0; k < nk; ++k) mma_i8(d, ad + 2 * k, bd + 2 * k, id, (c | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == GEMM_STAGES) { stage = 0; phase ^= 1; }
        });
        tc_commit(tmem_full);
        tphase ^= 1;
      }
    }
  } else {
    // ============================ epilogue (warps 2..5)
    const int lane_grp = warp & 3;  // TMEM lane quarter this warp may access
    const int r_local = lane_grp * 32 + lane;
    uint32_t tphase = 0;
    const bool has_t = p.k_text > 0, has_v = p.k_vis > 0, has_lr = p.k_lr > 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles) * GEMM_BM;
      const int n0 = (tile % n_tiles) * p.bn;
      const int row = m0 + r_local;
      const bool row_ok = row < M;
      mbar_wait(tmem_full, tphase);
      tphase ^= 1;
      tc_fence_after();

      float s_row = 0.f, st_row = 0.f, sv_row = 0.f, rho = 0.f;
      int zp = 0, zpt = 0, zpv = 0;
      if (row_ok) {
        if (p.row_s) s_row = p.row_s[row];
        if (p.row_zp) zp = p.row_zp[row];
        if (has_t) { st_row = p.row_st[row]; if (p.row_zpt) zpt = p.row_zpt[row]; }
        if (has_v) { sv_row = p.row_sv[row]; if (p.row_zpv) zpv = p.row_zpv[row]; }
        if (has_lr) rho = p.row_rho[row];
      }
      const uint32_t lane_addr = tmem_base + ((uint32_t)(lane_grp * 32) << 16);
      for (int c0 = 0; c0 < p.bn; c0 += 32) {
        uint32_t am[32], at[32], av[32], af[32];
        tmem_ld32(lane_addr + c0, am);
        if (has_t) tmem_ld32(lane_addr + p.bn + c0, at);
        if (has_v) tmem_ld32(lane_addr + 2 * p.bn + c0, av);
        if (has_lr) tmem_ld32(lane_addr + 3 * p.bn + c0, af);
        tmem_wait_ld();
        if (!row_ok) continue;
        if (p.mode == EPI_RAW) {
          int* o = reinterpret_cast<int*>(p.out);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + c0 + j;
            if (col < p.N) {
              const int64_t idx = (int64_t)row * p.ldo + col;
              o[idx] = (int)am[j];
              if (has_t && p.raw_t) p.raw_t[idx] = (int)at[j];
              if (has_v && p.raw_v) p.raw_v[idx] = (int)av[j];
              if (has_lr && p.raw_f) p.raw_f[idx] = to_f32(af[j]);
            }
          }
        } else if (p.mode == EPI_LR1) {
          __half* o = reinterpret_cast<__half*>(p.out);
          const int orow = p.row_map ? p.row_map[row] : row;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + c0 + j;
            if (col < p.N) {
              const int acc = (int)am[j] - (p.row_zp ? zp * p.col_cs[col] : 0);
              const float v = acc == 0 ? 0.f : s_row * p.col_s[col] * (float)acc;
              if (!(fabsf(v) <= 65504.f) && p.err) atomicOr(p.err, 8 /*ERR_LR_RANGE*/);
              o[(int64_t)orow * p.ldo + p.col_off + col] = __float2half_rn(v);
            }
          }
        } else {
          float y[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = min(n0 + c0 + j, p.N - 1);
            const int acc = (int)am[j] - (p.row_zp ? zp * p.col_cs[col] : 0);
            float v = s_row * p.col_s[col] * (float)acc;
            if (has_t) {
              const int a = (int)at[j] - (p.row_zpt ? zpt * p.col_cst[col] : 0);
              v += st_row * p.col_st[col] * (float)a;
            }
            if (has_v) {
              const int a = (int)av[j] - (p.row_zpv ? zpv * p.col_csv[col] : 0);
              v += sv_row * p.col_sv[col] * (float)a;
            }
            if (has_lr) v += rho * p.col_kappa[col] * to_f32(af[j]);
            y[j] = v;
          }
          const int64_t base = (int64_t)row * p.ldo + n0 + c0;
          const bool full_chunk = (n0 + c0 + 32 <= p.N) && ((p.ldo & 7) == 0);
          if (p.out_dtype == OUT_F32) {
            float* o = reinterpret_cast<float*>(p.out) + base;
            if (full_chunk) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(o + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
            } else {
              for (int j = 0; j < 32; ++j)
                if (n0 + c0 + j < p.N) o[j] = y[j];
            }
          } else if (p.out_dtype == OUT_F16) {
            __half* o = reinterpret_cast<__half*>(p.out) + base;
            if (full_chunk) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                uint4 pk;
                __half2 h0 = __floats2half2_rn(y[j], y[j + 1]);
                __half2 h1 = __floats2half2_rn(y[j + 2], y[j + 3]);
                __half2 h2 = __floats2half2_rn(y[j + 4], y[j + 5]);
                __half2 h3 = __floats2half2_rn(y[j + 6], y[j + 7]);
                pk.x = *reinterpret_cast<uint32_t*>(&h0);
                pk.y = *reinterpret_cast<uint32_t*>(&h1);
                pk.z = *reinterpret_cast<uint32_t*>(&h2);
                pk.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(o + j) = pk;
              }
            } else {
              for (int j = 0; j < 32; ++j)
                if (n0 + c0 + j < p.N) o[j] = __float2half_rn(y[j]);
            }
          } else {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + base;
            if (full_chunk) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                uint4 pk;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(y[j], y[j + 1]);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(y[j + 2], y[j + 3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(y[j + 4], y[j + 5]);
                __nv_bfloat162 h3 = __floats2bfloat162_rn(y[j + 6], y[j + 7]);
                pk.x = *reinterpret_cast<uint32_t*>(&h0);
                pk.y = *reinterpret_cast<uint32_t*>(&h1);
                pk.z = *reinterpret_cast<uint32_t*>(&h2);
                pk.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(o + j) = pk;
              }
            } else {
              for (int j = 0; j < 32; ++j)
                if (n0 + c0 + j < p.N) o[j] = __float2bfloat16_rn(y[j]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tmem_empty);
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, GEMM_TMEM_COLS);
  }
}

}  // namespace splitq
