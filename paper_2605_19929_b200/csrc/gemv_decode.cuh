// Decode-sized forwards: warp-MMA GEMV kernels for calls with at most
// GV_MAX_ROWS (8) token rows (one decoding step of a small batch).
//
// At a handful of token rows the work is one stream of the weights from HBM;
// the tcgen05 tile machinery (TMEM allocation, barrier set-up, a split-K
// finalize pass per GEMM, 128-row MMA tiles of which 8 rows are real) costs
// more than the stream. Here one launch per GEMM, no scratch:
//
//   gv_kernel<..., LR1=false>  y = S_a S_w (acc - zp cs) + rho kappa aux
//       main int8 GEMM (weights packed 4-bit or int8) + fp16 aux GEMM + the
//       SPLIT / RAW epilogue (g2_epi_split arithmetic)
//   gv_kernel<..., LR1=true>   the low-rank first stage (CWS / MAC): int8
//       GEMM + the g2_epi_lr1 epilogue (fp16 hi / lo into the aux operand)
//
// Layout. The output channels form blocks of 16 (the MMA's M); the token
// rows are the MMA's N = 8. A CTA (8 warps, persistent over channel blocks)
// stages the launch's activation rows in SMEM once, then streams each
// block's weight rows through a ring of SMEM stages filled by TMA (2-D boxes
// of 16 rows x 128 bytes, 128-byte swizzle) on mbarriers: a block is a
// sequence of units of up to GV_BPU boxes (main K first, then the aux K).
// In a unit the 8 warps split the (box, half) items; each item is 4 (packed
// 4-bit: 128 codes) or 2 (int8: 64 codes; fp16 aux: 32 halves) MMAs:
//   int8 : mma.sync.m16n8k32 s8 x (s8|u8) -> s32
//   aux  : mma.sync.m16n8k16 f16 x f16 -> f32
// The K order inside a box is permuted freely (a dot product does not care):
// thread (g, tig) reads 16-byte chunk 2 tig + half of its rows g and g + 8,
// which is bank-conflict free under the swizzle, and the activation pieces
// are staged in the same permuted order. Packed 4-bit words unpack to the
// MMA's int8 fragments with two logic ops each (sign extension by multiply).
// The warps' int32 partials meet in SMEM in warp order (exact); the fp32 aux
// partials likewise (deterministic; the order differs from the tensor path's
// MMA only within fp32 rounding).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>

#include "gemm2_sm100.cuh"
#include "sm100_ptx.cuh"

namespace splitq {

constexpr int GV_MAX_ROWS = 32;  // NT <= 4 MMA n-tiles of 8 token rows
constexpr int GV_WARPS = 8;                 // consumer (MMA) warps
constexpr int GV_THREADS = (GV_WARPS + 1) * 32;  // + one producer (TMA) warp
constexpr int GV_BPU = 8;         // 128-byte boxes per ring unit (16 KB stages)
constexpr int GV_MAX_STAGES = 12;
constexpr int GV_BOX_BYTES = 16 * 128;

struct GvArgs {
  const int8_t* a;      // activation codes [rows x lda] (natural channel order)
  int64_t lda;          // (bytes)
  int64_t a_bytes;      // valid bytes per activation row (<= lda)
  int nbox;             // main K boxes: 128 bytes of a weight row each
  int nbox_aux;         // aux K boxes: 64 halves each
  int units_main, units_aux;
  int stages;
  int act_stride, aux_stride;  // SMEM row strides of the staged activations (bytes)
  int srows;            // staged token rows (<= 8 NT): the launch's rows; the MMA's
                        // rows past them read the last staged row (their results are dropped)
  const __half* xa;     // aux operand rows [rows x k_aux] (SPLIT / RAW)
  // K split over CTAs (LR1: few channels, long K): ksplit CTAs per channel
  // block add their int32 partials into red [rows x N] (zeroed by the
  // caller) and the last to arrive (cnt[block * NT + n-tile]) applies the
  // epilogue
  int ksplit;
  int* red;
  unsigned* cnt;
};

struct GvMaps {
  CUtensorMap w;        // main weights [N x row bytes] (UINT8), box 16 x 128 B
  CUtensorMap x;        // aux weights [N x k_aux] (FLOAT16), box 16 x 64
};

// SMEM: the ring, staged activation rows (rows x act_stride), staged aux rows, barriers
__host__ __device__ inline int gv_smem_bytes(int rows, int act_stride, int aux_stride, int stages) {
  return rows * (act_stride + aux_stride) + stages * GV_BPU * GV_BOX_BYTES + 2 * GV_MAX_STAGES * 8 + 1024;
}

__device__ __forceinline__ uint32_t gv_sext4(uint32_t v) {  // 4 signed nibbles (low) -> 4 int8
  v &= 0x0F0F0F0Fu;
  return v | ((v & 0x08080808u) * 0x1Eu);
}
template <bool ASIGNED>
__device__ __forceinline__ void gv_mma_i8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  if (ASIGNED)
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void gv_mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void gv_bar_consumers() {  // named barrier of the 8 MMA warps
  asm volatile("bar.sync 1, %0;" ::"n"(GV_WARPS * 32) : "memory");
}

// The kernel body for one GEMM; bid / nbid: this CTA's index and the CTA
// count of the GEMM (a fused launch runs two GEMMs side by side).
template <bool PACKED, bool ASIGNED, bool LR1, int NT>
__device__ __forceinline__ void gv_body(const GvMaps& maps, const G2Params& p, const GvArgs& g, int blocks,
                                        int bid, int nbid) {
  extern __shared__ __align__(16) uint8_t gv_smem[];
  __shared__ int s_acc[GV_WARPS][32][4];
  __shared__ float s_aux[GV_WARPS][32][4];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tig = lane & 3;  // MMA fragment coordinates
  const int S = g.stages;
  // ring first (1024-byte aligned for the 128-byte swizzle), then the rows
  uint8_t* ring = gv_smem + ((1024u - (smem_u32(gv_smem) & 1023u)) & 1023u);
  uint8_t* sact = ring + S * GV_BPU * GV_BOX_BYTES;
  uint8_t* saux = sact + g.srows * g.act_stride;
  uint64_t* full = reinterpret_cast<uint64_t*>(saux + g.srows * g.aux_stride);
  uint64_t* empty = full + GV_MAX_STAGES;
  // units: main boxes first, then aux boxes; a K split takes a contiguous
  // range of the main units (LR1 only: no aux)
  const int ks_n = g.ksplit;
  const int um_per = (g.units_main + ks_n - 1) / ks_n;
  const int items = blocks * ks_n;
  auto unit_range = [&](int item, int& u0, int& u1) {
    const int ks = ks_n == 1 ? 0 : item % ks_n;
    u0 = ks * um_per;
    u1 = LR1 || ks_n > 1 ? min(g.units_main, u0 + um_per) : g.units_main + g.units_aux;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(full + s, 1), mbar_init(empty + s, GV_WARPS);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == GV_WARPS) {
    // ---- producer warp: weights do not depend on the preceding kernels, so
    // with programmatic dependent launch the ring fills while they finish
    if (lane == 0) {
      tma_prefetch(&maps.w);
      if (!LR1) tma_prefetch(&maps.x);
      int li = 0, st_i = 0;  // ring slot and fill round of unit li, kept incrementally
      uint32_t round = 0;    // (no integer division / modulo by the runtime S per unit)
      for (int item = bid; item < items; item += nbid) {
        int u0, u1;
        unit_range(item, u0, u1);
        const int cb = ks_n == 1 ? item : item / ks_n;
        for (int u = u0; u < u1; ++u, ++li) {
          const bool aux = u >= g.units_main;
          const int b0 = (aux ? u - g.units_main : u) * GV_BPU;
          const int nb = min(GV_BPU, (aux ? g.nbox_aux : g.nbox) - b0);
          if (li >= S) mbar_wait(empty + st_i, (round - 1u) & 1u);
          uint8_t* st = ring + st_i * GV_BPU * GV_BOX_BYTES;
          mbar_arrive_expect_tx(full + st_i, (uint32_t)(nb * GV_BOX_BYTES));
          for (int b = 0; b < nb; ++b)
            tma_load_2d(st + b * GV_BOX_BYTES, aux ? &maps.x : &maps.w, full + st_i,
                        aux ? (b0 + b) * 64 : (b0 + b) * 128, cb * 16);
          if (++st_i == S) st_i = 0, ++round;
        }
      }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ---- consumers: wait for the preceding kernels, stage the activation rows
  // (rows >= M and bytes past the row: zero) in the permuted piece order:
  // box b, chunk c = 2 tig + half -> slot 4 half + tig
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int M = p.m_count ? *p.m_count : p.M;  // MAC rows: device-side count
  constexpr int CT = GV_WARPS * 32;
  {
    constexpr int PB = PACKED ? 32 : 16;  // activation bytes per weight chunk
    const int pieces = g.nbox * 8;
    for (int i = threadIdx.x; i < g.srows * pieces; i += CT) {
      const int t = i / pieces, pc = i - t * pieces;
      const int b = pc >> 3, c = pc & 7;
      const int64_t src = (int64_t)(b * 8 + c) * PB;
      uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
      if (t < M && src < g.a_bytes) {
        const uint4* s4 = reinterpret_cast<const uint4*>(g.a + (int64_t)t * g.lda + src);
        v0 = __ldg(s4);
        if (PB == 32) v1 = src + 16 < g.a_bytes ? __ldg(s4 + 1) : v1;
      }
      uint4* d = reinterpret_cast<uint4*>(sact + t * g.act_stride + b * 8 * PB + (4 * (c & 1) + (c >> 1)) * PB);
      d[0] = v0;
      if (PB == 32) d[1] = v1;
    }
    if (!LR1) {
      const int xp = g.nbox_aux * 8;  // 16-byte pieces
      for (int i = threadIdx.x; i < g.srows * xp; i += CT) {
        const int t = i / max(xp, 1), pc = i - t * xp;
        const int b = pc >> 3, c = pc & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (t < M) v = __ldg(reinterpret_cast<const uint4*>(g.xa + (int64_t)t * p.k_aux) + b * 8 + c);
        *reinterpret_cast<uint4*>(saux + t * g.aux_stride + b * 128 + (4 * (c & 1) + (c >> 1)) * 16) = v;
      }
    }
  }
  // per-thread token constants: tokens 8 j + 2 tig + {0, 1} (accumulator columns)
  float t_s[NT][2], t_rho[NT][2];
  int t_zp[NT][2], t_orow[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int t = 8 * j + 2 * tig + e;
      t_s[j][e] = 0.f, t_rho[j][e] = 0.f, t_zp[j][e] = 0, t_orow[j][e] = t;
      if (t < M) {
        t_s[j][e] = p.row_s ? p.row_s[t] : 0.f;
        t_zp[j][e] = p.row_zp ? p.row_zp[t] : 0;
        if (!LR1 && p.k_aux > 0 && p.row_rho) t_rho[j][e] = p.row_rho[t];
        if (LR1 && p.row_map) t_orow[j][e] = p.row_map[t];
      }
    }
  gv_bar_consumers();  // staged rows visible

  // this thread's B-operand token rows 8 j + gq (clamped to the staged rows)
  const uint8_t* arow[NT];
  const uint8_t* xrow[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int r = min(8 * j + gq, g.srows - 1);
    arow[j] = sact + r * g.act_stride;
    xrow[j] = saux + r * g.aux_stride;
  }
  int li = 0, st_i = 0;
  uint32_t round = 0;
  for (int item = bid; item < items; item += nbid) {
    const int cb = ks_n == 1 ? item : item / ks_n;
    int u0, u1;
    unit_range(item, u0, u1);
    // the block's column constants (channels cb*16 + gq and + 8), loaded now
    // so their latency hides under the MMA units (warp 0 runs the epilogue)
    float c_s[2] = {0.f, 0.f}, c_k[2] = {0.f, 0.f};
    int c_cs[2] = {0, 0};
    if (warp == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = cb * 16 + gq + 8 * h;
        if (col < p.N) {
          c_s[h] = p.col_s[col];
          if (p.row_zp) c_cs[h] = p.col_cs[col];
          if (!LR1 && p.k_aux > 0 && p.mode != G2_RAW) c_k[h] = p.col_kappa[col];
        }
      }
    }
    int acc[NT][4];
    float ax[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = 0, ax[j][e] = 0.f;
    for (int u = u0; u < u1; ++u, ++li) {
      const bool aux = u >= g.units_main;
      const int b0 = (aux ? u - g.units_main : u) * GV_BPU;
      const int nb = min(GV_BPU, (aux ? g.nbox_aux : g.nbox) - b0);
      const uint8_t* st = ring + st_i * GV_BPU * GV_BOX_BYTES;
      mbar_wait(full + st_i, round & 1u);
      for (int it = warp; it < 2 * nb; it += GV_WARPS) {
        const int b = it >> 1, half = it & 1;
        const int c = 2 * tig + half;  // chunk of the 128-byte box row
        const uint8_t* bx = st + b * GV_BOX_BYTES;
        const uint4 wl = *reinterpret_cast<const uint4*>(bx + gq * 128 + ((c ^ gq) << 4));
        const uint4 wh = *reinterpret_cast<const uint4*>(bx + (gq + 8) * 128 + ((c ^ gq) << 4));
        const int slot = 4 * half + tig;
        if (!aux && PACKED) {
          const uint32_t lo[4] = {wl.x, wl.y, wl.z, wl.w}, hi[4] = {wh.x, wh.y, wh.z, wh.w};
          uint32_t fa[4][4];  // unpacked A fragments, shared by the n-tiles
#pragma unroll
          for (int i = 0; i < 4; ++i)
            fa[i][0] = gv_sext4(lo[i]), fa[i][1] = gv_sext4(hi[i]), fa[i][2] = gv_sext4(lo[i] >> 4),
            fa[i][3] = gv_sext4(hi[i] >> 4);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint4* ap =
                reinterpret_cast<const uint4*>(arow[j] + (b0 + b) * 256 + slot * 32);
            const uint4 x0 = ap[0], x1 = ap[1];
            const uint32_t av[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              gv_mma_i8<ASIGNED>(acc[j], fa[i][0], fa[i][1], fa[i][2], fa[i][3], av[2 * i], av[2 * i + 1]);
          }
        } else if (!aux) {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint4 x0 =
                *reinterpret_cast<const uint4*>(arow[j] + (b0 + b) * 128 + slot * 16);
            gv_mma_i8<ASIGNED>(acc[j], wl.x, wh.x, wl.y, wh.y, x0.x, x0.y);
            gv_mma_i8<ASIGNED>(acc[j], wl.z, wh.z, wl.w, wh.w, x0.z, x0.w);
          }
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint4 x0 =
                *reinterpret_cast<const uint4*>(xrow[j] + (b0 + b) * 128 + slot * 16);
            gv_mma_f16(ax[j], wl.x, wh.x, wl.y, wh.y, x0.x, x0.y);
            gv_mma_f16(ax[j], wl.z, wh.z, wl.w, wh.w, x0.z, x0.w);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st_i);  // this warp is done with the stage
      if (++st_i == S) st_i = 0, ++round;
    }
    // ---- per n-tile: the 8 warps' partials, summed in warp order by warp 0
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j) gv_bar_consumers();  // s_acc reused
#pragma unroll
      for (int e = 0; e < 4; ++e) s_acc[warp][lane][e] = acc[j][e], s_aux[warp][lane][e] = ax[j][e];
      gv_bar_consumers();
      if (warp != 0) continue;
      int sa[4];
      float sx[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sa[e] = 0, sx[e] = 0.f;
        for (int w = 0; w < GV_WARPS; ++w) sa[e] += s_acc[w][lane][e], sx[e] += s_aux[w][lane][e];
      }
      bool last = true;
      if (ks_n > 1) {  // K split over CTAs: integer partials meet in global memory (exact)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = cb * 16 + gq + 8 * (e >> 1), t = 8 * j + 2 * tig + (e & 1);
          if (col < p.N && t < M) atomicAdd(g.red + t * p.N + col, sa[e]);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) s_last = atomicAdd(g.cnt + cb * NT + j, 1u) == (unsigned)(ks_n - 1);
        __syncwarp();
        last = s_last;
        if (last) {
          __threadfence();
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int col = cb * 16 + gq + 8 * (e >> 1), t = 8 * j + 2 * tig + (e & 1);
            if (col < p.N && t < M) sa[e] = atomicAdd(g.red + t * p.N + col, 0);
          }
        }
      }
      // ---- epilogue: (channel cb*16 + gq + 8 (e >> 1), token 8 j + 2 tig + (e & 1))
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = cb * 16 + gq + 8 * (e >> 1), tk = e & 1, t = 8 * j + 2 * tig + tk;
        if (!last || col >= p.N || t >= M) continue;
        const int acc_c = sa[e] - (p.row_zp ? t_zp[j][tk] * c_cs[e >> 1] : 0);
        if (LR1) {
          __half* o = reinterpret_cast<__half*>(p.out);
          const float v = acc_c == 0 ? 0.f : t_s[j][tk] * c_s[e >> 1] * (float)acc_c;
          if (!(fabsf(v) <= 65504.f) && p.err) atomicOr(p.err, 8 /*ERR_LR_RANGE*/);
          const __half hv = __float2half_rn(v);
          o[(int64_t)t_orow[j][tk] * p.ldo + p.col_off + col] = hv;
          if (p.lo_off)
            o[(int64_t)t_orow[j][tk] * p.ldo + p.col_off + p.lo_off + col] = __float2half_rn(v - __half2float(hv));
        } else if (p.mode == G2_RAW) {
          const int64_t idx = (int64_t)t * p.ldo + col;
          reinterpret_cast<int*>(p.out)[idx] = sa[e];
          if (p.k_aux && p.raw_aux) p.raw_aux[idx] = sx[e];
        } else {
          float v = t_s[j][tk] * c_s[e >> 1] * (float)acc_c;
          if (p.k_aux > 0) v = fmaf(t_rho[j][tk] * c_k[e >> 1], sx[e], v);
          g2_store1(p, (int64_t)t * p.ldo + col, v);
        }
      }
    }
    gv_bar_consumers();  // s_acc reused by the next item
  }
}

template <bool PACKED, bool ASIGNED, bool LR1, int NT>
__global__ void __launch_bounds__(GV_THREADS) gv_kernel(const __grid_constant__ GvMaps maps,
                                                        const __grid_constant__ G2Params p,
                                                        const __grid_constant__ GvArgs g, int blocks) {
  gv_body<PACKED, ASIGNED, LR1, NT>(maps, p, g, blocks, blockIdx.x, gridDim.x);
}

// Both low-rank first stages (CWS over the main codes, MAC over the compact
// text-row residual codes) in one launch: CTAs [0, split) run the first,
// the rest the second (one launch fewer on the decode chain).
template <bool AS1, bool AS2, int NT>
__global__ void __launch_bounds__(GV_THREADS) gv_lr1_pair_kernel(
    const __grid_constant__ GvMaps maps1, const __grid_constant__ G2Params p1, const __grid_constant__ GvArgs g1,
    int blocks1, const __grid_constant__ GvMaps maps2, const __grid_constant__ G2Params p2,
    const __grid_constant__ GvArgs g2, int blocks2, int split) {
  if ((int)blockIdx.x < split)
    gv_body<false, AS1, true, NT>(maps1, p1, g1, blocks1, blockIdx.x, split);
  else
    gv_body<false, AS2, true, NT>(maps2, p2, g2, blocks2, blockIdx.x - split, gridDim.x - split);
}

}  // namespace splitq
