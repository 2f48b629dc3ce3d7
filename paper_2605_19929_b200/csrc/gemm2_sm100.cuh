// Split-linear GEMM v2 for sm_100a: CTA-pair (cta_group::2) tcgen05 MMA with
// M = 256 rows per tile, double-buffered TMEM accumulators, and every
// auxiliary branch folded into one fp32 accumulator.
//
// Reference semantics (numpy float64, pkg/src/modquant/layer.py):
//   y = x_hat @ Q(R) + (x_hat @ Q(U_s)) @ Q(V_s)            :141-151
//     + [text rows] (Q(e) @ Q(U_c)) @ Q(V_c)                 :157-166
//     + Q(X_t d_t) @ Q(W_t/d_t) + Q(X_v d_v) @ Q(W_v/d_v)    :106-115, 132-133, 171
// Per tile (each CTA of the pair owns 128 of the 256 rows):
//   R_main[b] (int32, TMEM) = sum_k a_code * w_code           tcgen05 kind::i8, exact
//   R_aux[b]  (fp32,  TMEM) = A_aux @ B_aux                    tcgen05 kind::f16
//     A_aux (fp16, per token) = [text hi | lo | hi][vision hi | lo | hi][CWS t1][MAC t1]
//     B_aux (fp16, per column) = [text hi | hi | lo][vision hi | hi | lo][CWS v][MAC v]
//   (the hi/lo splits make the outlier products exact to ~2^-22)
//   y = S_a[i] S_w[j] (R_main - zp_i cs_j) + rho_i kappa_j R_aux
// Warp roles per CTA (320 threads): 0 TMA producer, 1 TMEM alloc + MMA issue
// (leader CTA only), 2..5 epilogue, 6..9 weight unpack. Accumulators are
// double-buffered so the epilogue of tile t overlaps the MMAs of tile t+1.
//
// Swap-AB (p.swap, decode-sized token counts): the 256-row MMA tile runs over
// output channels (A = weights [N x K], B = token codes [M x K], both K-major
// as stored) and the tile's N over tokens, so a 16..64-token call does not pad
// the MMA to 256 token rows. TMEM lane = output channel, column = token; the
// epilogue swaps the row / column roles of the scales.
//
// Packed weights (p.packed_b): the main B operand lives in HBM as 4-bit
// two's-complement codes (W4, and W3 in the same container), two per byte,
// interleaved so that byte i of each 32-bit word holds codes 8g+i (low nibble)
// and 8g+4+i (high nibble). Each CTA's producer TMA-loads the packed half-box
// [bn/2 rows x 64 B] into a staging buffer (local mbarrier bfull); the unpack
// warps sign-extend it to s8 and store it in the 128-byte-swizzled K-major
// layout the UMMA descriptor expects (16-B chunk c of row r at c ^ (r & 7)),
// fence the generic-proxy writes for the async proxy, and arrive on the
// leader CTA's full barrier, which therefore counts the A bytes (TMA) plus one
// arrival per CTA's unpack group.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100_ptx.cuh"

namespace splitq {

constexpr int G2_BM = 256;                 // rows per CTA pair
constexpr int G2_BN = 160;                 // max tile N with the aux accumulator (3 bn <= 512 TMEM cols)
constexpr int G2_BN_MAX = 256;             // max tile N without it
constexpr int G2_A_BYTES = 128 * 128;      // per CTA: 128 rows x 128 B
constexpr int G2_MAX_STAGES = 12;
constexpr int G2_RING_BYTES = 192 * 1024;  // SMEM ring: stages of A (16 KB) + B (bn * 64 B)
constexpr int G2_THREADS = 192;         // producer, MMA, 4 epilogue warps
constexpr int G2_THREADS_PACKED = 320;  // + 4 weight-unpack warps
constexpr int G2_CONV_WARP0 = 6;  // warps 6..9 unpack packed weights
constexpr int G2_TMEM_COLS = 512;
// kind::mxf4 main path: TMEM columns [G2_SF_COL, 512) hold the block scale
// factors, every byte UE8M0 1.0 (0x7F), so A2 / W3 codes stored as E2M1
// multiply exactly; needs 3 bn <= G2_SF_COL (bn <= 160)
constexpr int G2_SF_COL = 496;
constexpr int G2_COLC_BYTES = 2048;        // per-tile column constants of the fast epilogue
constexpr int G2_SMEM_BYTES = G2_RING_BYTES + 1024 + 512 + G2_COLC_BYTES;

// stage geometry for a tile width: per CTA an A box (128 x 128 B), a B box
// (bn/2 x 128 B) and, with packed weights, the packed staging box (bn/2 x 64 B)
__host__ __device__ inline int g2_stage_bytes(int bn, int packed, int swap = 0) {
  return G2_A_BYTES + bn * 64 + (packed ? (swap ? 128 * 64 : bn * 32) : 0);
}
__host__ __device__ inline int g2_stages(int bn, int packed, int swap = 0) {
  const int s = G2_RING_BYTES / g2_stage_bytes(bn, packed, swap);
  return s < G2_MAX_STAGES ? s : G2_MAX_STAGES;
}

enum G2Mode : int { G2_SPLIT = 0, G2_RAW = 1, G2_LR1 = 2, G2_ACC = 3 };
// G2_ACC (split-K): work item = (tile, K range ks); the epilogue stores the
// int32 main / fp32 aux partial accumulators of range ks into its own slice
// acc_i32 / acc_f32 + ks * slice [rows x ld_acc] (plain coalesced stores, no
// atomics; ranges that did not touch an accumulator store zeros), and
// g2_finalize_kernel sums the slices in range order and applies the SPLIT /
// LR1 / RAW epilogue (same arithmetic, g2_epi_*): deterministic.
enum G2Out : int { G2_F32 = 0, G2_F16 = 1, G2_BF16 = 2 };

struct G2Maps {
  CUtensorMap a, b;      // main int8 operands: A [rows x K], B [N x K] (b: packed [N x K/2] when packed_b)
  CUtensorMap xa, xb;    // aux fp16 operands: A_aux [rows x K_aux], B_aux [N x K_aux]
};

struct G2Params {
  int M;              // rows (overridden by *m_count)
  const int* m_count;
  int N;              // columns
  int bn;             // tile N: multiple of 32, <= G2_BN (aux) or G2_BN_MAX
  int k_main;         // int8 K
  int k_aux;          // fp16 K (multiple of 64; 0 = no aux branch)
  uint32_t idesc_main, idesc_aux;
  int mode, out_dtype;
  int packed_b;         // weights as packed 4-bit codes (see header)
  int swap;             // swap-AB: tile rows = output channels, tile cols = tokens
  const float* row_s;   // S_a (SPLIT) or S/rho (LR1)
  const int* row_zp;    // zero points when A codes are u8
  const float* row_rho;
  const float* col_s;   // S_w (SPLIT) or S_u/sigma (LR1)
  const int* col_cs;    // column code sums (u8 zero-point correction)
  const float* col_kappa;
  void* out;
  int64_t ldo;
  const int* row_map;   // LR1: destination row
  int col_off;          // LR1: destination column
  int lo_off;           // LR1: > 0 -> also write the fp16 residual (v - fp16(v)) at col_off + lo_off
  float* raw_aux;       // RAW: fp32 aux plane
  int* err;
  int k_split;          // >= 1: K ranges per tile (G2_ACC when > 1)
  unsigned long long* trace;  // G2_TRACE builds: per-CTA phase timestamps (ns)
  int* acc_i32;         // G2_ACC scratch: k_split slices of [rows x ld_acc]
  float* acc_f32;
  int64_t ld_acc;
  int64_t acc_slice;    // elements per slice
  int tile_gm;          // > 0: tiles walk groups of tile_gm m-tiles, m fastest (L2 reuse of B)
  int mxf4;             // main operands are packed E2M1 codes (kind::mxf4, unit block scales):
                        // k_main counts bytes, the main accumulator is fp32 (exact integers)
  int epi_fast;         // SPLIT epilogue without zero points and with |acc| < 2^22 (or mxf4): column
                        // constants from SMEM, packed fp32 math, exact magic-number int -> float
};

__device__ __forceinline__ uint64_t g2_pk(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 g2_upk(uint64_t a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 g2_mul2(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(g2_pk(a)), "l"(g2_pk(b)));
  return g2_upk(r);
}
__device__ __forceinline__ float2 g2_add2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(g2_pk(a)), "l"(g2_pk(b)));
  return g2_upk(r);
}
__device__ __forceinline__ float2 g2_fma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(g2_pk(a)), "l"(g2_pk(b)), "l"(g2_pk(c)));
  return g2_upk(r);
}

// the main accumulator word of TMEM as the exact integer it holds
__device__ __forceinline__ int g2_acc(const G2Params& p, uint32_t w) {
  return p.mxf4 ? (int)__uint_as_float(w) : (int)w;
}

// tile index -> (m-tile, n-tile). Default: row-major (n fastest), so the
// concurrent CTA pairs share one A row block and stream B. With tile_gm > 0
// (wide N: B larger than an L2 partition), m runs fastest inside groups of
// tile_gm m-tiles: the group's A slab stays in L2 and B is streamed once per
// group instead of being re-fetched for every m-tile.
__device__ __forceinline__ void g2_tile(const G2Params& p, int tile, int m_tiles, int n_tiles, int& mt, int& nt) {
  if (p.tile_gm <= 0) {
    mt = tile / n_tiles;
    nt = tile - mt * n_tiles;
    return;
  }
  const int gsz = p.tile_gm * n_tiles;
  const int grp = tile / gsz, r = tile - grp * gsz;
  const int gm = min(p.tile_gm, m_tiles - grp * p.tile_gm);
  nt = r / gm;
  mt = grp * p.tile_gm + (r - nt * gm);
}

// ---------------------------------------------------------------- epilogue math
// One output of the SPLIT epilogue: y = S_a S_w (acc - zp cs) + rho kappa aux
__device__ __forceinline__ float g2_epi_split(const G2Params& p, int col, int acc_raw, int zp,
                                              float s_row, float rho, bool has_aux, float aux) {
  const int acc = acc_raw - (p.row_zp ? zp * p.col_cs[col] : 0);
  float v = s_row * p.col_s[col] * (float)acc;
  if (has_aux) v = fmaf(rho * p.col_kappa[col], aux, v);
  return v;
}
// One output of the LR1 epilogue: fp16 hi (+ lo) of (S/rho)(S_u/sigma) acc
__device__ __forceinline__ void g2_epi_lr1(const G2Params& p, int orow, int col, int acc_raw,
                                           int zp, float s_row) {
  __half* o = reinterpret_cast<__half*>(p.out);
  const int acc = acc_raw - (p.row_zp ? zp * p.col_cs[col] : 0);
  const float v = acc == 0 ? 0.f : s_row * p.col_s[col] * (float)acc;
  if (!(fabsf(v) <= 65504.f) && p.err) atomicOr(p.err, 8 /*ERR_LR_RANGE*/);
  const __half hv = __float2half_rn(v);
  o[(int64_t)orow * p.ldo + p.col_off + col] = hv;
  if (p.lo_off) o[(int64_t)orow * p.ldo + p.col_off + p.lo_off + col] = __float2half_rn(v - __half2float(hv));
}
__device__ __forceinline__ void g2_store1(const G2Params& p, int64_t idx, float v) {
  if (p.out_dtype == G2_F32) reinterpret_cast<float*>(p.out)[idx] = v;
  else if (p.out_dtype == G2_F16) reinterpret_cast<__half*>(p.out)[idx] = __float2half_rn(v);
  else reinterpret_cast<__nv_bfloat16*>(p.out)[idx] = __float2bfloat16_rn(v);
}

// ---------------------------------------------------------------- pair helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
// arrive on a (possibly remote) cluster barrier with the default .release.cta
// semantics: no GPU-scope membar (the unpack warps' generic-proxy writes are
// ordered for the tensor core by fence.proxy.async before this arrive)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA 2-D load whose completion is counted on the leader CTA's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map,
                                                 uint64_t* bar, int32_t c0, int32_t c1) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;  // peer bit cleared -> CTA 0 of the pair
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D (+)= A * B on packed E2M1 codes with block scale factors from TMEM
__device__ __forceinline__ void mma_mxf4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_f16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// commit: arrive on the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ int g2_chunks(int k_bytes) { return (k_bytes + 127) / 128; }

// one lane of a converged warp (the same lane every call)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ unsigned long long g2_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef G2_TRACE
#define G2_STAMP(slot) do { if (p.trace) p.trace[blockIdx.x * 8 + (slot)] = g2_now(); } while (0)
#else
#define G2_STAMP(slot) do { } while (0)
#endif

template <bool PACKED>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PACKED ? G2_THREADS_PACKED : G2_THREADS, 1)
    splitq_gemm2_kernel(const __grid_constant__ G2Maps maps, const G2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int STAGES = g2_stages(p.bn, PACKED, p.swap);
  const int STAGE_BYTES = g2_stage_bytes(p.bn, PACKED, p.swap);
  const int B_BYTES = p.bn * 64;  // per CTA: bn/2 rows x 128 B
  // the slot the weights land in (A with swap-AB, else B), its rows per CTA,
  // and where the packed staging box sits in the stage
  const int W_OFF = p.swap ? 0 : G2_A_BYTES;
  const int W_ROWS = p.swap ? 128 : p.bn / 2;
  const int STG_OFF = G2_A_BYTES + B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G2_RING_BYTES);
  uint64_t* empty = full + G2_MAX_STAGES;
  uint64_t* bfull = empty + G2_MAX_STAGES;  // packed staging landed (local)
  uint64_t* tfull = bfull + G2_MAX_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* aempty = tempty + 2;         // [1] aux accumulator drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);
  // fast epilogue: the tile's column constants, float4 per column pair
  // {sw_2i, sw_2i+1, kappa_2i, kappa_2i+1}
  float* colc = reinterpret_cast<float*>(smem + G2_RING_BYTES + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // Programmatic dependent launch: everything up to the first read of a
  // preceding kernel's output (barrier / TMEM set-up, the first ring slots'
  // weight loads) overlaps that kernel's tail; the threads that read its
  // outputs (producer for the activations, epilogue for the row constants)
  // wait first. A device-side row count is such an output: wait up front.
  if (p.m_count) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int M = p.m_count ? *p.m_count : p.M;
  // tile grid: 256-row MMA tiles over tokens (or over output channels, swap)
  const int m_tiles = ((p.swap ? p.N : M) + G2_BM - 1) / G2_BM;
  const int n_tiles = ((p.swap ? M : p.N) + p.bn - 1) / p.bn;
  const int num_tiles = m_tiles * n_tiles;
  const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
  // K loop per tile: the n_main int8 chunks first, then the n_aux fp16 chunks.
  // TMEM: main accumulators double-buffered at columns [0, bn) and [bn, 2bn),
  // the aux accumulator single-buffered at [2bn, 3bn): it is written only at
  // the end of a tile's K loop, so the epilogue of tile t drains it while tile
  // t+1's main chunks run (aempty), and bn can be 160 with the aux branch.
  const int n_aux = p.k_aux / 64, n_main = g2_chunks(p.k_main);
  const int stages_per_tile = n_aux + n_main;
  const int ksplit = p.k_split > 1 ? p.k_split : 1;
  const int num_items = num_tiles * ksplit;
  // work item -> (tile, stage range [s0, s1))
  auto item_of = [&](int item, int& tile, int& s0, int& s1) {
    tile = item / ksplit;
    const int ks = item - tile * ksplit;
    s0 = ks * stages_per_tile / ksplit;
    s1 = (ks + 1) * stages_per_tile / ksplit;
  };

  if (threadIdx.x == 0) G2_STAMP(0);  // kernel start
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], PACKED ? 3 : 1);  // producer (A tx) [+ one unpack arrival per CTA]
      mbar_init(&empty[s], 1);
      mbar_init(&bfull[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    mbar_init(aempty, 8);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, G2_TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (p.mxf4) {  // unit block scale factors for the E2M1 main MMAs, in both CTAs' TMEM
    if (warp >= 2 && warp < 6) {
      const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
      tmem_st16_fill(tmem + lanes + G2_SF_COL, 0x7F7F7F7Fu);
      tmem_wait_st();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
  }
  if (threadIdx.x == 0) G2_STAMP(1);  // setup done (barriers, TMEM, cluster sync)

  if (warp == 0) {
    // ================================================== TMA producer (both CTAs)
    if (num_tiles > 0) {
      if (elect_one()) {
        tma_prefetch(&maps.a);
        tma_prefetch(&maps.b);
      }
      const uint32_t tx = 2u * (G2_A_BYTES + (uint32_t)(p.bn / 2) * 128u);
      // packed main stages: only the activation slot comes through the pair TMA
      const uint32_t tx_a = p.swap ? 2u * (uint32_t)(p.bn / 2) * 128u : 2u * G2_A_BYTES;
      const uint32_t tx_bp = (uint32_t)W_ROWS * 64u;       // local packed staging box
      // one ring slot's loads; part: 1 = weights (+ the expect_tx), 2 =
      // activations / aux operand rows, 3 = both. swap-AB: the A slot takes
      // the weight rows (m0), B the token rows (n0).
      auto issue = [&](int v, int m0, int n0, int stage, int part) {
        uint8_t* sa = smem + stage * STAGE_BYTES;
        uint8_t* sb = sa + G2_A_BYTES;
        const bool pk = PACKED && v < n_main;
        if ((part & 1) && leader) mbar_arrive_expect_tx(&full[stage], pk ? tx_a : tx);
        if (v >= n_main) {
          const int va = v - n_main;
          if (part & 1) {
            if (p.swap) tma_load_2d_pair(sa, &maps.xb, &full[stage], va * 64, m0);
            else tma_load_2d_pair(sb, &maps.xb, &full[stage], va * 64, n0);
            if (PACKED) mbar_arrive(&bfull[stage]);
          }
          if (part & 2) {
            if (p.swap) tma_load_2d_pair(sb, &maps.xa, &full[stage], va * 64, n0);
            else tma_load_2d_pair(sa, &maps.xa, &full[stage], va * 64, m0);
          }
        } else if (pk) {
          // packed weights to the local staging box; activations through the pair TMA.
          // bfull advances once per ring slot use (packed: with the staging
          // bytes; otherwise a plain arrival) so its phase stays in lockstep
          // with the ring phase the unpack warps wait on.
          if (part & 1) {
            mbar_arrive_expect_tx(&bfull[stage], tx_bp);
            tma_load_2d(sa + STG_OFF, &maps.b, &bfull[stage], v * 64, p.swap ? m0 : n0);
          }
          if (part & 2) {
            if (p.swap) tma_load_2d_pair(sb, &maps.a, &full[stage], v * 128, n0);
            else tma_load_2d_pair(sa, &maps.a, &full[stage], v * 128, m0);
          }
        } else {
          if (part & 1) {
            if (p.swap) tma_load_2d_pair(sa, &maps.b, &full[stage], v * 128, m0);
            else tma_load_2d_pair(sb, &maps.b, &full[stage], v * 128, n0);
            if (PACKED) mbar_arrive(&bfull[stage]);
          }
          if (part & 2) {
            if (p.swap) tma_load_2d_pair(sb, &maps.a, &full[stage], v * 128, n0);
            else tma_load_2d_pair(sa, &maps.a, &full[stage], v * 128, m0);
          }
        }
      };
      // the first STAGES ring slots are free: their weight loads go out before
      // the wait for the preceding kernels, the activation loads after it
      int pre = 0;
      for (int item = pair; item < num_items && pre < STAGES; item += num_pairs) {
        int tile, s0, s1;
        item_of(item, tile, s0, s1);
        int mt, nt;
        g2_tile(p, tile, m_tiles, n_tiles, mt, nt);
        const int m0 = mt * G2_BM + (int)rank * 128;
        const int n0 = nt * p.bn + (int)rank * (p.bn / 2);
        for (int v = s0; v < s1 && pre < STAGES; ++v, ++pre)
          if (elect_one()) issue(v, m0, n0, pre, 1);
      }
      __syncwarp();
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int stage = 0, slot = 0;
      uint32_t phase = 0;
      for (int item = pair; item < num_items; item += num_pairs) {
        int tile, s0, s1;
        item_of(item, tile, s0, s1);
        int mt, nt;
        g2_tile(p, tile, m_tiles, n_tiles, mt, nt);
        const int m0 = mt * G2_BM + (int)rank * 128;
        const int n0 = nt * p.bn + (int)rank * (p.bn / 2);
        for (int v = s0; v < s1; ++v, ++slot) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) issue(v, m0, n0, stage, slot < pre ? 2 : 3);
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================== MMA issuer (leader CTA)
    // The whole warp walks the pipeline (values stay warp-uniform, so the
    // descriptors live in uniform registers); one elected lane issues.
    if (leader && num_tiles > 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, aux_uses = 0;
      const uint32_t smem0 = smem_u32(smem);
      for (int item = pair; item < num_items; item += num_pairs, ++it) {
        int tile, s0, s1;
        item_of(item, tile, s0, s1);
        const int first_aux = s0 > n_main ? s0 : n_main;  // first aux stage of the range
        const int b = it & 1;
        const uint32_t tph = (it >> 1) & 1;
        mbar_wait(&tempty[b], tph ^ 1);
        tc_fence_after();
        const uint32_t d_main = tmem + b * p.bn;
        const uint32_t d_aux = tmem + 2 * p.bn;
        for (int v = s0; v < s1; ++v) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0 && v == s0 && it == 0) G2_STAMP(2);  // first stage's data ready
          const uint32_t a_addr = smem0 + stage * STAGE_BYTES;
          const uint64_t ad = sw128_kmajor_desc(a_addr);
          const uint64_t bd = sw128_kmajor_desc(a_addr + G2_A_BYTES);
          if (v >= n_main) {
            if (v == first_aux) {  // the previous tile's epilogue has drained the aux accumulator
              if (aux_uses > 0) mbar_wait(aempty, (uint32_t)((aux_uses - 1) & 1));
              ++aux_uses;
              tc_fence_after();
            }
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < 4; ++k)  // K = 16 fp16 (32 B) per MMA
                mma_f16_pair(d_aux, ad + 2 * k, bd + 2 * k, p.idesc_aux, (v != first_aux) || k != 0);
              tc_commit_pair(&empty[stage]);
            }
          } else {
            const int c = v;
            const int nk = (p.k_main - c * 128 + 31) / 32;  // K = 32 int8 per MMA
            if (elect_one()) {
              if (p.mxf4) {  // 32 bytes = 64 E2M1 codes per MMA
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  if (k < nk)
                    mma_mxf4_pair(d_main, ad + 2 * k, bd + 2 * k, p.idesc_main, tmem + G2_SF_COL,
                                  tmem + G2_SF_COL + 8, (v != s0) || k != 0);
              } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  if (k < nk) mma_i8_pair(d_main, ad + 2 * k, bd + 2 * k, p.idesc_main, (v != s0) || k != 0);
              }
              tc_commit_pair(&empty[stage]);
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) tc_commit_pair(&tfull[b]);
        __syncwarp();
        if (lane == 0) G2_STAMP(3);  // last MMA issued
      }
    }
  } else if (PACKED && warp >= G2_CONV_WARP0) {
    // ================================================== weight unpack (warps 6..9, both CTAs)
    // All 128 unpack threads share each ring slot (W_ROWS x 8 16-byte chunks),
    // then one thread arrives on the leader's full barrier for this CTA.
    const int ct = threadIdx.x - 32 * G2_CONV_WARP0;  // 0..127
    const uint32_t full_leader = mapa_shared(&full[0], 0);
    const int outs = W_ROWS * 8;  // 16-byte output chunks per slot
    if (num_tiles > 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = pair; item < num_items; item += num_pairs) {
        int tile, s0, s1;
        item_of(item, tile, s0, s1);
        for (int v = s0; v < s1; ++v) {
          mbar_wait(&empty[stage], phase ^ 1);  // previous use of the slot drained
          if (v < n_main) {
            mbar_wait(&bfull[stage], phase);
            uint8_t* sb = smem + stage * STAGE_BYTES + W_OFF;
            const uint8_t* sp = smem + stage * STAGE_BYTES + STG_OFF;
#pragma unroll 4
            for (int o = ct; o < outs; o += 128) {
              const int r = o >> 3, c = o & 7;
              const uint2 w = *reinterpret_cast<const uint2*>(sp + r * 64 + c * 8);
              const uint32_t w0h = w.x >> 4, w1h = w.y >> 4;
              uint4 out;  // sign-extend 4-bit codes: (v & 0x0F..) | ((v & 0x08..) * 0x1E)
              out.x = (w.x & 0x0F0F0F0Fu) | ((w.x & 0x08080808u) * 0x1Eu);
              out.y = (w0h & 0x0F0F0F0Fu) | ((w0h & 0x08080808u) * 0x1Eu);
              out.z = (w.y & 0x0F0F0F0Fu) | ((w.y & 0x08080808u) * 0x1Eu);
              out.w = (w1h & 0x0F0F0F0Fu) | ((w1h & 0x08080808u) * 0x1Eu);
              *reinterpret_cast<uint4*>(sb + r * 128 + ((c ^ (r & 7)) << 4)) = out;
            }
            fence_proxy_async();  // generic-proxy SMEM writes -> async proxy (UMMA)
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (ct == 0) mbar_arrive_remote(full_leader + (uint32_t)(stage * sizeof(uint64_t)));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ================================================== epilogue (warps 2..5, both CTAs)
    asm volatile("griddepcontrol.wait;" ::: "memory");  // row constants come from K1
    const int lq = warp & 3;                 // TMEM lane quarter
    const int r_local = lq * 32 + lane;
    const uint32_t tempty_leader = mapa_shared(&tempty[0], 0);
    const uint32_t aempty_leader = mapa_shared(aempty, 0);
    const bool aux_buf = p.k_aux > 0;  // TMEM layout has the aux half
    int it = 0;
    for (int item = pair; item < num_items; item += num_pairs, ++it) {
      int tile, s0, s1;
      item_of(item, tile, s0, s1);
      const bool has_aux = aux_buf && s1 > (s0 > n_main ? s0 : n_main);  // range touched the aux accumulator
      const bool has_main = s0 < n_main;                                 // ... and the main one
      const int b = it & 1;
      const uint32_t tph = (it >> 1) & 1;
      int mt, nt;
      g2_tile(p, tile, m_tiles, n_tiles, mt, nt);
      const int m0 = mt * G2_BM + (int)rank * 128;
      const int n0 = nt * p.bn;
      if (p.swap) {
        // ---- swap-AB: TMEM lane = output channel j, column = token i
        const int j = m0 + r_local;
        const bool j_ok = j < p.N;
        mbar_wait(&tfull[b], tph);
        tc_fence_after();
        if (warp == 2 && lane == 0 && it == 0) G2_STAMP(6);  // accumulator ready
        const uint32_t lb = tmem + ((uint32_t)(lq * 32) << 16) + b * p.bn;
        const uint32_t lba = tmem + ((uint32_t)(lq * 32) << 16) + 2 * p.bn;  // aux accumulator
        // per-channel constants once; per-token ones loaded by lane jj of the
        // chunk and broadcast with shuffles (no per-element global loads)
        const float sw_j = j_ok && p.col_s ? p.col_s[j] : 0.f;
        const int cs_j = j_ok && p.row_zp && p.col_cs ? p.col_cs[j] : 0;
        const float kap_j = j_ok && has_aux && p.col_kappa ? p.col_kappa[j] : 0.f;
        const bool lr1 = p.mode == G2_LR1;
        __half* lo_out = reinterpret_cast<__half*>(p.out);
        for (int c0 = 0; c0 < p.bn; c0 += 32) {
          uint32_t am[32], af[32];
          tmem_ld32(lb + c0, am);
          if (has_aux) tmem_ld32(lba + c0, af);
          tmem_wait_ld();
          const int il = n0 + c0 + lane;
          const bool il_ok = il < M;
          const float s_l = il_ok && p.row_s ? p.row_s[il] : 0.f;
          const int zp_l = il_ok && p.row_zp ? p.row_zp[il] : 0;
          const float rho_l = il_ok && has_aux && p.row_rho ? p.row_rho[il] : 0.f;
          const int orow_l = il_ok && p.row_map ? p.row_map[il] : il;
          // one compact unrolled loop per mode (a single loop with every mode
          // inside unrolls to ~5.7k instructions and thrashes the i-cache)
          const int nrem = M - (n0 + c0);  // valid tokens in this chunk (may exceed 32)
          if (p.mode == G2_ACC) {
            const int64_t base = (int64_t)(item % ksplit) * p.acc_slice + (int64_t)(n0 + c0) * p.ld_acc + j;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              if (j_ok && jj < nrem) {
                p.acc_i32[base + (int64_t)jj * p.ld_acc] = has_main ? g2_acc(p, am[jj]) : 0;
                if (aux_buf) p.acc_f32[base + (int64_t)jj * p.ld_acc] = has_aux ? __uint_as_float(af[jj]) : 0.f;
              }
            }
          } else if (p.mode == G2_RAW) {
            const int64_t base = (int64_t)(n0 + c0) * p.ldo + j;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              if (j_ok && jj < nrem) {
                reinterpret_cast<int*>(p.out)[base + (int64_t)jj * p.ldo] = g2_acc(p, am[jj]);
                if (has_aux && p.raw_aux) p.raw_aux[base + (int64_t)jj * p.ldo] = __uint_as_float(af[jj]);
              }
            }
          } else if (lr1) {  // g2_epi_lr1 with the constants hoisted
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const float s_i = __shfl_sync(0xffffffffu, s_l, jj);
              const int zp_i = __shfl_sync(0xffffffffu, zp_l, jj);
              const int orow_i = __shfl_sync(0xffffffffu, orow_l, jj);
              if (j_ok && jj < nrem) {
                const int a2 = g2_acc(p, am[jj]) - zp_i * cs_j;
                const float v = a2 == 0 ? 0.f : s_i * sw_j * (float)a2;
                if (!(fabsf(v) <= 65504.f) && p.err) atomicOr(p.err, 8 /*ERR_LR_RANGE*/);
                const __half hv = __float2half_rn(v);
                __half* o = lo_out + (int64_t)orow_i * p.ldo + p.col_off + j;
                o[0] = hv;
                if (p.lo_off) o[p.lo_off] = __float2half_rn(v - __half2float(hv));
              }
            }
          } else {  // g2_epi_split with the constants hoisted
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const float s_i = __shfl_sync(0xffffffffu, s_l, jj);
              const int zp_i = __shfl_sync(0xffffffffu, zp_l, jj);
              const float rho_i = __shfl_sync(0xffffffffu, rho_l, jj);
              if (j_ok && jj < nrem) {
                float v = s_i * sw_j * (float)(g2_acc(p, am[jj]) - zp_i * cs_j);
                if (has_aux) v = fmaf(rho_i * kap_j, __uint_as_float(af[jj]), v);
                g2_store1(p, (int64_t)(n0 + c0 + jj) * p.ldo + j, v);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_cluster(tempty_leader + (uint32_t)(b * sizeof(uint64_t)));
          if (has_aux) mbar_arrive_cluster(aempty_leader);
        }
        continue;
      }
      const int row = m0 + r_local;
      const bool row_ok = row < M;
      // the tile's row and column constants do not depend on the accumulator:
      // loaded before the wait, so their latency hides under the MMAs (a
      // tile's epilogue is on the critical path for one-tile launches: LR1,
      // small calls, every CTA's last tile)
      float s_row = 0.f, rho = 0.f;
      int zp = 0;
      if (row_ok) {
        if (p.row_s) s_row = p.row_s[row];
        if (p.row_zp) zp = p.row_zp[row];
        if (has_aux && p.row_rho) rho = p.row_rho[row];
      }
      const int orow = row_ok && p.row_map ? p.row_map[row] : row;  // LR1 destination row
      const bool fast = p.mode == G2_SPLIT && p.epi_fast;
      if (p.mode == G2_LR1) {  // the tile's column constants: sw [0, bn), cs [256, 256 + bn)
        asm volatile("bar.sync 2, 128;" ::: "memory");  // previous tile's readers are done
        for (int c = r_local; c < p.bn; c += 128) {
          const int col = n0 + c;
          const bool ok = col < p.N;
          colc[c] = ok ? p.col_s[col] : 0.f;
          reinterpret_cast<int*>(colc)[256 + c] = ok && p.row_zp ? p.col_cs[col] : 0;
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
      }
      if (fast) {  // the 4 epilogue warps of this CTA stage the tile's column constants
        asm volatile("bar.sync 2, 128;" ::: "memory");  // previous tile's readers are done
        for (int c = r_local; c < p.bn; c += 128) {
          const int col = n0 + c;
          const bool ok = col < p.N;
          float* q = colc + 4 * (c >> 1) + (c & 1);
          q[0] = ok ? p.col_s[col] : 0.f;
          q[2] = ok && has_aux ? p.col_kappa[col] : 0.f;
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
      }
      mbar_wait(&tfull[b], tph);
      tc_fence_after();
      if (warp == 2 && lane == 0 && it == 0) G2_STAMP(6);  // accumulator ready
      const uint32_t lane_base = tmem + ((uint32_t)(lq * 32) << 16) + b * p.bn;
      const uint32_t lane_aux = tmem + ((uint32_t)(lq * 32) << 16) + 2 * p.bn;
      for (int c0 = 0; c0 < p.bn; c0 += 32) {
        uint32_t am[32], af[32];
        tmem_ld32(lane_base + c0, am);
        if (has_aux) tmem_ld32(lane_aux + c0, af);
        tmem_wait_ld();
        if (warp == 2 && lane == 0 && it == 0 && c0 == 0) G2_STAMP(7);  // first TMEM chunk in registers
        if (p.mode == G2_LR1) {
          // g2_epi_lr1 in the same rounding order, two columns at a time:
          // v = acc == 0 ? 0 : (s_row * sw) * acc, hi = fp16(v), lo = fp16(v - hi);
          // column constants from SMEM (broadcast reads)
          __half* o = reinterpret_cast<__half*>(p.out) + (int64_t)orow * p.ldo + p.col_off;
          const bool vec = ((p.ldo | p.col_off | p.lo_off) & 7) == 0;
          const float2 s2 = make_float2(s_row, s_row);
#pragma unroll
          for (int g = 0; g < 32; g += 8) {
            const int colg = n0 + c0 + g;
            const float4 swa = *reinterpret_cast<const float4*>(colc + c0 + g);
            const float4 swb = *reinterpret_cast<const float4*>(colc + c0 + g + 4);
            const float sw[8] = {swa.x, swa.y, swa.z, swa.w, swb.x, swb.y, swb.z, swb.w};
            int cs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (p.row_zp) {
              const int4 ca = *reinterpret_cast<const int4*>(reinterpret_cast<const int*>(colc) + 256 + c0 + g);
              const int4 cb = *reinterpret_cast<const int4*>(reinterpret_cast<const int*>(colc) + 256 + c0 + g + 4);
              cs[0] = ca.x; cs[1] = ca.y; cs[2] = ca.z; cs[3] = ca.w;
              cs[4] = cb.x; cs[5] = cb.y; cs[6] = cb.z; cs[7] = cb.w;
            }
            __half2 hv[4], lv[4];
            bool bad = false;
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const int a0 = g2_acc(p, am[g + j]) - zp * cs[j];
              const int a1 = g2_acc(p, am[g + j + 1]) - zp * cs[j + 1];
              float2 v = g2_mul2(g2_mul2(s2, make_float2(sw[j], sw[j + 1])),
                                 make_float2((float)a0, (float)a1));
              if (a0 == 0) v.x = 0.f;
              if (a1 == 0) v.y = 0.f;
              bad |= !(fabsf(v.x) <= 65504.f) || !(fabsf(v.y) <= 65504.f);
              const __half2 h = __floats2half2_rn(v.x, v.y);
              const float2 hf = __half22float2(h);
              const float2 r = g2_add2(v, make_float2(-hf.x, -hf.y));
              hv[j >> 1] = h;
              lv[j >> 1] = __floats2half2_rn(r.x, r.y);
            }
            bad = bad && row_ok;
            if (bad) {  // (columns past N are zero: never bad)
              if (p.err) atomicOr(p.err, 8 /*ERR_LR_RANGE*/);
            }
            if (!row_ok) continue;
            if (vec && colg + 8 <= p.N) {  // 8 columns -> one 16-byte store (+ one for lo)
              *reinterpret_cast<uint4*>(o + colg) = *reinterpret_cast<const uint4*>(hv);
              if (p.lo_off) *reinterpret_cast<uint4*>(o + p.lo_off + colg) = *reinterpret_cast<const uint4*>(lv);
            } else {
              const __half* hs = reinterpret_cast<const __half*>(hv);
              const __half* ls = reinterpret_cast<const __half*>(lv);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (colg + j < p.N) {
                  o[colg + j] = hs[j];
                  if (p.lo_off) o[p.lo_off + colg + j] = ls[j];
                }
            }
          }
          continue;
        }
        float y[32];
        if (fast) {  // g2_epi_split in the same rounding order: (s_row * sw) * acc, fma(rho * kappa, aux, .)
          const float4* cc = reinterpret_cast<const float4*>(colc) + (c0 >> 1);
          const float2 s2 = make_float2(s_row, s_row), r2 = make_float2(rho, rho);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float4 k4 = cc[j >> 1];
            float2 a2;
            if (p.mxf4) {
              a2 = make_float2(__uint_as_float(am[j]), __uint_as_float(am[j + 1]));
            } else {  // |acc| < 2^22: 1.5 * 2^23 + acc is exact, and so is the subtraction
              a2 = g2_add2(make_float2(__int_as_float((int)am[j] + 0x4B400000),
                                       __int_as_float((int)am[j + 1] + 0x4B400000)),
                           make_float2(-12582912.f, -12582912.f));
            }
            float2 v = g2_mul2(g2_mul2(s2, make_float2(k4.x, k4.y)), a2);
            if (has_aux)
              v = g2_fma2(g2_mul2(r2, make_float2(k4.z, k4.w)),
                          make_float2(__uint_as_float(af[j]), __uint_as_float(af[j + 1])), v);
            y[j] = v.x;
            y[j + 1] = v.y;
          }
        } else if (p.mode == G2_SPLIT) {  // g2_epi_split, column constants broadcast from one load per lane
          const int cl = min(n0 + c0 + lane, p.N - 1);
          const float sw_l = p.col_s[cl];
          const int cs_l = p.row_zp ? p.col_cs[cl] : 0;
          const float kap_l = has_aux ? p.col_kappa[cl] : 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float sw = __shfl_sync(0xffffffffu, sw_l, j);
            const int cs = __shfl_sync(0xffffffffu, cs_l, j);
            const float kap = __shfl_sync(0xffffffffu, kap_l, j);
            float v = s_row * sw * (float)(g2_acc(p, am[j]) - zp * cs);
            if (has_aux) v = fmaf(rho * kap, __uint_as_float(af[j]), v);
            y[j] = v;
          }
        }
        if (!row_ok) continue;
        if (p.mode == G2_ACC) {
          const int64_t so = (int64_t)(item % ksplit) * p.acc_slice;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + c0 + j;
            if (col < p.N) {
              const int64_t idx = so + (int64_t)row * p.ld_acc + col;
              p.acc_i32[idx] = has_main ? g2_acc(p, am[j]) : 0;
              if (aux_buf) p.acc_f32[idx] = has_aux ? __uint_as_float(af[j]) : 0.f;
            }
          }
        } else if (p.mode == G2_RAW) {
          int* o = reinterpret_cast<int*>(p.out);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + c0 + j;
            if (col < p.N) {
              const int64_t idx = (int64_t)row * p.ldo + col;
              o[idx] = g2_acc(p, am[j]);
              if (has_aux && p.raw_aux) p.raw_aux[idx] = __uint_as_float(af[j]);
            }
          }
        } else {
          const int64_t base = (int64_t)row * p.ldo + n0 + c0;
          const bool full_chunk = (n0 + c0 + 32 <= p.N) && ((p.ldo & 7) == 0);
          if (p.out_dtype == G2_F32) {
            float* o = reinterpret_cast<float*>(p.out) + base;
            if (full_chunk) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(o + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
            } else {
              for (int j = 0; j < 32; ++j)
                if (n0 + c0 + j < p.N) o[j] = y[j];
            }
          } else if (p.out_dtype == G2_F16) {
            __half* o = reinterpret_cast<__half*>(p.out) + base;
            if (full_chunk) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                __half2 h[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) h[q] = __floats2half2_rn(y[j + 2 * q], y[j + 2 * q + 1]);
                *reinterpret_cast<uint4*>(o + j) = *reinterpret_cast<uint4*>(h);
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
                __nv_bfloat162 h[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  h[q] = __floats2bfloat162_rn(y[j + 2 * q], y[j + 2 * q + 1]);
                *reinterpret_cast<uint4*>(o + j) = *reinterpret_cast<uint4*>(h);
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
      if (lane == 0) {
        mbar_arrive_cluster(tempty_leader + (uint32_t)(b * sizeof(uint64_t)));
        if (has_aux) mbar_arrive_cluster(aempty_leader);
      }
    }
  }

  if (warp == 2 && lane == 0) G2_STAMP(4);  // epilogue done (this CTA)
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, G2_TMEM_COLS);
  }
  if (threadIdx.x == 0) G2_STAMP(5);  // kernel end
}

// Finalize of a split-K (G2_ACC) launch: one thread per output element;
// `mode` is the epilogue the single-pass kernel would have run.
__global__ void g2_finalize_kernel(const G2Params p, int mode, int has_aux) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the split-K slices
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int M = p.m_count ? *p.m_count : p.M;
  const int64_t total = (int64_t)M * p.N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / p.N), col = (int)(e - (int64_t)row * p.N);
    const int64_t ai = (int64_t)row * p.ld_acc + col;
    int acc = 0;
    float aux = 0.f;
    for (int ks = 0; ks < p.k_split; ++ks) {  // fixed order: deterministic sums
      acc += p.acc_i32[ks * p.acc_slice + ai];
      if (has_aux) aux += p.acc_f32[ks * p.acc_slice + ai];
    }
    const float s_row = p.row_s ? p.row_s[row] : 0.f;
    const int zp = p.row_zp ? p.row_zp[row] : 0;
    if (mode == G2_RAW) {
      const int64_t idx = (int64_t)row * p.ldo + col;
      reinterpret_cast<int*>(p.out)[idx] = acc;
      if (has_aux && p.raw_aux) p.raw_aux[idx] = aux;
    } else if (mode == G2_LR1) {
      g2_epi_lr1(p, p.row_map ? p.row_map[row] : row, col, acc, zp, s_row);
    } else {
      const float rho = (has_aux && p.row_rho) ? p.row_rho[row] : 0.f;
      g2_store1(p, (int64_t)row * p.ldo + col, g2_epi_split(p, col, acc, zp, s_row, rho, has_aux, aux));
    }
  }
}

}  // namespace splitq
