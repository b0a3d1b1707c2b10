// tcgen05 / TMEM / TMA grouped GEMM for sm_100a (bf16 in, fp32 accumulate).
//
// Replaces the reference's grouped_gemm (armt/tensor_ops.py:237-264): every
// matmul of a diagonal step (QKV, O, gate/up, down, memory projections,
// associative read, LM head) is ONE launch over all members of the step, each
// member using its own layer's weights via per-member (slot, layer) tables that
// become TMA coordinates.
//
// Structure (one CTA per SM, persistent over tiles, 256 threads):
//   warp 0      TMA producer: A tile (128 x 64) + B tile (BN x 64) per stage,
//               128B-swizzled, signalled on a full mbarrier (expect_tx).
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16)
//               x4 per stage into a TMEM accumulator; tcgen05.commit frees the
//               stage; the last k-block commits "accumulator full".
//   warp 2      TMEM allocator (2 accumulators x BN columns, double buffered
//               so the epilogue of tile i overlaps the mainloop of tile i+1).
//   warps 4-11  epilogue, two warpgroups: warpgroup e drains TMEM accumulator e
//               (every other tile), so each has two mainloop durations to run
//               tcgen05.ld 32 lanes x 32 cols -> registers -> fused epilogue
//               (residual / guarded retrieve / SwiGLU / RoPE) -> HBM.
//
// Tiles are ordered (member, n-block, m-block) with m fastest, so the CTAs in
// flight share a few weight tiles (read once from HBM) and the member's
// activation (L2-resident).

#include <cuda.h>
#include <cudaTypedefs.h>
#include <vector>
#include <mutex>
#include <cstdlib>
#include <cstring>

#include "tc_ptx.cuh"

namespace armt {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NUM_THREADS = 384;  // 4 control warps + 2 epilogue warpgroups

struct Params {
  int G, M, N, K;
  int tiles_m, tiles_n, num_tiles, k_blocks;
  int c_dtype;
  void* C; long long ldc, c_stride;
  const float* R; long long ldr, r_stride;
  __nv_bfloat16* C2; long long ldc2, c2_stride; int c2_split;
  float* ssq_out; const float* ssq_in; long long ssq_stride; int ssq_np; int norm_d; float norm_eps;
  float2* lse_part; long long lse_ld; const long long* targets; float* lse_tgt; int lse_rows;
  const float* den; long long den_stride;
  float eps;
  const float* rope_cos; const float* rope_sin; int head_dim; int rope_cols; int rope_ld;
  int swiglu_block;
  int max_ctas;
  int row0;    // first row of every member this launch covers (rows [row0, M))
  int* tile_ctr;  // dynamic tile scheduling: {next tile, CTAs done} for this launch (nullptr = static)
  int cst;     // bf16 outputs stored through the smem transpose (coalesced 64 B row segments)
  int xpose;   // residual/retrieve epilogue through the smem transpose (coalesced 128 B rows)
  int prof;    // ARMT_GEMM_PROF=1: accumulate wait cycles of the producer / MMA issuer
  short a_slot[ARMT_MAX_MEMBERS];
  short b_index[ARMT_MAX_MEMBERS];
  short c_slot[ARMT_MAX_MEMBERS];
  short e_index[ARMT_MAX_MEMBERS];
  const float* z; int nu;
  int a_kwrap, b_kwrap;   // operand K-column reuse (see ArmtGemmArgs)
};

// PAIR: a 2-CTA cluster computes a 256 x BN tile with one cta_group::2 MMA per K
// step; each CTA holds its 128 A rows and half (BN/2) of the B rows, so per-CTA
// operand traffic per flop drops by a third and 6 stages fit in the same smem.
// TMAE: TMA epilogue for the short-K residual / retrieve GEMMs — the residual tile is
// TMA-loaded into swizzled smem ahead of the accumulator, and the f32 result and its bf16
// copy leave by TMA stores; it trades mainloop stages for 16 KB of epilogue buffers per warp.
template <int BN, bool PAIR = false, bool TMAE = false> struct Cfg {
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;
  static constexpr int STAGES = TMAE ? (PAIR ? 3 : (BN == 256 ? 2 : (BN == 128 ? 3 : 4)))
                                     : (PAIR ? 6 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8)));
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 512 /*barriers, tile queue*/;
  // residual/retrieve epilogues: one 32 x 32 f32 transpose tile per epilogue warp
  static constexpr int XPOSE_BYTES = 8 * 32 * 32 * 4;
  static constexpr int SMEM_XPOSE = SMEM_BYTES + XPOSE_BYTES;
  // TMAE: per epilogue warp 2 f32 tiles (32 x 32, 128B-swizzled) + 4 bf16 tiles (32 x 32, 64B-swizzled)
  static constexpr int EW_BYTES = 2 * 4096 + 4 * 2048;
  static constexpr int SMEM_TMAE = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + 8 * EW_BYTES;
};

using namespace tcx;

// ---------------------------------------------------------------- epilogues
enum : int { E_STORE = 0, E_RESIDUAL = 1, E_RETRIEVE = 2, E_SWIGLU = 3, E_ROPE = 4, E_LSE = 5, E_DPFP = 6,
             E_FOLDR = 7 };

__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2; exp2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed f32x2 arithmetic (round-to-nearest, the scalar ops' rounding)
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fast_rcp(float x) {  // MUFU.RCP
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifndef ARMT_SWIGLU_FAST
#define ARMT_SWIGLU_FAST 1
#endif

// Store 32 consecutive values of one row starting at column n0 (< N).
__device__ __forceinline__ void store_row32(void* base, int dtype, long long off, int n0, int N,
                                            long long ld, const float (&v)[32]) {
  const int cnt = min(32, N - n0);
  if (dtype == ARMT_BF16) {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base) + off + n0;
    if (cnt == 32 && ((ld & 7) == 0) && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        q[j] = make_uint4(pack_bf16x2(v[8 * j + 0], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                          pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < cnt) p[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* p = reinterpret_cast<float*>(base) + off + n0;
    if (cnt == 32 && ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < cnt) p[j] = v[j];
    }
  }
}

__device__ __forceinline__ void load_row32_f32(const float* p, int cnt, bool vec, float (&v)[32]) {
  if (cnt == 32 && vec) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 t = q[j];
      v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j < cnt ? p[j] : 0.f;
  }
}

// Coalesced bf16 store of a 32-row x 32-column chunk held row-per-lane (lane = row
// wrow0 + lane): bf16 rows go through a 64 B-per-row swizzled smem tile (2 KB per warp)
// and leave as 16 B per lane with 4 lanes per row segment, so each store instruction
// writes 8 full 64 B row segments instead of 32 scattered 16 B pieces.
__device__ __forceinline__ void store_chunk_bf16_coalesced(uint4* tb, int lane, const float (&v)[32],
                                                           __nv_bfloat16* base, long long ld, int wrow0,
                                                           int M, int col0) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    tb[lane * 4 + (c ^ ((lane >> 1) & 3))] =
        make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                   pack_bf16x2(v[8 * c + 4], v[8 * c + 5]), pack_bf16x2(v[8 * c + 6], v[8 * c + 7]));
  __syncwarp();
  const int c = lane & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = (lane >> 2) + 8 * k;
    const uint4 val = tb[r * 4 + (c ^ ((r >> 1) & 3))];
    if (wrow0 + r < M) *reinterpret_cast<uint4*>(base + (long long)(wrow0 + r) * ld + col0 + 8 * c) = val;
  }
  __syncwarp();
}

// RoPE over one chunk of CH (>= DH, multiple of DH) columns held in registers.
// Pairs (i, i + DH/2) inside each head; position = row within the segment.
// cos/sin tables are (DH/2, ld) so a warp (32 consecutive rows) reads one line.
template <int DH, int CH>
__device__ __forceinline__ void rope_chunk(float (&x)[CH], const float* cos_col, const float* sin_col, int ld) {
  constexpr int H2 = DH / 2;
#pragma unroll
  for (int h = 0; h < CH / DH; ++h) {
#pragma unroll
    for (int i = 0; i < H2; ++i) {
      const float c = cos_col[(long long)i * ld], s = sin_col[(long long)i * ld];
      const float a = x[h * DH + i], b = x[h * DH + i + H2];
      x[h * DH + i] = a * c - b * s;
      x[h * DH + i + H2] = b * c + a * s;
    }
  }
}

// ---------------------------------------------------------------- kernel
// [0] MMA: cycles waiting for a full stage, [1] MMA: waiting for a free accumulator,
// [2] MMA: total cycles in the tile loop, [3] producer: waiting for an empty stage,
// [4] tiles, [5] epilogue: cycles waiting for a full accumulator, [6] epilogue: total
__device__ unsigned long long g_gemm_prof[8];

// MC: a 2-CTA cluster of single-CTA MMAs whose two tiles share one operand: the pair
// (m, n), (m+1, n) shares the B tile and (m, n), (m, n+1) the A tile; each CTA loads
// its own unshared operand and HALF of the shared one, multicast into both CTAs'
// smem, so per-CTA L2->SM operand traffic drops by a third with no tile padding.
template <int BN, int EPI, int DH, bool PAIR, bool MC = false, bool TMAE = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
            const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmC,
            const __grid_constant__ CUtensorMap tmC2, const __grid_constant__ Params p) {
  using C = Cfg<BN, PAIR, TMAE>;
  static_assert(!TMAE || EPI == E_RESIDUAL || EPI == E_RETRIEVE, "TMA epilogue: residual / retrieve only");
  constexpr bool CLUSTER = PAIR || MC;
  constexpr int TM = PAIR ? 2 * BM : BM;   // rows per tile (per pair)
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  float4* xpose = reinterpret_cast<float4*>(smem + STAGES * C::STAGE_BYTES + 512);  // residual epilogues
  // dynamic tile queue (single-CTA mode): the producer claims tiles from a global counter
  // and hands them to the MMA thread and the epilogue warpgroups through a smem ring
  constexpr int QD = 8;
  uint64_t* tq_full = bars + 2 * STAGES + 5;
  uint64_t* tq_empty = tq_full + QD;
  volatile int* tq_ids = reinterpret_cast<volatile int*>(tq_empty + QD);
  // TMAE: two residual-tile barriers per epilogue warp, then the per-warp tile buffers
  uint64_t* rbar = bars + 2 * STAGES + 5 + 2 * QD + 4;
  uint8_t* ebuf = smem + STAGES * C::STAGE_BYTES + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CLUSTER ? cluster_ctarank() : 0;
  const int tile0 = CLUSTER ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstep = CLUSTER ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], MC ? 2 : 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], PAIR ? 8 : 4); }
    for (int i = 0; i < QD; ++i) { mbar_init(&tq_full[i], 1); mbar_init(&tq_empty[i], 5); }
    if constexpr (TMAE)
      for (int i = 0; i < 24; ++i) mbar_init(&rbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(C::TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(C::TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CLUSTER) cluster_sync_all();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, tensor maps): overlap it with the previous kernel's tail
  pdl_launch_dependents();
  pdl_wait();

  const int tiles_mn = p.tiles_m * p.tiles_n;
  const bool dyn = !CLUSTER && p.tile_ctr != nullptr;
  // tile index -> (member, n-block, m-block); MC: index = pair slot, see the kernel comment
  bool share_a = false;
  auto decode = [&](int tile, int& g, int& nb, int& mb) {
    if constexpr (MC) {
      const int per_g = (p.tiles_n >> 1) * p.tiles_m;
      g = tile / per_g;
      const int rem = tile - g * per_g, j = rem / p.tiles_m, q = rem - j * p.tiles_m;
      if (q < (p.tiles_m & ~1)) { share_a = false; mb = (q & ~1) + (int)rank; nb = 2 * j + (q & 1); }
      else { share_a = true; mb = p.tiles_m - 1; nb = 2 * j + (int)rank; }
    } else {
      g = tile / tiles_mn;
      const int r = tile - g * tiles_mn;
      nb = r / p.tiles_m;
      mb = r - nb * p.tiles_m;
    }
  };
  // consumer side of the queue: entry k (MMA reads every k, epilogue group eg every k = eg mod 2)
  auto tq_pop = [&](int k, bool epi_warp) -> int {
    const int qs = k % QD;
    mbar_wait_sleep(&tq_full[qs], (uint32_t)((k / QD) & 1));
    const int t = tq_ids[qs];
    if (!epi_warp || lane == 0) mbar_arrive(&tq_empty[qs]);
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0; uint32_t phase = 0;
      unsigned long long w_empty = 0;
      int qk = 0;
      auto tq_push = [&](int t) {
        const int qs = qk % QD;
        mbar_wait(&tq_empty[qs], (uint32_t)(((qk / QD) & 1) ^ 1));
        tq_ids[qs] = t;
        mbar_arrive(&tq_full[qs]);
        ++qk;
      };
      auto claim = [&]() -> int {
        int t = atomicAdd(p.tile_ctr, 1);
        if (t >= p.num_tiles) { tq_push(-1); tq_push(-1); return -1; }  // one sentinel per epilogue group
        tq_push(t);
        return t;
      };
      for (int tile = dyn ? claim() : (tile0 < p.num_tiles ? tile0 : -1); tile >= 0;
           tile = dyn ? claim() : (tile + tstep < p.num_tiles ? tile + tstep : -1)) {
        int g, nb, mb;
        decode(tile, g, nb, mb);
        const int a_slot = p.a_slot[g], b_idx = p.b_index[g];
        const int a_row = p.row0 + mb * TM + (PAIR ? (int)rank * BM : 0);
        const int b_row = nb * BN + (PAIR ? (int)rank * C::B_ROWS : 0);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          if (p.prof) {
            const long long t0 = clock64();
            mbar_wait(&empty[stage], phase ^ 1);
            w_empty += clock64() - t0;
          }
          // K coordinates: a bf16x3 operand stored as [hi | lo] re-reads hi as its third part
          const int ka = (p.a_kwrap > 0 && kb * BK >= p.a_kwrap) ? kb * BK - p.a_kwrap : kb * BK;
          const int kbb = (p.b_kwrap > 0 && kb * BK >= p.b_kwrap) ? kb * BK - p.b_kwrap : kb * BK;
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's full barrier; the leader arms it
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            const uint32_t lbar = mapa_shared(&full[stage], 0);
            tma_load_3d_pair(sA + stage * C::A_BYTES, &tmA, lbar, ka, a_row, a_slot);
            tma_load_3d_pair(sB + stage * C::B_BYTES, &tmB, lbar, kbb, b_row, b_idx);
          } else if constexpr (MC) {
            // own operand unicast; half of the shared one multicast to both CTAs
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            if (!share_a) {
              tma_load_3d(sA + stage * C::A_BYTES, &tmA, &full[stage], ka, a_row, a_slot);
              tma_load_3d_mc(sB + stage * C::B_BYTES + rank * (C::B_BYTES / 2), &tmB2, &full[stage], kbb,
                             b_row + (int)rank * (BN / 2), b_idx, (uint16_t)3);
            } else {
              tma_load_3d(sB + stage * C::B_BYTES, &tmB, &full[stage], kbb, b_row, b_idx);
              tma_load_3d_mc(sA + stage * C::A_BYTES + rank * (C::A_BYTES / 2), &tmA2, &full[stage], ka,
                             a_row + (int)rank * (BM / 2), a_slot, (uint16_t)3);
            }
          } else {
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_3d(sA + stage * C::A_BYTES, &tmA, &full[stage], ka, a_row, a_slot);
            tma_load_3d(sB + stage * C::B_BYTES, &tmB, &full[stage], kbb, b_row, b_idx);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (p.prof) atomicAdd(&g_gemm_prof[3], w_empty);
      if (dyn) {
        // last CTA out resets the launch's counter pair (graph replays start from zero)
        __threadfence();
        if (atomicAdd(p.tile_ctr + 1, 1) == (int)gridDim.x - 1) {
          atomicExch(p.tile_ctr, 0);
          atomicExch(p.tile_ctr + 1, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (!PAIR || rank == 0)) {
      // ---------------- MMA issuer (single thread; the pair leader in PAIR mode)
      constexpr uint32_t idesc = instr_desc<TM, BN>();
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      unsigned long long w_full = 0, w_acc = 0, n_tiles = 0;
      const long long t_start = clock64();
      int qk = 0;
      for (int tile = dyn ? tq_pop(qk++, false) : (tile0 < p.num_tiles ? tile0 : -1); tile >= 0;
           tile = dyn ? tq_pop(qk++, false) : (tile + tstep < p.num_tiles ? tile + tstep : -1)) {
        if (p.prof) {
          const long long t0 = clock64();
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          w_acc += clock64() - t0;
          ++n_tiles;
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          if (p.prof) {
            const long long t0 = clock64();
            mbar_wait(&full[stage], phase);
            w_full += clock64() - t0;
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a_desc = smem_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t b_desc = smem_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {  // +32 B per K=16 step inside the swizzle atom
            if constexpr (PAIR) mma_bf16_pair(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
            else mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (PAIR) mma_commit_pair(&empty[stage]);
          else if constexpr (MC) mma_commit_mc(&empty[stage], (uint16_t)3);  // both CTAs may refill
          else mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR) mma_commit_pair(&tfull[acc]);
        else mma_commit(&tfull[acc]);
        acc ^= 1; if (acc == 0) acc_phase ^= 1;
      }
      if (p.prof) {
        atomicAdd(&g_gemm_prof[0], w_full);
        atomicAdd(&g_gemm_prof[1], w_acc);
        atomicAdd(&g_gemm_prof[2], (unsigned long long)(clock64() - t_start));
        atomicAdd(&g_gemm_prof[4], n_tiles);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warpgroup eg owns accumulator eg; TMEM lanes 32*(warp%4) .. +31
    const int ew = warp & 3;
    const int eg = (warp - 4) >> 2;
    const int acc = eg;
    uint32_t acc_phase = 0;
    uint32_t rph = 0;   // TMAE: parity of this warp's residual-tile barriers (one bit per buffer)
    int qk = eg;
    auto first = [&]() { const int t = tile0 + eg * tstep; return t < p.num_tiles ? t : -1; };
    for (int tile = dyn ? tq_pop(qk, true) : first(); tile >= 0;
         tile = dyn ? tq_pop(qk += 2, true) : (tile + 2 * tstep < p.num_tiles ? tile + 2 * tstep : -1)) {
      int g, nb, mb;
      decode(tile, g, nb, mb);
      const int row = p.row0 + mb * TM + (PAIR ? (int)rank * BM : 0) + ew * 32 + lane;
      const bool live = row < p.M;
      const int c_slot = p.c_slot[g];
      // TMAE: chunks of this tile inside N, and the first two residual tiles requested now
      // (they do not depend on the MMA, so they land while the mainloop runs)
      const int ncv = TMAE ? min(BN / 32, (p.N - nb * BN + 31) / 32) : 0;
      uint8_t* wbuf = ebuf + (warp - 4) * C::EW_BYTES;
      // residual buffers in flight per warp: three when there is no [hi | lo] split output
      // (the lo staging space holds the third f32 tile), else two
      const int nbuf = p.c2_split > 0 ? 2 : 3;
      auto fbuf = [&](int b) { return wbuf + (b < 2 ? b * 4096 : 12288); };
      if constexpr (TMAE) {
        if (lane == 0) {
          bulk_wait_read0();   // the previous tile's stores have left these buffers
          const int wr0 = p.row0 + mb * TM + (PAIR ? (int)rank * BM : 0) + ew * 32;
          for (int c = 0; c < nbuf && c < ncv; ++c) {
            mbar_expect_tx(&rbar[3 * (warp - 4) + c], 4096);
            tma_load_3d(fbuf(c), &tmR, &rbar[3 * (warp - 4) + c], nb * BN + 32 * c, wr0, c_slot);
          }
        }
      }
      if (p.prof && lane == 0) {
        const long long t0 = clock64();
        mbar_wait_sleep(&tfull[acc], acc_phase);
        atomicAdd(&g_gemm_prof[5], (unsigned long long)(clock64() - t0));
      }
      // one warp of the warpgroup polls the accumulator barrier; the other three wait on a
      // named barrier (blocked in hardware, no issue slots or power spent re-polling)
      __syncwarp();
      if (ew == 0) mbar_wait_sleep(&tfull[acc], acc_phase);
      asm volatile("bar.sync %0, 128;" ::"r"(1 + eg) : "memory");
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      const long long off = (long long)c_slot * p.c_stride + (long long)row * p.ldc;
      // fused RMSNorm of the A rows: acc * 1/sqrt(mean(x^2) + eps) (gains live in the weights)
      float rs = 1.f;
      if constexpr (EPI == E_SWIGLU || EPI == E_ROPE) {
        if (p.ssq_in != nullptr && live) {
          const float* part = p.ssq_in + (long long)g * p.ssq_stride + (long long)row * p.ssq_np;
          float t = 0.f;
          int q = 0;
          if ((p.ssq_np & 3) == 0) {  // float4 loads, all issued before the (fixed-order) sum
            float4 v[8];
            for (; q + 32 <= p.ssq_np; q += 32) {
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = reinterpret_cast<const float4*>(part + q)[u];
#pragma unroll
              for (int u = 0; u < 8; ++u) t += ((v[u].x + v[u].y) + (v[u].z + v[u].w));
            }
            for (; q < p.ssq_np; q += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(part + q);
              t += ((w4.x + w4.y) + (w4.z + w4.w));
            }
          }
          for (; q < p.ssq_np; ++q) t += part[q];  // fixed order: deterministic
          rs = 1.f / sqrtf(t / (float)p.norm_d + p.norm_eps);
        }
      }

      if constexpr (EPI == E_DPFP) {
        // acc row = q (d_mem = DH <= 64 columns): phi = DPFP_nu(q) straight to bf16 (the
        // retrieval numerator's A operand) and den = phi . z[layer], one row per thread
        // (armt/memory.py:34-45,137-147); replaces the q f32 round trip + a separate kernel
        static_assert(DH >= 8 && DH <= 64, "DPFP epilogue: d_mem in [8, 64]");
        float qv[64];
        __syncwarp();
        tmem_ld32(tbase, *reinterpret_cast<float(*)[32]>(qv));
        if constexpr (DH > 32) {
          __syncwarp();
          tmem_ld32(tbase + 32, *reinterpret_cast<float(*)[32]>(qv + 32));
        }
        const float* zr = p.z + (long long)p.e_index[g] * (2 * DH * p.nu);
        __nv_bfloat16* cb = reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)c_slot * p.c_stride;
        uint4* tb = reinterpret_cast<uint4*>(xpose) + (warp - 4) * 128;
        float dacc = 0.f;
        auto rv = [&](int i) { return i < DH ? fmaxf(qv[i], 0.f) : fmaxf(-qv[i - DH], 0.f); };
#pragma unroll
        for (int j = 1; j <= 3; ++j) {
          if (j > p.nu) break;  // warp-uniform
#pragma unroll
          for (int c0 = 0; c0 < 2 * DH; c0 += 32) {
            float ph[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const int i = c0 + t;
              ph[t] = (i < 2 * DH) ? rv(i) * rv((i + j) % (2 * DH)) : 0.f;
            }
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (c0 + t < 2 * DH) dacc = fmaf(ph[t], zr[(j - 1) * 2 * DH + c0 + t], dacc);
            const int col0 = (j - 1) * 2 * DH + c0;
            if constexpr ((2 * DH) % 32 == 0) {
              store_chunk_bf16_coalesced(tb, lane, ph, cb, p.ldc, row - lane, p.M, col0);
            } else {
              if (live) store_row32(p.C, ARMT_BF16, off, col0, col0 + min(32, 2 * DH - c0), p.ldc, ph);
            }
          }
        }
        if (live) const_cast<float*>(p.den)[(long long)g * p.den_stride + row] = dacc;  // (RETRIEVE reads den)
      } else if constexpr (EPI == E_FOLDR) {
        // The fold's transposed projection (memory_tc.cu): acc[r][i] = (A0 phi_i)[r]. Row r of
        // member g's output, segments of seg = c2_split token columns:
        //   [V hi | P hi | V lo | P lo],  V[r][i] = v_i[r] (R: token-major value rows)
        // i.e. the bf16x3 A operand of the fold's update GEMM A_M = A0 + [V^T | P^T] [Y ; Z]^T,
        // whose third part [V hi | P hi] is re-read from the first through a K wrap.
        const int seg = p.c2_split;
        __nv_bfloat16* cb = reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)c_slot * p.c_stride;
        const float* vb = p.R + (long long)c_slot * p.r_stride;
        uint4* tb = reinterpret_cast<uint4*>(xpose) + (warp - 4) * 128;
        const int wrow0 = row - lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          const int n0 = nb * BN + c0;
          if (n0 >= seg) break;  // warp-uniform
          float v[32];
          __syncwarp();
          tmem_ld32(tbase + c0, v);
          float vv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) vv[j] = (live && n0 + j < p.N) ? vb[(long long)(n0 + j) * p.ldr + row] : 0.f;
          float hi[32], lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            hi[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
            lo[j] = v[j] - hi[j];
            v[j] = __bfloat162float(__float2bfloat16_rn(vv[j]));   // V hi
            vv[j] = vv[j] - v[j];                                  // V lo
          }
          if (n0 + 32 <= seg) {  // warp-uniform: whole 32-column chunks through the smem transpose
            store_chunk_bf16_coalesced(tb, lane, v, cb, p.ldc, wrow0, p.M, n0);
            store_chunk_bf16_coalesced(tb, lane, hi, cb, p.ldc, wrow0, p.M, seg + n0);
            store_chunk_bf16_coalesced(tb, lane, vv, cb, p.ldc, wrow0, p.M, 2 * seg + n0);
            store_chunk_bf16_coalesced(tb, lane, lo, cb, p.ldc, wrow0, p.M, 3 * seg + n0);
          } else if (live) {
            __nv_bfloat16* o = cb + (long long)row * p.ldc + n0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (n0 + j < seg) {
                o[j] = __float2bfloat16_rn(v[j]);
                o[seg + j] = __float2bfloat16_rn(hi[j]);
                o[2 * seg + j] = __float2bfloat16_rn(vv[j]);
                o[3 * seg + j] = __float2bfloat16_rn(lo[j]);
              }
            }
          }
        }
      } else if constexpr (EPI == E_LSE) {
        // fused next-token NLL: online (max, sum 2^x) of the row's logits in base 2
        constexpr float LOG2E = 1.4426950408889634f;
        float m = -INFINITY, ssum = 0.f, tv = 0.f;
        const long long tgt = (live && row < p.lse_rows) ? p.targets[row] : -1;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tbase + c0, v);
          const int n0 = nb * BN + c0;
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = (n0 + j < p.N) ? v[j] * LOG2E : -INFINITY;
            cm = fmaxf(cm, v[j]);
            if (n0 + j == tgt) tv = v[j];
          }
          const float mn = fmaxf(m, cm);
          if (mn == -INFINITY) continue;  // whole chunk past N
          float cs = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) cs += fast_exp2(v[j] - mn);
          ssum = (m == -INFINITY ? 0.f : ssum * fast_exp2(m - mn)) + cs;
          m = mn;
        }
        if (live && row < p.lse_rows) {
          p.lse_part[(long long)row * p.lse_ld + nb] = make_float2(m, ssum);
          if (tgt >= (long long)nb * BN && tgt < (long long)nb * BN + BN && tgt < p.N) p.lse_tgt[row] = tv;
        }
      } else if constexpr (EPI == E_SWIGLU) {
        const int out_n0 = nb * (BN / 2);
#pragma unroll 1
        for (int c0 = 0; c0 < BN / 2; c0 += 32) {
          float gte[32], up[32];
          __syncwarp();
          tmem_ld32(tbase + c0, gte);
          tmem_ld32(tbase + BN / 2 + c0, up);
#if ARMT_SWIGLU_FAST
          // silu(g) = g / (1 + 2^(-g log2 e)): MUFU.EX2 + MUFU.RCP (approximate, ~2 ulp, far
          // below the bf16 rounding of the output) instead of the IEEE reciprocal sequence.
          // The multiplies and the add run as packed f32x2 pairs (the same IEEE operations in
          // the same order as the scalar form, so bitwise the same result, in half the issues).
          const unsigned long long rs2 = pk2(rs, rs), nl2 = pk2(-1.4426950408889634f, -1.4426950408889634f),
                                   one2 = pk2(1.f, 1.f);
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const unsigned long long gv = fmul2(pk2(gte[j], gte[j + 1]), rs2);
            float e0, e1;
            upk2(fmul2(nl2, gv), e0, e1);
            const unsigned long long den = fadd2(one2, pk2(fast_exp2(e0), fast_exp2(e1)));
            float d0, d1;
            upk2(den, d0, d1);
            const unsigned long long a = fmul2(gv, pk2(fast_rcp(d0), fast_rcp(d1)));
            upk2(fmul2(a, fmul2(pk2(up[j], up[j + 1]), rs2)), gte[j], gte[j + 1]);
          }
#else
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float gv = gte[j] * rs;
            gte[j] = gv * __frcp_rn(1.f + __expf(-gv)) * (up[j] * rs);
          }
#endif
          if (p.cst && out_n0 + c0 + 32 <= p.N / 2) {
            store_chunk_bf16_coalesced(reinterpret_cast<uint4*>(xpose) + (warp - 4) * 128, lane, gte,
                                       reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)c_slot * p.c_stride,
                                       p.ldc, row - lane, p.M, out_n0 + c0);
          } else if (live && out_n0 + c0 < p.N / 2) {
            store_row32(p.C, ARMT_BF16, off, out_n0 + c0, p.N / 2, p.ldc, gte);
          }
        }
      } else if constexpr (EPI == E_ROPE) {
        // tables are (DH/2, M) column-major in position: lane = row reads consecutive words
        const long long tr = live ? row : 0;
        const float* cos_col = p.rope_cos + tr;
        const float* sin_col = p.rope_sin + tr;
        constexpr int CH = DH > 32 ? DH : 32;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += CH) {
          const int n0 = nb * BN + c0;
          const bool rot = n0 < p.rope_cols;
          if constexpr (DH >= 64) {
            // pairs (i, i + DH/2): rotate in 32-column sub-chunks to bound registers
#pragma unroll 1
            for (int q = 0; q < DH / 64; ++q) {
              float x1[32], x2[32];
              __syncwarp();
              tmem_ld32(tbase + c0 + 32 * q, x1);
              tmem_ld32(tbase + c0 + DH / 2 + 32 * q, x2);
              if (live && n0 < p.N) {
#pragma unroll
                for (int j = 0; j < 32; ++j) { x1[j] *= rs; x2[j] *= rs; }
                if (rot) {
#pragma unroll
                  for (int j = 0; j < 32; ++j) {
                    const float cs = cos_col[(long long)(32 * q + j) * p.rope_ld], sn = sin_col[(long long)(32 * q + j) * p.rope_ld];
                    const float a = x1[j], b = x2[j];
                    x1[j] = a * cs - b * sn;
                    x2[j] = b * cs + a * sn;
                  }
                }
                if (!p.cst) {
                  store_row32(p.C, ARMT_BF16, off, n0 + 32 * q, p.N, p.ldc, x1);
                  store_row32(p.C, ARMT_BF16, off, n0 + DH / 2 + 32 * q, p.N, p.ldc, x2);
                }
              }
              if (p.cst && n0 + DH <= p.N) {  // (warp-uniform: every lane stores through smem)
                uint4* tb = reinterpret_cast<uint4*>(xpose) + (warp - 4) * 128;
                __nv_bfloat16* cb = reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)c_slot * p.c_stride;
                store_chunk_bf16_coalesced(tb, lane, x1, cb, p.ldc, row - lane, p.M, n0 + 32 * q);
                store_chunk_bf16_coalesced(tb, lane, x2, cb, p.ldc, row - lane, p.M, n0 + DH / 2 + 32 * q);
              } else if (p.cst && live && n0 < p.N) {
                store_row32(p.C, ARMT_BF16, off, n0 + 32 * q, p.N, p.ldc, x1);
                store_row32(p.C, ARMT_BF16, off, n0 + DH / 2 + 32 * q, p.N, p.ldc, x2);
              }
            }
          } else {
            float x[32];
            __syncwarp();
            tmem_ld32(tbase + c0, x);
            if (live && n0 < p.N) {
#pragma unroll
              for (int j = 0; j < 32; ++j) x[j] *= rs;
              if (rot) rope_chunk<DH, 32>(x, cos_col, sin_col, p.rope_ld);
              store_row32(p.C, ARMT_BF16, off, n0, p.N, p.ldc, x);
            }
          }
        }
      } else {
        float rden = 1.f; bool guarded = false;
        float ssq = 0.f;
        if constexpr (EPI == E_RETRIEVE) {
          const float den = live ? p.den[(long long)g * p.den_stride + row] : 1.f;
          guarded = fabsf(den) <= p.eps;
          rden = 1.f / den;
        }
        if constexpr (EPI == E_RESIDUAL || EPI == E_RETRIEVE) {
          if constexpr (TMAE) {
            // lane = row. Residual tile (f32, 128B swizzle: 16-byte chunk k of row r at k ^ (r & 7))
            // -> o = R + f(acc) written back in place -> TMA store; bf16 copy (64B swizzle: chunk k
            // of row r at k ^ ((r >> 1) & 3)) -> TMA store. Row sums of squares per 64 columns in the
            // same order as the xpose path (4-column fma chains, then a fixed pairwise tree).
            const int wrow0 = p.row0 + mb * TM + (PAIR ? (int)rank * BM : 0) + ew * 32;
            const int wi = warp - 4;
            const bool split = p.c2_split > 0;
            float sq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sq[k] = 0.f;
#pragma unroll 1
            for (int c = 0, b = 0; c < ncv; ++c, b = b + 1 == nbuf ? 0 : b + 1) {
              const int h = c & 1, c0 = 32 * c, n0 = nb * BN + c0;
              float v[32];
              __syncwarp();
              tmem_ld32(tbase + c0, v);
              mbar_wait(&rbar[3 * wi + b], (rph >> b) & 1);
              rph ^= 1u << b;
              // refill the previous chunk's buffer now: its stores have had this chunk's TMEM
              // load and barrier wait to finish reading it
              if (c >= 1 && lane == 0) {
                const int pb = b == 0 ? nbuf - 1 : b - 1;
                if (c - 1 + nbuf < ncv) {
                  bulk_wait_read0();
                  mbar_expect_tx(&rbar[3 * wi + pb], 4096);
                  tma_load_3d(fbuf(pb), &tmR, &rbar[3 * wi + pb], n0 - 32 + 32 * nbuf, wrow0, c_slot);
                }
              }
              if (nbuf == 3 && c >= 2) {   // the bf16 staging buffer h was last stored by chunk c - 2
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
              }
              float4* fb = reinterpret_cast<float4*>(fbuf(b)) + lane * 8;
              uint4* hb = reinterpret_cast<uint4*>(wbuf + 8192 + h * 2048) + lane * 4;
              uint4* lb = reinterpret_cast<uint4*>(wbuf + 8192 + (2 + h) * 2048) + lane * 4;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float4 r4 = fb[k ^ (lane & 7)];
                float a0 = v[4 * k], a1 = v[4 * k + 1], a2 = v[4 * k + 2], a3 = v[4 * k + 3];
                if constexpr (EPI == E_RETRIEVE) {
                  a0 = guarded ? 0.f : a0 * rden; a1 = guarded ? 0.f : a1 * rden;
                  a2 = guarded ? 0.f : a2 * rden; a3 = guarded ? 0.f : a3 * rden;
                }
                float4 o;
                o.x = r4.x + a0; o.y = r4.y + a1; o.z = r4.z + a2; o.w = r4.w + a3;
                fb[k ^ (lane & 7)] = o;
                sq[k] = fmaf(o.w, o.w, fmaf(o.z, o.z, fmaf(o.y, o.y, fmaf(o.x, o.x, sq[k]))));
                v[4 * k] = o.x; v[4 * k + 1] = o.y; v[4 * k + 2] = o.z; v[4 * k + 3] = o.w;
              }
              if (p.C2 != nullptr) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int pk = k ^ ((lane >> 1) & 3);
                  hb[pk] = make_uint4(pack_bf16x2(v[8 * k], v[8 * k + 1]), pack_bf16x2(v[8 * k + 2], v[8 * k + 3]),
                                      pack_bf16x2(v[8 * k + 4], v[8 * k + 5]), pack_bf16x2(v[8 * k + 6], v[8 * k + 7]));
                  if (split) {
                    float l[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) l[u] = v[8 * k + u] - __bfloat162float(__float2bfloat16_rn(v[8 * k + u]));
                    lb[pk] = make_uint4(pack_bf16x2(l[0], l[1]), pack_bf16x2(l[2], l[3]),
                                        pack_bf16x2(l[4], l[5]), pack_bf16x2(l[6], l[7]));
                  }
                }
              }
              fence_async_smem();   // generic-proxy smem writes -> visible to the TMA engine
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&tmC, fbuf(b), n0, wrow0, c_slot);
                if (p.C2 != nullptr) {
                  tma_store_3d(&tmC2, wbuf + 8192 + h * 2048, n0, wrow0, c_slot);
                  if (split) tma_store_3d(&tmC2, wbuf + 8192 + (2 + h) * 2048, n0 + p.c2_split, wrow0, c_slot);
                }
                bulk_commit();

              }
              if (p.ssq_out != nullptr && ((n0 & 63) == 32 || n0 + 32 >= p.N)) {
                const float t = ((sq[0] + sq[1]) + (sq[2] + sq[3])) + ((sq[4] + sq[5]) + (sq[6] + sq[7]));
                if (live) p.ssq_out[(long long)g * p.ssq_stride + (long long)row * p.ssq_np + (n0 >> 6)] = t;
#pragma unroll
                for (int k = 0; k < 8; ++k) sq[k] = 0.f;
              }
            }
            goto epi_done;
          }
          if (p.xpose) {
            // Each 32 x 32 chunk: TMEM -> registers (lane = row) -> swizzled smem tile ->
            // registers with lane = (row group, 4-column group): the residual load and the
            // f32 / bf16 stores then move whole 128 B / 64 B row segments per 8 lanes
            // (4x fewer L1 wavefronts than row-per-lane 16 B accesses).
            float4* tb = xpose + (warp - 4) * 256;
            const int m4 = lane & 7, rq = lane >> 3;
            const int wrow0 = p.row0 + mb * TM + (PAIR ? (int)rank * BM : 0) + ew * 32;
            const float* rbase = p.R + (long long)c_slot * p.r_stride;
            float* cbase = reinterpret_cast<float*>(p.C) + (long long)c_slot * p.c_stride;
            __nv_bfloat16* c2base = p.C2 == nullptr ? nullptr : p.C2 + (long long)c_slot * p.c2_stride;
            float sq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sq[k] = 0.f;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
              float v[32];
              __syncwarp();
              tmem_ld32(tbase + c0, v);
              const int n0 = nb * BN + c0;
              if (n0 >= p.N) break;  // warp-uniform
              if constexpr (EPI == E_RETRIEVE) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = guarded ? 0.f : v[j] * rden;
              }
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4)
                tb[lane * 8 + (c4 ^ (lane & 7))] = make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
              __syncwarp();
              const int col = n0 + 4 * m4;
              const bool cok = col < p.N;
              float4 res[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int grow = wrow0 + rq + 4 * k;
                res[k] = (cok && grow < p.M) ? *reinterpret_cast<const float4*>(rbase + (long long)grow * p.ldr + col)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int r = rq + 4 * k, grow = wrow0 + r;
                const float4 a = tb[r * 8 + (m4 ^ (r & 7))];
                float4 o;
                o.x = res[k].x + a.x; o.y = res[k].y + a.y; o.z = res[k].z + a.z; o.w = res[k].w + a.w;
                if (cok && grow < p.M) {
                  *reinterpret_cast<float4*>(cbase + (long long)grow * p.ldc + col) = o;
                  if (c2base != nullptr) {
                    __nv_bfloat16* q = c2base + (long long)grow * p.ldc2 + col;
                    const uint2 hi = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
                    *reinterpret_cast<uint2*>(q) = hi;
                    if (p.c2_split > 0) {
                      const uint2 lo = make_uint2(
                          pack_bf16x2(o.x - __bfloat162float(__float2bfloat16_rn(o.x)),
                                      o.y - __bfloat162float(__float2bfloat16_rn(o.y))),
                          pack_bf16x2(o.z - __bfloat162float(__float2bfloat16_rn(o.z)),
                                      o.w - __bfloat162float(__float2bfloat16_rn(o.w))));
                      *reinterpret_cast<uint2*>(q + p.c2_split) = lo;
                    }
                  }
                }
                sq[k] = fmaf(o.w, o.w, fmaf(o.z, o.z, fmaf(o.y, o.y, fmaf(o.x, o.x, sq[k]))));
              }
              __syncwarp();  // the tile is rewritten by the next chunk
              if (p.ssq_out != nullptr && ((n0 & 63) == 32 || n0 + 32 >= p.N)) {
                // row sums over the 8 lanes of each row group (fixed butterfly order)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  float t = sq[k];
                  t += __shfl_xor_sync(0xffffffffu, t, 1);
                  t += __shfl_xor_sync(0xffffffffu, t, 2);
                  t += __shfl_xor_sync(0xffffffffu, t, 4);
                  const int grow = wrow0 + rq + 4 * k;
                  if (m4 == 0 && grow < p.M)
                    p.ssq_out[(long long)g * p.ssq_stride + (long long)grow * p.ssq_np + (n0 >> 6)] = t;
                  sq[k] = 0.f;
                }
              }
            }
            goto epi_done;
          }
        }
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tbase + c0, v);
          const int n0 = nb * BN + c0;
          if constexpr (EPI == E_STORE) {
            if (p.cst && p.c_dtype == ARMT_BF16 && n0 + 32 <= p.N) {  // warp-uniform
              store_chunk_bf16_coalesced(reinterpret_cast<uint4*>(xpose) + (warp - 4) * 128, lane, v,
                                         reinterpret_cast<__nv_bfloat16*>(p.C) + (long long)c_slot * p.c_stride,
                                         p.ldc, row - lane, p.M, n0);
              continue;
            }
          }
          if (!live || n0 >= p.N) continue;  // after the warp-wide load: safe
          if constexpr (EPI == E_RESIDUAL || EPI == E_RETRIEVE) {
            const float* rp = p.R + (long long)c_slot * p.r_stride + (long long)row * p.ldr + n0;
            float res[32];
            load_row32_f32(rp, min(32, p.N - n0),
                           ((p.ldr & 3) == 0) && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0), res);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if constexpr (EPI == E_RETRIEVE) v[j] = res[j] + (guarded ? 0.f : v[j] * rden);
              else v[j] = res[j] + v[j];
            }
            store_row32(p.C, ARMT_F32, off, n0, p.N, p.ldc, v);
            if (p.ssq_out != nullptr) {
              // partial sum of squares per 64-column block (two 32-column chunks)
#pragma unroll
              for (int j = 0; j < 32; ++j) ssq = (n0 + j < p.N) ? fmaf(v[j], v[j], ssq) : ssq;
              if ((n0 & 63) == 32 || n0 + 32 >= p.N) {
                p.ssq_out[(long long)g * p.ssq_stride + (long long)row * p.ssq_np + (n0 >> 6)] = ssq;
                ssq = 0.f;
              }
            }
            if (p.C2 != nullptr) {
              const long long off2 = (long long)c_slot * p.c2_stride + (long long)row * p.ldc2;
              if (p.c2_split > 0) {
                // bf16x3 operand layout [hi | lo] (hi re-read as the third part through a K wrap):
                // v ~= hi + lo to ~2^-16 relative
                float hi[32], lo[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  hi[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
                  lo[j] = v[j] - hi[j];
                }
                store_row32(p.C2, ARMT_BF16, off2, n0, p.N, p.ldc2, hi);
                store_row32(p.C2, ARMT_BF16, off2 + p.c2_split, n0, p.N, p.ldc2, lo);
              } else {
                store_row32(p.C2, ARMT_BF16, off2, n0, p.N, p.ldc2, v);
              }
            }
          } else {
            store_row32(p.C, p.c_dtype, off, n0, p.N, p.ldc, v);
          }
        }
      }
    epi_done:
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_remote(mapa_shared(&tempty[acc], 0));  // leader's barrier
        else mbar_arrive(&tempty[acc]);
      }
      acc_phase ^= 1;
    }
  }

  if constexpr (TMAE) {
    if (warp >= 4 && lane == 0) bulk_wait0();   // TMA stores complete before the CTA's smem goes away
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if constexpr (CLUSTER) cluster_sync_all();  // the peer may still read our smem / signal our barriers
  tc_fence_after();
  if (warp == 2) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(C::TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(C::TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3D bf16 map: (cols=K contiguous, rows, batch) with a (64, box_rows, 1) box, 128B swizzle.
static int make_map(CUtensorMap* map, const void* base, long long cols, long long rows,
                    long long batches, long long ld, long long batch_stride, int box_rows) {
  auto encode = get_encode();
  ARMT_REQUIRE(encode != nullptr, ARMT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  ARMT_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, ARMT_ERR_DIM, "TMA base not 16B aligned");
  ARMT_REQUIRE((ld * 2) % 16 == 0 && (batch_stride * 2) % 16 == 0, ARMT_ERR_DIM,
               "TMA strides must be multiples of 16 bytes (ld=%lld, batch=%lld)", ld, batch_stride);
  if (batches == 1) batch_stride = rows * ld;  // unused dimension; any legal stride
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batches};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(batch_stride * 2)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ARMT_REQUIRE(r == CUDA_SUCCESS, ARMT_ERR_DIM, "cuTensorMapEncodeTiled failed (%d): cols=%lld rows=%lld batches=%lld ld=%lld",
               (int)r, cols, rows, batches, ld);
  return ARMT_OK;
}

// Epilogue tile maps (TMAE): (cols, rows, batch) with a (32, 32, 1) box; f32 tiles 128B-swizzled,
// bf16 tiles 64B-swizzled (the swizzles the epilogue's row-per-lane smem accesses assume).
static int make_epi_map(CUtensorMap* map, bool f32, const void* base, long long cols, long long rows,
                        long long batches, long long ld, long long batch_stride) {
  auto encode = get_encode();
  ARMT_REQUIRE(encode != nullptr, ARMT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const long long es = f32 ? 4 : 2;
  if (batches == 1) batch_stride = rows * ld;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batches};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * es), (cuuint64_t)(batch_stride * es)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ARMT_REQUIRE(r == CUDA_SUCCESS, ARMT_ERR_DIM, "epilogue tensor map failed (%d)", (int)r);
  return ARMT_OK;
}

struct Maps { CUtensorMap a, b, a2, b2, r, c, c2; };

template <int BN, int EPI, int DH, bool PAIR, bool MC, bool TMAE = false>
static int launch(const Maps& m, const Params& p, cudaStream_t s) {
  auto kern = gemm_kernel<BN, EPI, DH, PAIR, MC, TMAE>;
  constexpr int smem = TMAE ? Cfg<BN, PAIR, true>::SMEM_TMAE
                            : (EPI == E_LSE) ? Cfg<BN, PAIR>::SMEM_BYTES : Cfg<BN, PAIR>::SMEM_XPOSE;
  static_assert(smem <= 227 * 1024, "GEMM shared memory budget");
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_done = true;
  }
  const int cap = p.max_ctas > 0 && p.max_ctas < num_sms() ? p.max_ctas : num_sms();
  if constexpr (PAIR || MC) {
    // one 2-CTA cluster per pair of SMs, persistent over pair tiles / pair slots
    const int pairs = cap / 2 < 1 ? 1 : cap / 2;
    const int grid = 2 * (p.num_tiles < pairs ? p.num_tiles : pairs);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m.a, m.b, m.a2, m.b2, m.r, m.c, m.c2, p);
    ARMT_REQUIRE(e == cudaSuccess, ARMT_ERR_CUDA, "tcgen05 cluster gemm launch: %s", cudaGetErrorString(e));
  } else {
    const int grid = p.num_tiles < cap ? p.num_tiles : cap;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m.a, m.b, m.a2, m.b2, m.r, m.c, m.c2, p);
    ARMT_REQUIRE(e == cudaSuccess, ARMT_ERR_CUDA, "tcgen05 gemm launch: %s", cudaGetErrorString(e));
  }
  ARMT_CHECK_LAUNCH("tcgen05 gemm launch");
  return ARMT_OK;
}

static int pick_bn(const ArmtGemmArgs& a) {
  if (a.epilogue == ARMT_EPI_SWIGLU) return 2 * a.swiglu_block;
  if (a.epilogue == ARMT_EPI_LSE) return 256;  // lse_ld = ceil(N / 256) partials per row
  if (a.epilogue == ARMT_EPI_DPFP) return 64;  // one tile holds a whole q row
  if (a.epilogue == ARMT_EPI_FOLDR) return a.N <= 64 ? 64 : 128;  // token columns (n_mem <= 128)
  if (const char* f = getenv("ARMT_GEMM_BN")) {  // tests: force a tile width
    const int v = atoi(f);
    if ((v == 64 || v == 128 || v == 256) && (a.epilogue != ARMT_EPI_ROPE || (v >= 128 && v % a.head_dim == 0)))
      return v;
  }
  const int sms = num_sms();
  const long long tm = (a.M + BM - 1) / BM;
  const bool rope = a.epilogue == ARMT_EPI_ROPE;
  int best = rope ? 128 : 64;
  double best_score = -1.0;
  for (int bn : {256, 128, 64}) {
    if (rope && (bn < 128 || bn % a.head_dim != 0)) continue;
    const long long tn = (a.N + bn - 1) / bn;
    const long long tiles = (long long)a.G * tm * tn;
    const long long waves = (tiles + sms - 1) / sms;
    const double fill = (double)tiles / (double)(waves * sms);      // wave quantisation
    const double useful = (double)a.N / (double)(tn * bn);          // N padding
    const double size = bn == 256 ? 1.0 : bn == 128 ? 0.93 : 0.8;   // per-tile efficiency
    // a single wave leaves every CTA's epilogue exposed (nothing to overlap it with):
    // small grouped GEMMs (memory-token k/v/beta, fold) prefer two tiles per CTA
    const double one_wave = (waves == 1 && tiles > sms / 2) ? 0.8 : 1.0;
    const double score = fill * useful * size * one_wave;
    if (score > best_score + 1e-9) { best_score = score; best = bn; }
  }
  return best;
}

template <int BN, bool PAIR, bool MC>
static int dispatch_epi(const ArmtGemmArgs& a, const Maps& m, const Params& p,
                        cudaStream_t s, bool tmae) {
  switch (a.epilogue) {
    case ARMT_EPI_STORE: return launch<BN, E_STORE, 0, PAIR, MC>(m, p, s);
    case ARMT_EPI_RESIDUAL:
      if (tmae) return launch<BN, E_RESIDUAL, 0, PAIR, MC, true>(m, p, s);
      return launch<BN, E_RESIDUAL, 0, PAIR, MC>(m, p, s);
    case ARMT_EPI_RETRIEVE:
      if (tmae) return launch<BN, E_RETRIEVE, 0, PAIR, MC, true>(m, p, s);
      return launch<BN, E_RETRIEVE, 0, PAIR, MC>(m, p, s);
    case ARMT_EPI_LSE:
      if constexpr (BN == 256) return launch<BN, E_LSE, 0, PAIR, MC>(m, p, s);
      break;
    case ARMT_EPI_DPFP:
      if constexpr (BN == 64 && !PAIR && !MC) {
        switch (a.N) {
          case 16: return launch<BN, E_DPFP, 16, false, false>(m, p, s);
          case 32: return launch<BN, E_DPFP, 32, false, false>(m, p, s);
          case 64: return launch<BN, E_DPFP, 64, false, false>(m, p, s);
          default: break;
        }
      }
      break;
    case ARMT_EPI_SWIGLU:
      if constexpr (BN == 64 || BN == 256) return launch<BN, E_SWIGLU, 0, PAIR, MC>(m, p, s);
      break;
    case ARMT_EPI_FOLDR:
      if constexpr ((BN == 64 || BN == 128) && !PAIR && !MC) return launch<BN, E_FOLDR, 0, false, false>(m, p, s);
      break;
    case ARMT_EPI_ROPE:
      if constexpr (BN >= 128) {
        switch (a.head_dim) {
          case 8: return launch<BN, E_ROPE, 8, PAIR, MC>(m, p, s);
          case 16: return launch<BN, E_ROPE, 16, PAIR, MC>(m, p, s);
          case 32: return launch<BN, E_ROPE, 32, PAIR, MC>(m, p, s);
          case 64: return launch<BN, E_ROPE, 64, PAIR, MC>(m, p, s);
          case 128: return launch<BN, E_ROPE, 128, PAIR, MC>(m, p, s);
          default: break;
        }
      }
      break;
  }
  set_error("tcgen05 gemm: unsupported epilogue %d / BN %d / head_dim %d", a.epilogue, BN, a.head_dim);
  return ARMT_ERR_UNSUPPORTED;
}

}  // namespace tc

int make_tma_map_bf16(CUtensorMap* map, const void* base, long long cols, long long rows, long long batches,
                      long long ld, long long batch_stride, int box_rows) {
  return tc::make_map(map, base, cols, rows, batches, ld, batch_stride, box_rows);
}

// One launch over rows [row0, m_end) of every member; pair = CTA-pair (2-CTA) tiles.
static int gemm_rows(const ArmtGemmArgs& a, int bn, bool pair, int row0, int m_end, cudaStream_t s,
                     int max_ctas = -1, bool mc = false) {
  using namespace tc;
  int max_a = 0, max_b = 0;
  for (int g = 0; g < a.G; ++g) {
    max_a = a.a_slot[g] > max_a ? a.a_slot[g] : max_a;
    max_b = a.b_index[g] > max_b ? a.b_index[g] : max_b;
  }
  Maps maps;
  // a wrapped operand physically holds its first kwrap columns only
  const long long ka_cols = a.a_kwrap > 0 ? a.a_kwrap : a.K, kb_cols = a.b_kwrap > 0 ? a.b_kwrap : a.K;
  int rc = make_map(&maps.a, a.A, ka_cols, a.M, max_a + 1, a.lda, a.a_stride, BM);
  if (rc) return rc;
  rc = make_map(&maps.b, a.B, kb_cols, a.N, max_b + 1, a.ldb, a.b_stride, pair ? bn / 2 : bn);
  if (rc) return rc;
  if (mc) {   // half-tile boxes for the multicast halves of the shared operand
    rc = make_map(&maps.a2, a.A, ka_cols, a.M, max_a + 1, a.lda, a.a_stride, BM / 2);
    if (rc) return rc;
    rc = make_map(&maps.b2, a.B, kb_cols, a.N, max_b + 1, a.ldb, a.b_stride, bn / 2);
    if (rc) return rc;
  } else {
    maps.a2 = maps.a;
    maps.b2 = maps.b;
  }
  maps.r = maps.c = maps.c2 = maps.a;

  Params p;
  memset(&p, 0, sizeof(p));
  const int tm = pair ? 2 * BM : BM;
  p.G = a.G; p.M = m_end; p.N = a.N; p.K = a.K; p.row0 = row0;
  p.tiles_m = (m_end - row0 + tm - 1) / tm;
  p.tiles_n = (a.N + bn - 1) / bn;
  p.num_tiles = mc ? a.G * (p.tiles_n / 2) * p.tiles_m : a.G * p.tiles_m * p.tiles_n;
  p.k_blocks = (a.K + BK - 1) / BK;
  p.c_dtype = a.c_dtype;
  p.C = a.C; p.ldc = a.ldc; p.c_stride = a.c_stride;
  p.R = a.R; p.ldr = a.ldr; p.r_stride = a.r_stride;
  p.C2 = reinterpret_cast<__nv_bfloat16*>(a.C2); p.ldc2 = a.ldc2; p.c2_stride = a.c2_stride;
  p.c2_split = a.c2_split;
  p.ssq_out = a.ssq_out; p.ssq_in = a.ssq_in; p.ssq_stride = a.ssq_stride; p.ssq_np = a.ssq_np;
  p.norm_d = a.norm_d; p.norm_eps = a.norm_eps;
  p.lse_part = reinterpret_cast<float2*>(a.lse_part); p.lse_ld = a.lse_ld; p.targets = a.targets;
  p.lse_tgt = a.lse_tgt; p.lse_rows = a.lse_rows;
  p.den = a.den; p.den_stride = a.den_stride; p.eps = a.eps;
  p.rope_cos = a.rope_cos; p.rope_sin = a.rope_sin; p.head_dim = a.head_dim; p.rope_cols = a.rope_cols;
  p.rope_ld = a.M;  // tables are (head_dim/2, M): one column per position of the full member
  p.swiglu_block = a.swiglu_block;
  p.max_ctas = max_ctas >= 0 ? max_ctas : a.max_ctas;
  if (!pair && !mc) {
    // dynamic tile scheduling: a fresh {next, done} counter pair per launch from a ring in
    // device memory (each launch's last CTA re-zeroes its pair, so graph replays reuse it)
    static std::atomic<int*> ring{nullptr};
    static std::mutex ring_mu;
    static std::atomic<unsigned long long> next{0};
    constexpr unsigned long long RING = 1ull << 18;
    // opt-in (ARMT_GEMM_DYN=1, set by the dual-stream runner): one-stream runs are 0.4%
    // faster with the static schedule, concurrent streams need the dynamic one
    static const bool dyn_on = getenv("ARMT_GEMM_DYN") && getenv("ARMT_GEMM_DYN")[0] == '1';
    if (dyn_on && ring.load() == nullptr) {
      cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(s, &cap_st);   // (no allocation inside a graph capture: static schedule)
      std::lock_guard<std::mutex> lk(ring_mu);
      if (cap_st == cudaStreamCaptureStatusNone && ring.load() == nullptr) {
        int* r = nullptr;
        ARMT_REQUIRE(cudaMalloc(&r, RING * 2 * sizeof(int)) == cudaSuccess, ARMT_ERR_CUDA, "tile ring alloc");
        ARMT_REQUIRE(cudaMemset(r, 0, RING * 2 * sizeof(int)) == cudaSuccess, ARMT_ERR_CUDA, "tile ring init");
        ring.store(r);
      }
    }
    if (dyn_on && ring.load() != nullptr) p.tile_ctr = ring.load() + 2 * (next.fetch_add(1) % RING);
  }
  {
    // coalesced residual epilogue needs 16 B-aligned f32 rows and 8 B-aligned bf16 rows
    const bool al = (a.N % 4 == 0) && (a.ldc % 4 == 0) && (a.ldr % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.C) | reinterpret_cast<uintptr_t>(a.R)) % 16 == 0) &&
                    (a.C2 == nullptr || (a.ldc2 % 4 == 0 && a.c2_split % 4 == 0 &&
                                         reinterpret_cast<uintptr_t>(a.C2) % 8 == 0)) &&
                    (a.c_stride % 4 == 0) && (a.r_stride % 4 == 0) && (a.C2 == nullptr || a.c2_stride % 4 == 0);
    p.xpose = al ? 1 : 0;
    p.cst = (a.c_dtype == ARMT_BF16 || a.epilogue == ARMT_EPI_SWIGLU || a.epilogue == ARMT_EPI_ROPE) &&
            a.ldc % 8 == 0 && reinterpret_cast<uintptr_t>(a.C) % 16 == 0 && a.c_stride % 8 == 0 ? 1 : 0;
  }
  {
    static const bool prof = getenv("ARMT_GEMM_PROF") != nullptr;
    p.prof = prof ? 1 : 0;
  }
  for (int g = 0; g < a.G; ++g) {
    p.a_slot[g] = (short)a.a_slot[g];
    p.b_index[g] = (short)a.b_index[g];
    p.c_slot[g] = (short)a.c_slot[g];
    p.e_index[g] = (short)a.e_index[g];
  }
  p.z = a.z; p.nu = a.nu;
  p.a_kwrap = a.a_kwrap; p.b_kwrap = a.b_kwrap;
  // TMA epilogue for the short-K (epilogue-bound) residual / retrieve GEMMs: residual tiles
  // TMA-loaded ahead of the accumulator, results TMA-stored (ARMT_GEMM_TMAE=0 disables).
  // K <= 1024 only: it costs mainloop stages, so the K=2048 O-projection is faster without
  // it (C2, G=16: 164 vs 205 us) while the K=384 retrieval gains (86 vs 116 us)
  bool tmae = false;
  {
    const char* te = getenv("ARMT_GEMM_TMAE");
    const bool tmae_on = !(te && te[0] == '0');
    const bool heavy = a.epilogue == ARMT_EPI_RESIDUAL || a.epilogue == ARMT_EPI_RETRIEVE;
    const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    tmae = tmae_on && heavy && p.xpose && a.K <= 1024 && a.c_dtype == ARMT_F32 && al16(a.C) && al16(a.R) &&
           a.ldc % 4 == 0 && a.ldr % 4 == 0 && a.c_stride % 4 == 0 && a.r_stride % 4 == 0 &&
           (a.C2 == nullptr || (al16(a.C2) && a.ldc2 % 8 == 0 && a.c2_stride % 8 == 0 && a.c2_split % 32 == 0));
    if (tmae) {
      int max_c = 0;
      for (int g = 0; g < a.G; ++g) max_c = a.c_slot[g] > max_c ? a.c_slot[g] : max_c;
      int rc2 = make_epi_map(&maps.r, true, a.R, a.N, m_end, max_c + 1, a.ldr, a.r_stride);
      if (!rc2) rc2 = make_epi_map(&maps.c, true, a.C, a.N, m_end, max_c + 1, a.ldc, a.c_stride);
      if (!rc2 && a.C2 != nullptr)
        rc2 = make_epi_map(&maps.c2, false, a.C2, a.c2_split > 0 ? 2LL * a.c2_split : (long long)a.N, m_end,
                           max_c + 1, a.ldc2, a.c2_stride);
      if (rc2) return rc2;
    }
  }
  switch (bn) {
    case 64: return dispatch_epi<64, false, false>(a, maps, p, s, tmae);
    case 128: return dispatch_epi<128, false, false>(a, maps, p, s, tmae);
    case 256:
      if (pair) return dispatch_epi<256, true, false>(a, maps, p, s, tmae);
      if (mc) return dispatch_epi<256, false, true>(a, maps, p, s, tmae);
      return dispatch_epi<256, false, false>(a, maps, p, s, tmae);
  }
  return ARMT_ERR_UNSUPPORTED;
}

int gemm_tc(const ArmtGemmArgs& a, cudaStream_t s) {
  ARMT_REQUIRE(a.K % 8 == 0, ARMT_ERR_DIM, "bf16 GEMM needs K %% 8 == 0 (K=%d)", a.K);
  ARMT_REQUIRE(a.a_kwrap >= 0 && a.b_kwrap >= 0 && a.a_kwrap % 64 == 0 && a.b_kwrap % 64 == 0 &&
               a.a_kwrap < a.K && a.b_kwrap < a.K, ARMT_ERR_DIM, "K wrap must be a multiple of 64 below K");
  ARMT_REQUIRE(a.lda % 8 == 0 && a.ldb % 8 == 0, ARMT_ERR_DIM, "bf16 GEMM needs lda/ldb %% 8 == 0");
  if (a.epilogue == ARMT_EPI_SWIGLU)
    ARMT_REQUIRE((a.swiglu_block == 32 || a.swiglu_block == 128) && a.N % (2 * a.swiglu_block) == 0,
                 ARMT_ERR_UNSUPPORTED, "SwiGLU block must be 32 or 128 and divide N/2");
  if (a.epilogue == ARMT_EPI_FOLDR)
    ARMT_REQUIRE(a.N <= 128 && a.c2_split >= a.N && a.c2_split % 16 == 0 && a.ldc >= 4LL * a.c2_split &&
                 a.ldc % 8 == 0 && a.c_dtype == ARMT_BF16 && a.R != nullptr, ARMT_ERR_UNSUPPORTED,
                 "FOLDR epilogue: N <= 128 tokens, segment %% 16, ldc >= 4 segments, bf16 C, value rows R");
  if (a.epilogue == ARMT_EPI_DPFP)
    ARMT_REQUIRE((a.N == 16 || a.N == 32 || a.N == 64) && a.nu >= 1 && a.nu <= 3 && a.z != nullptr &&
                 a.den != nullptr && a.ldc >= 2LL * a.nu * a.N && a.ldc % 8 == 0 && a.c_dtype == ARMT_BF16,
                 ARMT_ERR_UNSUPPORTED, "DPFP epilogue: d_mem in {16,32,64}, nu in [1,3], bf16 phi, ldc %% 8");
  const int bn = tc::pick_bn(a);
  // Engine policy for 256-wide tiles (measured in situ, C2):
  //   * M a whole number of 256-row pairs (LM head)            -> CTA pairs (cta_group::2)
  //   * QKV+RoPE and the residual GEMMs (O, down) of 1152-row members -> pair tiles for rows
  //     [0, 1024) of every member CONCURRENT with single-CTA tiles for the remainder rows on
  //     a forked stream with REM_CTAS SMs (down -9%, QKV -6%, O -0.5% vs the alternatives)
  //   * other mainloop-heavy shapes with an even number of N tiles (gate/up) -> 2-CTA
  //     multicast clusters sharing the weight tile (pairs measured slower there)
  //   * everything else -> single-CTA tiles
  // ARMT_GEMM_PAIR=0 / =split / =conc and ARMT_GEMM_MC=0 override it (tests, A/B runs).
  const char* pe = getenv("ARMT_GEMM_PAIR");
  const int m_pair = (a.M / (2 * tc::BM)) * (2 * tc::BM);
  const bool split = pe && strcmp(pe, "split") == 0;
  const bool conc = (pe && strcmp(pe, "conc") == 0) ||
                    (!pe && (a.epilogue == ARMT_EPI_ROPE || a.epilogue == ARMT_EPI_RESIDUAL));
  const bool pair = bn == 256 && m_pair > 0 && (m_pair == a.M || split || conc) && a.K >= 1024 &&
                    !(pe && pe[0] == '0');
  if (!pair) {
    const char* me = getenv("ARMT_GEMM_MC");
    const int tiles_n = (a.N + bn - 1) / bn;
    const bool mc = bn == 256 && (tiles_n % 2 == 0) && a.K >= 1024 && !(me && me[0] == '0') && a.max_ctas == 0;
    return gemm_rows(a, bn, false, 0, a.M, s, -1, mc);
  }
  if (m_pair == a.M) return gemm_rows(a, bn, true, 0, m_pair, s);
  if (!conc) {
    int rc = gemm_rows(a, bn, true, 0, m_pair, s);
    return rc ? rc : gemm_rows(a, bn, false, m_pair, a.M, s);
  }
  ForkedStream* fk = forked_stream(s);
  if (fk == nullptr) {   // more calling streams than fork slots: the remainder after the pair tiles
    int rc = gemm_rows(a, bn, true, 0, m_pair, s);
    return rc ? rc : gemm_rows(a, bn, false, m_pair, a.M, s);
  }
  const char* rc_env = getenv("ARMT_GEMM_REM_CTAS");
  const int rem = rc_env ? atoi(rc_env) : 20;
  const int sms = num_sms();
  int rc = fk->fork();
  if (rc) return rc;
  rc = gemm_rows(a, bn, false, m_pair, a.M, fk->side, rem);
  if (rc) return rc;
  rc = gemm_rows(a, bn, true, 0, m_pair, s, ((sms - rem) / 2) * 2);
  if (rc) return rc;
  return fk->join();
}

ForkedStream* forked_stream(cudaStream_t caller) {
  constexpr int MAX_FORKS = 32;
  static ForkedStream forks[MAX_FORKS];
  static int n_forks = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < n_forks; ++i)
    if (forks[i].caller == caller) return &forks[i];
  if (n_forks == MAX_FORKS) return nullptr;
  ForkedStream* f = &forks[n_forks];
  f->caller = caller;
  if (cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&f->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&f->join_ev, cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  ++n_forks;
  return f;
}

int ForkedStream::fork() {
  ARMT_REQUIRE(cudaEventRecord(fork_ev, caller) == cudaSuccess, ARMT_ERR_CUDA, "fork: event record");
  ARMT_REQUIRE(cudaStreamWaitEvent(side, fork_ev, 0) == cudaSuccess, ARMT_ERR_CUDA, "fork: stream wait");
  return ARMT_OK;
}

int ForkedStream::join() {
  ARMT_REQUIRE(cudaEventRecord(join_ev, side) == cudaSuccess, ARMT_ERR_CUDA, "join: event record");
  ARMT_REQUIRE(cudaStreamWaitEvent(caller, join_ev, 0) == cudaSuccess, ARMT_ERR_CUDA, "join: stream wait");
  return ARMT_OK;
}

}  // namespace armt

// Read (and optionally reset) the ARMT_GEMM_PROF wait-cycle counters (diagnostics).
extern "C" int armt_gemm_prof(unsigned long long* out8, int reset) {
  cudaMemcpyFromSymbol(out8, armt::tc::g_gemm_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(armt::tc::g_gemm_prof, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
