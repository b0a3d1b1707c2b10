// tcgen05 causal segment attention (bf16, d_head in {64, 128}).
//
// Reference: armt/layers.py:211-223 (scores = q k^T / sqrt(dh) + causal mask
// over all T rows, max-subtracted softmax, ctx = P v, heads merged).
//
// Persistent CTAs (2 per SM for d_head 64) walk 128-query tiles of every
// (member, head), heaviest first; KV tiles of 128 keys.
//   warp 0      TMA: Q once, then K_j / V_j into a 2-stage ring (128B swizzle,
//               read in place from the (T, 3d) QKV rows of the member)
//   warp 1      MMA (one thread): S_j = Q K_j^T -> TMEM S[j%2] (M=128, N=128);
//               O_j = P_j V_j -> TMEM O[j%2] (M=128, N=dh, V as MN-major B)
//   warp 2      TMEM allocator (512 columns: S0, S1, O0, O1)
//   warps 4-7   softmax, thread = query row = TMEM lane: two tcgen05.ld passes
//               over S_j (row max, then exp2 / row sum / bf16 pack), P_j written
//               to smem in the UMMA K-major SW128 layout; O_j folded into a
//               register accumulator with the running max rescale
//               (O = O * exp(m_prev - m) + O_j), so TMEM never needs a
//               read-modify-write.
// S_{j+1} is issued before PV_j, so the softmax of tile j+1 overlaps PV_j.

#include "tc_ptx.cuh"

namespace armt {

int make_tma_map_bf16(CUtensorMap* map, const void* base, long long cols, long long rows, long long batches,
                      long long ld, long long batch_stride, int box_rows);

namespace attn_tc {

using namespace tcx;

constexpr int BQ = 128, BKV = 128, NTHREADS = 256;

__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2, flushes denormals; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DH> struct Cfg {
  static constexpr int KB = DH / 64;                    // 64-column sub-tiles per Q/K/V tile
  static constexpr int TILE = 128 * 64 * 2;             // one 128 x 64 bf16 sub-tile (16 KB)
  static constexpr int Q_BYTES = KB * TILE;
  static constexpr int KV_BYTES = 2 * KB * TILE;        // K + V of one stage
  static constexpr int P_BYTES = 2 * TILE;              // 128 queries x 128 keys
  static constexpr int NP = 1;                          // P buffers
  static constexpr int NS = 1;                          // S buffers in TMEM
  static constexpr int O_COL = NS * 128;                // O[0], O[1] follow S
  static constexpr int TMEM_COLS = (O_COL + 2 * DH) <= 256 ? 256 : 512;  // d_head 64: 2 CTAs per SM
  // no alignment slack: dynamic smem starts 1 KB-aligned (after the 1 KB system area),
  // which keeps d_head 64 at 2 CTAs per SM (2 x 113 KB)
  static constexpr int SMEM = Q_BYTES + 2 * KV_BYTES + NP * P_BYTES + 256;
};

struct Params {
  __nv_bfloat16* ctx;
  long long ld_ctx, ctx_stride;
  int T, H, G, d, nq;
  float scale_log2;
};

template <int DH>
__global__ void __launch_bounds__(NTHREADS, DH == 64 ? 2 : 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ Params p) {
  using C = Cfg<DH>;
  constexpr int KB = C::KB, NP = C::NP, NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();  // SW128 operand tiles need 1 KB alignment
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::Q_BYTES;                      // stage s: K at s*KV_BYTES, V at +KB*TILE
  uint8_t* sP = sKV + 2 * C::KV_BYTES;                 // buffer b: 2 sub-tiles (keys 0-63, 64-127)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + NP * C::P_BYTES);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;    // [2]
  uint64_t* kv_empty = bar + 3;   // [2]
  uint64_t* s_full = bar + 5;     // [2]
  uint64_t* s_empty = bar + 7;    // [2]
  uint64_t* p_full = bar + 9;     // [2]
  uint64_t* p_empty = bar + 11;   // [2]
  uint64_t* o_full = bar + 13;    // [2]
  uint64_t* o_empty = bar + 15;   // [2]
  uint64_t* q_empty = bar + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HG = p.H * p.G;
  const int n_items = p.nq * HG;
  const int n_kvmax = (p.T + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4); mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1); mbar_init(&o_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(C::TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Persistent over work items (q-tile, head, member), heaviest q-tiles first.
  // Every role walks the same item sequence; pipeline phases derive from the
  // running KV-tile counter tt (and the item counter it for the Q buffer).
  auto item = [&](int w, int& qt, int& h, int& g) {
    qt = p.nq - 1 - w / HG;
    const int rem = w - (w / HG) * HG;
    h = rem % p.H;
    g = rem / p.H;
  };

  if (warp == 0) {
    if (lane == 0) {
      int tt = 0, it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        int qt, h, g;
        item(w, qt, h, g);
        const int nkv = min(qt + 1, n_kvmax);
        const int colQ = h * DH, colK = p.d + h * DH, colV = 2 * p.d + h * DH;
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_expect_tx(q_full, C::Q_BYTES);
        for (int kb = 0; kb < KB; ++kb) tma_load_3d(sQ + kb * C::TILE, &tm, q_full, colQ + 64 * kb, qt * BQ, g);
        for (int j = 0; j < nkv; ++j) {
          const int u = tt + j, st = u & 1;
          mbar_wait(&kv_empty[st], ((u >> 1) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], C::KV_BYTES);
          uint8_t* base = sKV + st * C::KV_BYTES;
          for (int kb = 0; kb < KB; ++kb) {
            tma_load_3d(base + kb * C::TILE, &tm, &kv_full[st], colK + 64 * kb, j * BKV, g);
            tma_load_3d(base + (KB + kb) * C::TILE, &tm, &kv_full[st], colV + 64 * kb, j * BKV, g);
          }
        }
        tt += nkv;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = instr_desc<128, 128, 0>();
      constexpr uint32_t idO = instr_desc<128, DH, 1>();
      auto issue_pv = [&](int u) {
        const int st = u & 1, pb = u % NP;
        mbar_wait(&p_full[pb], (u / NP) & 1);
        mbar_wait(&o_empty[st], ((u >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t pbase = smem_u32(sP + pb * C::P_BYTES);
        const uint32_t vbase = smem_u32(sKV + st * C::KV_BYTES + KB * C::TILE);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          // A = P (K-major SW128, 64-key sub-tiles); B = V (MN-major SW128:
          // SBO = 1024 B per 8 keys, LBO = 16 KB per 64 dh columns, +2048 B per 16 keys)
          const uint64_t a = smem_desc_sw128(pbase + (k >> 2) * C::TILE) + 2 * (k & 3);
          const uint64_t b = (smem_desc_sw128(vbase) | ((uint64_t)(C::TILE >> 4) << 16)) + (uint64_t)((2048 * k) >> 4);
          mma_bf16(tmem + C::O_COL + st * DH, a, b, idO, k > 0);
        }
        mma_commit(&o_full[st]);
        mma_commit(&kv_empty[st]);
        mma_commit(&p_empty[pb]);
      };
      int tt = 0, it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        int qt, h, g;
        item(w, qt, h, g);
        const int nkv = min(qt + 1, n_kvmax);
        mbar_wait(q_full, it & 1);
        for (int j = 0; j < nkv; ++j) {
          const int u = tt + j, st = u & 1, sb = u % NS;
          mbar_wait(&kv_full[st], (u >> 1) & 1);
          mbar_wait(&s_empty[sb], ((u / NS) & 1) ^ 1);
          tc_fence_after();
          const uint32_t qbase = smem_u32(sQ);
          const uint32_t kbase = smem_u32(sKV + st * C::KV_BYTES);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            mma_bf16(tmem + sb * 128, smem_desc_sw128(qbase + (k >> 2) * C::TILE) + 2 * (k & 3),
                     smem_desc_sw128(kbase + (k >> 2) * C::TILE) + 2 * (k & 3), idS, k > 0);
          mma_commit(&s_full[sb]);
          if (j > 0) issue_pv(u - 1);
        }
        mma_commit(q_empty);  // every S MMA of this item has read Q
        issue_pv(tt + nkv - 1);
        tt += nkv;
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax: thread = query row r (TMEM lane)
    const int ew = warp & 3;
    const int r = ew * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(ew * 32) << 16);
    const float sl2 = p.scale_log2;
    int tt = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      int qt, h, g;
      item(w, qt, h, g);
      const int nkv = min(qt + 1, n_kvmax);
      const int q0 = qt * BQ;
      const int qrow = q0 + r;
      float o[DH];
#pragma unroll
      for (int c = 0; c < DH; ++c) o[c] = 0.f;
      float m = -INFINITY, l = 0.f, corr_prev = 1.f;
      auto fold_o = [&](int u, float corr) {
        const int st = u & 1;
        mbar_wait(&o_full[st], (u >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tl + C::O_COL + st * DH + c0, v);
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c0 + c] = fmaf(o[c0 + c], corr, v[c]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[st]);
      };
      for (int j = 0; j < nkv; ++j) {
        const int u = tt + j, sb = u % NS, pb = u % NP;
        const int k0 = j * BKV;
        // valid keys of this row in the tile: c <= lim (causal and key < T)
        const int lim = min(qrow, p.T - 1) - k0;
        mbar_wait(&s_full[sb], (u / NS) & 1);
        tc_fence_after();
        // pass 1: row max (tree per 32-column chunk: no 128-long serial FMNMX chain)
        const bool full = lim >= BKV - 1;  // warp-uniform for the tiles below the diagonal
        float mx = m;
#pragma unroll 1
        for (int c0 = 0; c0 < BKV; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tl + sb * 128 + c0, v);
          if (!full) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (c0 + c <= lim) ? v[c] : -INFINITY;
          }
#pragma unroll
          for (int w2 = 16; w2 > 0; w2 >>= 1)
#pragma unroll
            for (int c = 0; c < w2; ++c) v[c] = fmaxf(v[c], v[c + w2]);
          mx = fmaxf(mx, v[0]);
        }
        const float corr = ex2((m - mx) * sl2);  // m = -inf on the first tile -> 0
        m = mx;
        const float nm = -mx * sl2;
        if (u >= NP) mbar_wait(&p_empty[pb], ((u / NP) & 1) ^ 1);
        // pass 2: p = exp2(s*sl2 - m*sl2), row sum (tree), bf16 P row into the swizzled tile
        float rs = 0.f;
        uint8_t* prow = sP + pb * C::P_BYTES + r * 128;
#pragma unroll 1
        for (int c0 = 0; c0 < BKV; c0 += 32) {
          float v[32];
          __syncwarp();
          tmem_ld32(tl + sb * 128 + c0, v);
          if (!full) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = (c0 + c <= lim) ? v[c] : -INFINITY;
          }
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            v[c] = ex2(fmaf(v[c], sl2, nm));
            v[c + 1] = ex2(fmaf(v[c + 1], sl2, nm));
            pk[c >> 1] = pack_bf16x2(v[c], v[c + 1]);
          }
#pragma unroll
          for (int w2 = 16; w2 > 0; w2 >>= 1)
#pragma unroll
            for (int c = 0; c < w2; ++c) v[c] += v[c + w2];
          rs += v[0];
          // keys c0..c0+31 = 4 chunks of 8 in sub-tile (c0 / 64), chunk index (c0 % 64) / 8 + q
          uint8_t* sub = prow + (c0 >> 6) * C::TILE;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = ((c0 & 63) >> 3) + q;
            *reinterpret_cast<uint4*>(sub + ((chunk ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        l = l * corr + rs;
        fence_async_smem();  // make the generic-proxy P stores visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
        if (j > 0) fold_o(u - 1, corr_prev);
        corr_prev = corr;
      }
      fold_o(tt + nkv - 1, corr_prev);
      tt += nkv;
      if (qrow < p.T) {
        const float inv = 1.f / l;
        __nv_bfloat16* out = p.ctx + (long long)g * p.ctx_stride + (long long)qrow * p.ld_ctx + h * DH;
#pragma unroll
        for (int c = 0; c < DH; c += 8)
          *reinterpret_cast<uint4*>(out + c) =
              make_uint4(pack_bf16x2(o[c] * inv, o[c + 1] * inv), pack_bf16x2(o[c + 2] * inv, o[c + 3] * inv),
                         pack_bf16x2(o[c + 4] * inv, o[c + 5] * inv), pack_bf16x2(o[c + 6] * inv, o[c + 7] * inv));
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
}

template <int DH>
static int launch(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                  long long ctx_stride, int T, int H, float scale, cudaStream_t s) {
  CUtensorMap tm;
  int rc = make_tma_map_bf16(&tm, qkv, ld_qkv, T, G, ld_qkv, qkv_stride, 128);
  if (rc) return rc;
  Params p;
  p.ctx = reinterpret_cast<__nv_bfloat16*>(ctx);
  p.ld_ctx = ld_ctx; p.ctx_stride = ctx_stride;
  p.T = T; p.H = H; p.G = G; p.d = H * DH; p.nq = (T + BQ - 1) / BQ;
  p.scale_log2 = scale * 1.4426950408889634f;
  auto kern = attn_tc_kernel<DH>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<DH>::SMEM);
    attr = true;
  }
  const int items = p.nq * H * G;
  const int per_sm = DH == 64 ? 2 : 1;
  const int grid = items < per_sm * num_sms() ? items : per_sm * num_sms();
  kern<<<grid, NTHREADS, Cfg<DH>::SMEM, s>>>(tm, p);
  ARMT_CHECK_LAUNCH("attention tcgen05");
  return ARMT_OK;
}

}  // namespace attn_tc

int attention_tc(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                 long long ctx_stride, int T, int H, int dh, float scale, cudaStream_t s) {
  if (dh == 64) return attn_tc::launch<64>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, scale, s);
  if (dh == 128) return attn_tc::launch<128>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, scale, s);
  return ARMT_ERR_UNSUPPORTED;
}

}  // namespace armt
