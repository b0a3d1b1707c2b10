// Causal segment attention over T = segment + memory rows, per member and head.
//
// Reference: armt/layers.py:211-223 — scores = q k^T * (1/sqrt(dh)) + causal
// mask over ALL T rows (memory rows see every segment token; token rows never
// see memory rows), max-subtracted softmax, ctx = P v, heads merged back into
// (T, d). Here q/k/v are read in place from the (T, 3d) QKV rows (q, k already
// rotated) and ctx is written merged, so no head split/merge copies exist.
//
//  * bf16: flash-style online softmax on mma.sync m16n8k16 (fp32 accumulate),
//    64 query rows per CTA (16 per warp), 64-key K/V tiles double-buffered
//    with cp.async, heaviest (last) query blocks scheduled first.
//  * f32:  SIMT online softmax for the 1e-4 parity mode.

#include <stdlib.h>
#include "common.cuh"

namespace armt {
namespace attn {

// ============================================================== f32 (SIMT)
constexpr int FQ = 32;   // query rows per CTA (8 per warp)
constexpr int FK = 32;   // keys per tile

__global__ void __launch_bounds__(128) attn_f32_kernel(const float* __restrict__ qkv, long long ld_qkv,
                                                       long long qkv_stride, float* __restrict__ ctx, long long ld_ctx,
                                                       long long ctx_stride, int T, int H, int dh, float scale) {
  extern __shared__ float sm[];
  const int dhp = dh + 1;
  float* Qs = sm;                    // [FQ][dh]
  float* Ks = Qs + FQ * dh;          // [FK][dh+1]
  float* Vs = Ks + FK * dhp;         // [FK][dh]
  const int nqb = (T + FQ - 1) / FQ;
  const int qb = nqb - 1 - blockIdx.x;
  const int h = blockIdx.y, g = blockIdx.z;
  const int d = H * dh;
  const float* base = qkv + (long long)g * qkv_stride;
  const int q0 = qb * FQ;
  for (int e = threadIdx.x; e < FQ * dh; e += blockDim.x) {
    const int r = e / dh, c = e - r * dh;
    Qs[e] = q0 + r < T ? base[(long long)(q0 + r) * ld_qkv + h * dh + c] : 0.f;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RPW = FQ / 4;
  float m[RPW], l[RPW], acc[RPW][4];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    m[r] = -INFINITY; l[r] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[r][j] = 0.f;
  }
  const int q_last = min(T - 1, q0 + FQ - 1);
  const int n_kt = q_last / FK + 1;
  for (int kt = 0; kt < n_kt; ++kt) {
    __syncthreads();
    const int k0 = kt * FK;
    for (int e = threadIdx.x; e < FK * dh; e += blockDim.x) {
      const int r = e / dh, c = e - r * dh;
      const bool ok = k0 + r < T;
      const long long off = (long long)(k0 + r) * ld_qkv + h * dh + c;
      Ks[r * dhp + c] = ok ? base[off + d] : 0.f;
      Vs[r * dh + c] = ok ? base[off + 2 * d] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int lr = warp * RPW + r;
      const int qi = q0 + lr;
      if (qi >= T || k0 > qi) continue;
      const int kj = k0 + lane;
      float s = -INFINITY;
      if (kj <= qi && kj < T) {
        float dot = 0.f;
        for (int c = 0; c < dh; ++c) dot = fmaf(Qs[lr * dh + c], Ks[lane * dhp + c], dot);
        s = dot * scale;
      }
      const float mx = fmaxf(m[r], warp_max(s));
      const float p = s == -INFINITY ? 0.f : expf(s - mx);
      const float corr = m[r] == -INFINITY ? 0.f : expf(m[r] - mx);
      l[r] = l[r] * corr + warp_sum(p);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[r][j] *= corr;
      for (int jk = 0; jk < FK; ++jk) {
        const float pj = __shfl_sync(0xffffffffu, p, jk);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = lane + 32 * j;
          if (c < dh) acc[r][j] = fmaf(pj, Vs[jk * dh + c], acc[r][j]);
        }
      }
      m[r] = mx;
    }
  }
  float* out = ctx + (long long)g * ctx_stride;
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int qi = q0 + warp * RPW + r;
    if (qi >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = lane + 32 * j;
      if (c < dh) out[(long long)qi * ld_ctx + h * dh + c] = acc[r][j] / l[r];
    }
  }
}

// ============================================================== bf16 (mma.sync)
constexpr int BQ = 64, BKV = 64;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Load a 64-row x DH tile (row stride ld elements, column offset col0) into smem
// rows of DH+8 bf16; rows >= T and columns >= dh are zero-filled.
template <int DH>
__device__ __forceinline__ void load_tile(__nv_bfloat16* dst, const __nv_bfloat16* src, long long ld, int row0,
                                          int T, int dh) {
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  for (int e = threadIdx.x; e < 64 * CH; e += blockDim.x) {
    const int r = e / CH, c = (e - r * CH) * 8;
    const bool ok = (row0 + r < T) && (c < dh);
    const __nv_bfloat16* s = ok ? src + (long long)(row0 + r) * ld + c : src;
    cp_async16(dst + r * (DH + 8) + c, s, ok);
  }
}

template <int DH>
__global__ void __launch_bounds__(128) attn_bf16_kernel(const __nv_bfloat16* __restrict__ qkv, long long ld_qkv,
                                                        long long qkv_stride, __nv_bfloat16* __restrict__ ctx,
                                                        long long ld_ctx, long long ctx_stride, int T, int H, int dh,
                                                        float scale_log2) {
  constexpr int LD = DH + 8;
  extern __shared__ __align__(16) uint8_t smraw[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smraw);
  __nv_bfloat16* Ks = Qs + BQ * LD;        // [2][BKV][LD]
  __nv_bfloat16* Vs = Ks + 2 * BKV * LD;   // [2][BKV][LD]

  const int nqb = (T + BQ - 1) / BQ;
  const int qb = nqb - 1 - blockIdx.x;
  const int h = blockIdx.y, g = blockIdx.z;
  const int d = H * dh;
  const __nv_bfloat16* base = qkv + (long long)g * qkv_stride;
  const int q0 = qb * BQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;

  load_tile<DH>(Qs, base + h * dh, ld_qkv, q0, T, dh);
  load_tile<DH>(Ks, base + d + h * dh, ld_qkv, 0, T, dh);
  load_tile<DH>(Vs, base + 2 * d + h * dh, ld_qkv, 0, T, dh);
  cp_commit();

  const int q_last = min(T - 1, q0 + BQ - 1);
  const int n_kt = q_last / BKV + 1;

  uint32_t qf[DH / 16][4];
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int qr0 = q0 + warp * 16 + gid;  // rows owned: qr0 and qr0 + 8

  for (int kt = 0; kt < n_kt; ++kt) {
    cp_wait_all();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk)
        ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LD + kk * 16 + (lane >> 4) * 8);
    }
    if (kt + 1 < n_kt) {
      const int nb = (kt + 1) & 1;
      load_tile<DH>(Ks + nb * BKV * LD, base + d + h * dh, ld_qkv, (kt + 1) * BKV, T, dh);
      load_tile<DH>(Vs + nb * BKV * LD, base + 2 * d + h * dh, ld_qkv, (kt + 1) * BKV, T, dh);
    }
    cp_commit();
    const __nv_bfloat16* Kb = Ks + (kt & 1) * BKV * LD;
    const __nv_bfloat16* Vb = Vs + (kt & 1) * BKV * LD;

    // S = Q K^T (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t b[4];
        ldsm_x4(b, Kb + (nt * 8 + (lane & 7) + (lane >> 4) * 8) * LD + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(s[nt], qf[kk], b[0], b[1]);
        mma16816(s[nt + 1], qf[kk], b[2], b[3]);
      }
    }
    // online softmax: running max on raw scores; p = exp2(s*scale_log2 - m*scale_log2)
    // (one FFMA + EX2 per element; masked scores are -inf and exp2(-inf) = 0).
    const int k0 = kt * BKV;
    if ((k0 + BKV - 1 > q0 + warp * 16) || (k0 + BKV > T)) {  // diagonal / tail tile only
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = qr0 + (e >> 1) * 8;
          const int key = k0 + nt * 8 + 2 * tig + (e & 1);
          if (key > row || key >= T) s[nt][e] = -INFINITY;
        }
    }
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    // every processed tile holds at least one unmasked key per row, so mx is finite
    const float corr0 = exp2f((mrow[0] - mx[0]) * scale_log2);
    const float corr1 = exp2f((mrow[1] - mx[1]) * scale_log2);
    mrow[0] = mx[0];
    mrow[1] = mx[1];
    const float nm0 = -mx[0] * scale_log2, nm1 = -mx[1] * scale_log2;
    float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(fmaf(s[nt][0], scale_log2, nm0));
      s[nt][1] = exp2f(fmaf(s[nt][1], scale_log2, nm0));
      s[nt][2] = exp2f(fmaf(s[nt][2], scale_log2, nm1));
      s[nt][3] = exp2f(fmaf(s[nt][3], scale_log2, nm1));
      ls0 += s[nt][0] + s[nt][1];
      ls1 += s[nt][2] + s[nt][3];
    }
    lrow[0] = lrow[0] * corr0 + ls0;
    lrow[1] = lrow[1] * corr1 + ls1;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= corr0; o[i][1] *= corr0;
      o[i][2] *= corr1; o[i][3] *= corr1;
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4];
      a[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int nt = 0; nt < DH / 8; nt += 2) {
        uint32_t b[4];
        ldsm_x4_t(b, Vb + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD + nt * 8 + (lane >> 4) * 8);
        mma16816(o[nt], a, b[0], b[1]);
        mma16816(o[nt + 1], a, b[2], b[3]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  __nv_bfloat16* out = ctx + (long long)g * ctx_stride;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = qr0 + r * 8;
    if (row >= T) continue;
    const float inv = 1.f / lrow[r];
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) {
      const int c = nt * 8 + 2 * tig;
      if (c < dh)
        *reinterpret_cast<uint32_t*>(out + (long long)row * ld_ctx + h * dh + c) =
            pack_bf16x2(o[nt][2 * r] * inv, o[nt][2 * r + 1] * inv);
    }
  }
}

template <int DH>
static int launch_bf16(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                       long long ctx_stride, int T, int H, int dh, float scale, cudaStream_t s) {
  const size_t smem = sizeof(__nv_bfloat16) * (size_t)(BQ + 4 * BKV) * (DH + 8);
  auto kern = attn_bf16_kernel<DH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((T + BQ - 1) / BQ, H, G);
  kern<<<grid, 128, smem, s>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), ld_qkv, qkv_stride,
                               reinterpret_cast<__nv_bfloat16*>(ctx), ld_ctx, ctx_stride, T, H, dh,
                               scale * 1.4426950408889634f);
  ARMT_CHECK_LAUNCH("attention bf16");
  return ARMT_OK;
}

}  // namespace attn
}  // namespace armt

namespace armt {
int attention_pp(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                 long long ctx_stride, int T, int H, float scale, cudaStream_t s);
int attention_tc(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                 long long ctx_stride, int T, int H, int dh, float scale, cudaStream_t s);
int attention_pp128(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx, long long ld_ctx,
                    long long ctx_stride, int T, int H, float scale, cudaStream_t s);
}
using namespace armt;

extern "C" int armt_attention(int G, const void* qkv, long long ld_qkv, long long qkv_stride, void* ctx,
                              long long ld_ctx, long long ctx_stride, int dtype, int T, int H, int dh, float scale,
                              void* stream) {
  using namespace armt::attn;
  ARMT_REQUIRE(G >= 1 && T >= 1 && H >= 1 && dh >= 2, ARMT_ERR_DIM, "attention: bad sizes");
  ARMT_REQUIRE(qkv && ctx, ARMT_ERR_INPUT, "attention: null pointer");
  cudaStream_t s = as_stream(stream);
  if (dtype == ARMT_F32) {
    ARMT_REQUIRE(dh <= 128, ARMT_ERR_UNSUPPORTED, "attention f32: head dim %d > 128", dh);
    const size_t smem = sizeof(float) * ((size_t)FQ * dh + (size_t)FK * (dh + 1) + (size_t)FK * dh);
    cudaFuncSetAttribute(attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((T + FQ - 1) / FQ, H, G);
    attn_f32_kernel<<<grid, 128, smem, s>>>(reinterpret_cast<const float*>(qkv), ld_qkv, qkv_stride,
                                            reinterpret_cast<float*>(ctx), ld_ctx, ctx_stride, T, H, dh, scale);
    ARMT_CHECK_LAUNCH("attention f32");
    return ARMT_OK;
  }
  ARMT_REQUIRE(dh % 8 == 0 && ld_qkv % 8 == 0 && ld_ctx % 2 == 0, ARMT_ERR_DIM,
               "attention bf16: head dim and row strides must be multiples of 8");
  // tcgen05 kernels: ping-pong pairs for d_head 64 and 128
  // (ARMT_ATTN=mma forces the mma.sync kernel, ARMT_ATTN=tc the single-tile
  // tcgen05 kernel, for A/B runs)
  const char* force_env = getenv("ARMT_ATTN");   // read per call: tests switch kernels in one process
  const char force = force_env != nullptr ? force_env[0] : '\0';
  if (dh == 64 && force != 'm' && force != 't')
    return attention_pp(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, scale, s);
  if (dh == 128 && force != 'm' && force != 't')
    return attention_pp128(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, scale, s);
  if ((dh == 64 || dh == 128) && force != 'm')
    return attention_tc(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, dh, scale, s);
  if (dh <= 16) return launch_bf16<16>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, dh, scale, s);
  if (dh <= 32) return launch_bf16<32>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, dh, scale, s);
  if (dh <= 64) return launch_bf16<64>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, dh, scale, s);
  if (dh <= 128) return launch_bf16<128>(G, qkv, ld_qkv, qkv_stride, ctx, ld_ctx, ctx_stride, T, H, dh, scale, s);
  set_error("attention bf16: head dim %d > 128", dh);
  return ARMT_ERR_UNSUPPORTED;
}
