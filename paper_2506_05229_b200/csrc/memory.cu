// Associative-memory write path: the delta-rule fold of update_stack.
//
// Reference: armt/memory.py:94-125 (_delta_fold) driven by :155-180. For
// token i = 0..M-1 IN ORDER (token i sees tokens < i):
//   zq = z.phi_i ; nrm = phi_i.phi_i
//   vbar = |zq| <= eps ? 0 : (A phi_i) / zq ; gamma = nrm <= eps ? 0 : 1 - zq/nrm
//   A += beta_i (v_i - vbar) phi_i^T ; z += gamma phi_i
//
// The z chain never reads A, so it runs first (fold_prep, one CTA per member)
// and publishes zq_i and beta_i. Rows of A are then independent: fold_main
// gives each warp RPW rows of A held in REGISTERS (lane owns columns
// lane + 32j), keeps phi for all M tokens in shared memory, and per token does
// one warp-shuffle dot product and one axpy per row. A is read once and written
// once per fold (the bandwidth floor), fp32 throughout; the bf16 shadow of A
// used by the tensor-core retrieval is refreshed in the same pass.

#include "common.cuh"

namespace armt {
namespace fold {

constexpr int NJ_MAX = 16;  // d_phi <= 512

struct Ws {
  float* phi;   // [G][M][dphi]
  float* zq;    // [G][M]
  float* beta;  // [G][M]
};

__host__ __device__ inline Ws carve(void* ws, int G, int M, int dphi) {
  float* f = reinterpret_cast<float*>(ws);
  Ws w;
  w.phi = f;
  w.zq = f + (long long)G * M * dphi;
  w.beta = w.zq + (long long)G * M;
  return w;
}

__device__ __forceinline__ float relu_split(const float* k, int i, int d_mem) {
  return i < d_mem ? fmaxf(k[i], 0.f) : fmaxf(-k[i - d_mem], 0.f);
}

__global__ void __launch_bounds__(256) fold_prep_kernel(const __grid_constant__ ArmtMembers mem,
                                                        const float* __restrict__ kvb, long long ld_kvb,
                                                        long long kvb_stride, int k_off, int b_off,
                                                        float* __restrict__ z, int M, int d_mem, int nu, float eps,
                                                        Ws ws) {
  extern __shared__ float sphi[];
  const int g = blockIdx.x;
  const int dphi = 2 * nu * d_mem, two_m = 2 * d_mem;
  const float* kv = kvb + (long long)g * kvb_stride;
  float* gphi = ws.phi + (long long)g * M * dphi;
  // phase 1: phi_i = DPFP(k_i) for all tokens (armt/memory.py:173), beta = sigmoid (:172)
  for (int e = threadIdx.x; e < M * dphi; e += blockDim.x) {
    const int i = e / dphi, c = e - i * dphi;
    const int j = c / two_m + 1, ii = c - (j - 1) * two_m;
    const float* k = kv + (long long)i * ld_kvb + k_off;
    const float v = relu_split(k, ii, d_mem) * relu_split(k, (ii + j) % two_m, d_mem);
    sphi[e] = v;
    gphi[e] = v;
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x)
    ws.beta[(long long)g * M + i] = sigmoid_ref(kv[(long long)i * ld_kvb + b_off]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  // phase 2: the z chain (one warp; lane owns columns lane + 32j)
  const int lane = threadIdx.x;
  float* zl = z + (long long)mem.layer[g] * dphi;
  float zr[NJ_MAX];
#pragma unroll
  for (int j = 0; j < NJ_MAX; ++j) {
    const int c = lane + 32 * j;
    zr[j] = c < dphi ? zl[c] : 0.f;
  }
  for (int i = 0; i < M; ++i) {
    float p[NJ_MAX];
    float zq = 0.f, nrm = 0.f;
#pragma unroll
    for (int j = 0; j < NJ_MAX; ++j) {
      const int c = lane + 32 * j;
      p[j] = c < dphi ? sphi[i * dphi + c] : 0.f;
      zq = fmaf(zr[j], p[j], zq);
      nrm = fmaf(p[j], p[j], nrm);
    }
    zq = warp_sum(zq);
    nrm = warp_sum(nrm);
    const float gamma = nrm <= eps ? 0.f : 1.f - zq / nrm;
#pragma unroll
    for (int j = 0; j < NJ_MAX; ++j) zr[j] = fmaf(gamma, p[j], zr[j]);
    if (lane == 0) ws.zq[(long long)g * M + i] = zq;
  }
#pragma unroll
  for (int j = 0; j < NJ_MAX; ++j) {
    const int c = lane + 32 * j;
    if (c < dphi) zl[c] = zr[j];
  }
}

template <int RPW, int NJ>
__global__ void __launch_bounds__(256) fold_main_kernel(const __grid_constant__ ArmtMembers mem,
                                                        const float* __restrict__ kvb, long long ld_kvb,
                                                        long long kvb_stride, int v_off, float* __restrict__ A,
                                                        __nv_bfloat16* __restrict__ shadow, long long ld_shadow, int d,
                                                        int M, int dphi, float eps, Ws ws) {
  constexpr int R = 8 * RPW;  // rows per CTA
  extern __shared__ float sm[];
  float* sphi = sm;                       // [M][dphi]
  float* sv = sphi + M * dphi;            // [M][R]
  float* szq = sv + M * R;                // [M]
  float* sbeta = szq + M;                 // [M]
  const int g = blockIdx.y;
  const int row0 = blockIdx.x * R;
  const float* gphi = ws.phi + (long long)g * M * dphi;
  for (int e = threadIdx.x; e < M * dphi; e += blockDim.x) sphi[e] = gphi[e];
  const float* kv = kvb + (long long)g * kvb_stride;
  for (int e = threadIdx.x; e < M * R; e += blockDim.x) {
    const int i = e / R, rr = e - i * R;
    sv[e] = row0 + rr < d ? kv[(long long)i * ld_kvb + v_off + row0 + rr] : 0.f;
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    szq[i] = ws.zq[(long long)g * M + i];
    sbeta[i] = ws.beta[(long long)g * M + i];
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int layer = mem.layer[g];
  float* Al = A + (long long)layer * d * dphi;
  float a[RPW][NJ];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int row = row0 + warp * RPW + r;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
      a[r][j] = (row < d && c < dphi) ? Al[(long long)row * dphi + c] : 0.f;
    }
  }
  for (int i = 0; i < M; ++i) {
    float p[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
      p[j] = c < dphi ? sphi[i * dphi + c] : 0.f;
    }
    const float zq = szq[i], beta = sbeta[i];
    const bool guarded = fabsf(zq) <= eps;
    float dot[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < NJ; ++j) s = fmaf(a[r][j], p[j], s);
      dot[r] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < RPW; ++r) dot[r] += __shfl_xor_sync(0xffffffffu, dot[r], o);
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const float vbar = guarded ? 0.f : dot[r] / zq;
      const float coef = beta * (sv[i * R + warp * RPW + r] - vbar);
#pragma unroll
      for (int j = 0; j < NJ; ++j) a[r][j] = fmaf(coef, p[j], a[r][j]);
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int row = row0 + warp * RPW + r;
    if (row >= d) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
      if (c < dphi) {
        Al[(long long)row * dphi + c] = a[r][j];
        if (shadow) shadow[(long long)layer * d * ld_shadow + (long long)row * ld_shadow + c] = __float2bfloat16_rn(a[r][j]);
      }
    }
  }
}

template <int RPW, int NJ>
static int launch_main(const ArmtMembers& mem, const float* kvb, long long ld_kvb, long long kvb_stride, int v_off,
                       float* A, __nv_bfloat16* shadow, long long ld_shadow, int d, int M, int dphi, float eps, Ws ws,
                       cudaStream_t s) {
  constexpr int R = 8 * RPW;
  const size_t smem = sizeof(float) * ((size_t)M * dphi + (size_t)M * R + 2 * (size_t)M);
  ARMT_REQUIRE(smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold: M*d_phi too large for shared memory (%zu B)", smem);
  auto kern = fold_main_kernel<RPW, NJ>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((d + R - 1) / R, mem.G);
  kern<<<grid, 256, smem, s>>>(mem, kvb, ld_kvb, kvb_stride, v_off, A, shadow, ld_shadow, d, M, dphi, eps, ws);
  ARMT_CHECK_LAUNCH("fold_main");
  return ARMT_OK;
}

template <int RPW>
static int dispatch_nj(int nj, const ArmtMembers& mem, const float* kvb, long long ld_kvb, long long kvb_stride,
                       int v_off, float* A, __nv_bfloat16* shadow, long long ld_shadow, int d, int M, int dphi,
                       float eps, Ws ws, cudaStream_t s) {
#define ARMT_FOLD_NJ(N) \
  if (nj <= N) return launch_main<RPW, N>(mem, kvb, ld_kvb, kvb_stride, v_off, A, shadow, ld_shadow, d, M, dphi, eps, ws, s);
  ARMT_FOLD_NJ(1) ARMT_FOLD_NJ(2) ARMT_FOLD_NJ(3) ARMT_FOLD_NJ(4) ARMT_FOLD_NJ(6) ARMT_FOLD_NJ(8)
  ARMT_FOLD_NJ(12) ARMT_FOLD_NJ(16)
#undef ARMT_FOLD_NJ
  set_error("fold: d_phi=%d exceeds %d", dphi, 32 * NJ_MAX);
  return ARMT_ERR_UNSUPPORTED;
}

}  // namespace fold
}  // namespace armt

using namespace armt;

extern "C" long long armt_fold_workspace_bytes(int G, int n_mem, int d_phi) {
  return (long long)sizeof(float) * G * n_mem * (d_phi + 2);
}

extern "C" int armt_mem_fold(const ArmtMembers* mem, const float* kvb, long long ld_kvb, long long kvb_stride,
                             int v_off, int k_off, int b_off, float* A, float* z, void* A_shadow, long long ld_shadow,
                             int d, int n_mem, int d_mem, int nu, float eps, void* ws, void* stream) {
  using namespace armt::fold;
  ARMT_REQUIRE(mem && mem->G >= 1 && mem->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "fold: bad member count");
  ARMT_REQUIRE(kvb && A && z && ws, ARMT_ERR_INPUT, "fold: null pointer");
  ARMT_REQUIRE(nu >= 1 && d_mem >= 1 && d >= 1, ARMT_ERR_DIM, "fold: bad sizes");
  if (n_mem == 0) return ARMT_OK;
  for (int g = 0; g < mem->G; ++g)
    for (int h = g + 1; h < mem->G; ++h)
      ARMT_REQUIRE(mem->layer[g] != mem->layer[h], ARMT_ERR_INPUT,
                   "fold: duplicate layer %d in one group (two writers per memory slot)", mem->layer[g]);
  const int dphi = 2 * nu * d_mem;
  ARMT_REQUIRE(dphi <= 32 * NJ_MAX, ARMT_ERR_UNSUPPORTED, "fold: d_phi=%d > %d", dphi, 32 * NJ_MAX);
  cudaStream_t s = as_stream(stream);
  Ws w = carve(ws, mem->G, n_mem, dphi);
  const size_t prep_smem = sizeof(float) * (size_t)n_mem * dphi;
  ARMT_REQUIRE(prep_smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold: M*d_phi too large");
  cudaFuncSetAttribute(fold_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prep_smem);
  fold_prep_kernel<<<mem->G, 256, prep_smem, s>>>(*mem, kvb, ld_kvb, kvb_stride, k_off, b_off, z, n_mem, d_mem, nu,
                                                   eps, w);
  ARMT_CHECK_LAUNCH("fold_prep");
  const int nj = (dphi + 31) / 32;
  auto* sh = reinterpret_cast<__nv_bfloat16*>(A_shadow);
  // few members: more, smaller CTAs (latency); many members: 32 rows per CTA
  const long long ctas_rpw4 = (long long)mem->G * ((d + 31) / 32);
  if (ctas_rpw4 < 2LL * num_sms())
    return dispatch_nj<2>(nj, *mem, kvb, ld_kvb, kvb_stride, v_off, A, sh, ld_shadow, d, n_mem, dphi, eps, w, s);
  return dispatch_nj<4>(nj, *mem, kvb, ld_kvb, kvb_stride, v_off, A, sh, ld_shadow, d, n_mem, dphi, eps, w, s);
}
