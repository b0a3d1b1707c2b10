// Tensor-core delta-rule fold (bf16 path): the chunked form of _delta_fold.
//
// Reference semantics (armt/memory.py:94-125): for tokens i = 0..M-1 in order,
//   zq_i = z_i.phi_i ; u_i = beta_i (v_i - [|zq_i| > eps] A_i phi_i / zq_i)
//   A_{i+1} = A_i + u_i phi_i^T ; z_{i+1} = z_i + gamma_i phi_i.
// Since A_i phi_i = A_0 phi_i + sum_{j<i} u_j (phi_j.phi_i), the u_i solve a
// unit lower-triangular system:
//   (I + diag(c) tril(Phi Phi^T, -1)) U = diag(beta) V - diag(c) Phi A_0^T,
//   c_i = beta_i [|zq_i| > eps] / zq_i,       A_M = A_0 + U^T Phi.
// So the fold is two grouped tcgen05 GEMMs plus O(M^2 d) of triangular solve:
//   fold_phi   phi (fp32), c_i = z0.phi_i, |phi_i|^2, beta; bf16x3 split copies
//   GEMM1      [P | c' | K] = Phi_s . memop^T   (memop rows: A_0 split, z split, Phi' split)
//   fold_chain the scalar z/gamma chain on (c, K) -> zq, coef, L; z_M (fp32)
//   fold_solve U = L^{-1} R per 128-column slice (16-row blocked substitution)
//   GEMM3      A_M = A_0 + U^T Phi (RESIDUAL epilogue), memop rows refreshed in
//              the same epilogue as the [hi | lo | hi] split of A_M.
// bf16x3: a ~ a_hi + a_lo; [a_hi|a_hi|a_lo].[b_hi|b_lo|b_hi] = hi.hi + hi.lo + lo.hi
// (~2^-16 relative), accumulated in fp32 TMEM. The f32 parity mode keeps the
// SIMT fold (memory.cu).

#include <algorithm>
#include "common.cuh"

namespace armt {

int gemm_tc(const ArmtGemmArgs& a, cudaStream_t s);

namespace foldtc {

struct Geom {
  int G, M, Mp, d, dphi, P, NB, NP1;
};

__host__ __device__ inline Geom geom(int G, int M, int d, int dphi) {
  Geom g;
  g.G = G; g.M = M; g.d = d; g.dphi = dphi;
  g.Mp = (M + 15) / 16 * 16;
  g.P = (dphi + 7) / 8 * 8;
  g.NB = d + 8 + g.Mp;
  g.NP1 = (d + 8 + g.Mp + 3) / 4 * 4;
  return g;
}

struct Ws {
  float *phi32, *c, *nrm, *beta, *coef, *L, *Pf;
  __nv_bfloat16 *Phis, *PhiTs, *UTs;
};

__host__ __device__ inline long long align256(long long x) { return (x + 63) / 64 * 64; }  // in floats

__host__ __device__ inline Ws carve(void* base, const Geom& q, long long* total_bytes = nullptr) {
  float* f = reinterpret_cast<float*>(base);
  Ws w;
  long long o = 0;
  auto take = [&](long long n) { float* p = f + o; o += align256(n); return p; };
  w.phi32 = take((long long)q.G * q.M * q.dphi);
  w.c = take((long long)q.G * q.Mp);
  w.nrm = take((long long)q.G * q.Mp);
  w.beta = take((long long)q.G * q.Mp);
  w.coef = take((long long)q.G * q.Mp);
  w.L = take((long long)q.G * q.Mp * q.Mp);
  w.Pf = take((long long)q.G * q.M * q.NP1);
  // bf16 regions (counted in floats: 2 bf16 per float)
  w.Phis = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.M * 3 * q.P + 1) / 2));
  w.PhiTs = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.P * 3 * q.Mp + 1) / 2));
  w.UTs = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.d * 3 * q.Mp + 1) / 2));
  if (total_bytes) *total_bytes = o * 4;
  return w;
}

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// ---------------------------------------------------------------- phi
// grid (Mp/16, G): each CTA handles 16 tokens. phi is built in shared memory
// (fp32), then written out coalesced in every layout the fold needs.
constexpr int PT = 16;  // tokens per CTA
__global__ void __launch_bounds__(256) fold_phi_kernel(const __grid_constant__ ArmtMembers mem,
                                                       const float* __restrict__ kvb, long long ld_kvb,
                                                       long long kvb_stride, int k_off, int b_off,
                                                       const float* __restrict__ z, __nv_bfloat16* __restrict__ memop,
                                                       int d_mem, int nu, Geom q, Ws w) {
  extern __shared__ float sm[];
  const int two_m = 2 * d_mem, P = q.P, Mp = q.Mp;
  float* sr = sm;                    // [PT][2m]
  float* sp = sr + PT * two_m;       // [PT][P + 1]
  const int g = blockIdx.y, layer = mem.layer[g];
  const int i0 = blockIdx.x * PT;
  const float* kv = kvb + (long long)g * kvb_stride;
  for (int e = threadIdx.x; e < PT * d_mem; e += blockDim.x) {
    const int t = e / d_mem, c = e - t * d_mem;
    const float k = (i0 + t < q.M) ? kv[(long long)(i0 + t) * ld_kvb + k_off + c] : 0.f;
    sr[t * two_m + c] = fmaxf(k, 0.f);
    sr[t * two_m + d_mem + c] = fmaxf(-k, 0.f);
  }
  if (threadIdx.x < PT) {
    const int i = i0 + threadIdx.x;
    w.beta[(long long)g * Mp + i] = i < q.M ? sigmoid_ref(kv[(long long)i * ld_kvb + b_off]) : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < PT * P; e += blockDim.x) {
    const int t = e / P, c = e - t * P;
    float v = 0.f;
    if (c < q.dphi && i0 + t < q.M) {
      const int j = c / two_m + 1, ii = c - (j - 1) * two_m;
      v = sr[t * two_m + ii] * sr[t * two_m + (ii + j) % two_m];
    }
    sp[t * (P + 1) + c] = v;
  }
  __syncthreads();
  // row layouts (token-major): phi32, Phi_s [hi|hi|lo], memop Phi' rows [hi|lo|hi]
  __nv_bfloat16* mrow = memop + ((long long)layer * q.NB + q.d + 8) * 3 * P;
  for (int e = threadIdx.x; e < PT * P; e += blockDim.x) {
    const int t = e / P, c = e - t * P, i = i0 + t;
    if (i >= q.M) continue;
    const float v = sp[t * (P + 1) + c];
    if (c < q.dphi) w.phi32[((long long)g * q.M + i) * q.dphi + c] = v;
    __nv_bfloat16 hi, lo;
    split_bf16(v, hi, lo);
    __nv_bfloat16* a = w.Phis + ((long long)g * q.M + i) * 3 * P;
    a[c] = hi; a[P + c] = hi; a[2 * P + c] = lo;
    __nv_bfloat16* b = mrow + (long long)i * 3 * P;
    b[c] = hi; b[P + c] = lo; b[2 * P + c] = hi;
  }
  // feature-major layout Phi^T_s [hi|lo|hi] over tokens: PT consecutive tokens per row
  for (int e = threadIdx.x; e < P * PT; e += blockDim.x) {
    const int c = e / PT, t = e - c * PT;
    __nv_bfloat16 hi, lo;
    split_bf16(sp[t * (P + 1) + c], hi, lo);
    __nv_bfloat16* r = w.PhiTs + ((long long)g * P + c) * 3 * Mp + i0 + t;
    r[0] = hi; r[Mp] = lo; r[2 * Mp] = hi;
  }
  // c_i = z0.phi_i and |phi_i|^2 in fp32 (warp per token)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* zl = z + (long long)layer * q.dphi;
  for (int t = warp; t < PT; t += blockDim.x / 32) {
    float cz = 0.f, nn = 0.f;
    for (int c = lane; c < q.dphi; c += 32) {
      const float v = sp[t * (P + 1) + c];
      cz = fmaf(v, zl[c], cz);
      nn = fmaf(v, v, nn);
    }
    cz = warp_sum(cz);
    nn = warp_sum(nn);
    if (lane == 0) {
      w.c[(long long)g * Mp + i0 + t] = cz;
      w.nrm[(long long)g * Mp + i0 + t] = nn;
    }
  }
}

// ---------------------------------------------------------------- chain
// zq_i = c_i + sum_{j<i} gamma_j K_ij ; gamma_i = nrm_i <= eps ? 0 : 1 - zq_i / nrm_i
// (armt/memory.py:101-106,116-119 with z_i expanded over earlier tokens);
// then coef_i, L_ij = coef_i K_ij (j < i), and z_M = z_0 + sum_i gamma_i phi_i.
constexpr int QMAX = 8;  // M <= 256
template <int QM>   // register slots per lane for the token chain: ceil(M / 32) <= QM
__global__ void __launch_bounds__(512) fold_chain_kernel(const __grid_constant__ ArmtMembers mem, float* __restrict__ z,
                                                         __nv_bfloat16* __restrict__ memop, float eps, Geom q, Ws w) {
  extern __shared__ float sm[];
  const int Mp = q.Mp, M = q.M;
  float* sK = sm;                  // [Mp][Mp], K_ij (K is symmetric up to rounding; rows read by lanes)
  float* szq = sK + (Mp * Mp > 4 * q.dphi ? Mp * Mp : 4 * q.dphi);  // (sK region doubles as z partials)
  float* sgam = szq + Mp;          // [Mp]
  float* snrm = sgam + Mp;         // [Mp]
  const int g = blockIdx.x, layer = mem.layer[g];
  const float* Pf = w.Pf + (long long)g * M * q.NP1;
  for (int e0 = threadIdx.x; e0 < Mp * Mp; e0 += 16 * blockDim.x) {  // 16 loads in flight
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = e0 + u * blockDim.x, i = e / Mp, j = e - i * Mp;
      v[u] = (e < Mp * Mp && i < M && j < M) ? Pf[(long long)i * q.NP1 + q.d + 8 + j] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (e0 + u * blockDim.x < Mp * Mp) sK[e0 + u * blockDim.x] = v[u];
  }
  __syncthreads();
  const int rmax = (M + 31) / 32;
  const float* cg = w.c + (long long)g * Mp;
  for (int i = threadIdx.x; i < Mp; i += blockDim.x) snrm[i] = w.nrm[(long long)g * Mp + i];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    float e[QM];
#pragma unroll
    for (int r = 0; r < QM; ++r) {
      const int t = lane + 32 * r;
      e[r] = t < M ? cg[t] : 0.f;
    }
    // blocks of 4 tokens: every lane redundantly runs the 4-step scalar chain
    // (4 shuffles in parallel, K entries as smem broadcasts), then all owned
    // tokens absorb the block's 4 gammas at once.
    for (int i0 = 0; i0 < M; i0 += 4) {
      const int qi = i0 >> 5, l0 = i0 & 31;
      float mine = 0.f;
#pragma unroll
      for (int r = 0; r < QM; ++r)
        if (r == qi) mine = e[r];
      float zq[4], gam[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) zq[u] = __shfl_sync(0xffffffffu, mine, l0 + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
#pragma unroll
        for (int v = 0; v < u; ++v) zq[u] = fmaf(gam[v], sK[(i0 + v) * Mp + i], zq[u]);
        const float nrm = i < M ? snrm[i] : 0.f;
        gam[u] = (i < M && nrm > eps) ? 1.f - __fdividef(zq[u], nrm) : 0.f;
      }
      if (lane < 4 && i0 + lane < M) {
        szq[i0 + lane] = lane == 0 ? zq[0] : lane == 1 ? zq[1] : lane == 2 ? zq[2] : zq[3];
        sgam[i0 + lane] = lane == 0 ? gam[0] : lane == 1 ? gam[1] : lane == 2 ? gam[2] : gam[3];
      }
#pragma unroll
      for (int r = 0; r < QM; ++r) {
        if (r < rmax) {
          const int t = lane + 32 * r;
          if (t >= i0 + 4 && t < M) {
            float acc = e[r];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = fmaf(gam[u], sK[(i0 + u) * Mp + t], acc);
            e[r] = acc;
          }
        }
      }
    }
  }
  __syncthreads();
  float* coef = w.coef + (long long)g * Mp;
  const float* beta = w.beta + (long long)g * Mp;
  for (int i = threadIdx.x; i < Mp; i += blockDim.x) {
    float cf = 0.f;
    if (i < M) {
      const float zq = szq[i];
      cf = fabsf(zq) <= eps ? 0.f : beta[i] / zq;
    }
    coef[i] = cf;
    szq[i] = cf;  // reuse as coef
  }
  __syncthreads();
  float* LT = w.L + (long long)g * Mp * Mp;  // LT[j][i] = L_ij = coef_i K_ij (j < i)
  for (int e = threadIdx.x; e < Mp * Mp; e += blockDim.x) {
    const int j = e / Mp, i = e - j * Mp;
    LT[e] = j < i ? szq[i] * sK[j * Mp + i] : 0.f;
  }
  // z_M = z_0 + sum_i gamma_i phi_i (fp32), plus its split row in memop
  float* zl = z + (long long)layer * q.dphi;
  __nv_bfloat16* zrow = memop + ((long long)layer * q.NB + q.d) * 3 * q.P;
  const float* ph = w.phi32 + (long long)g * M * q.dphi;
  for (int c = threadIdx.x; c < q.dphi; c += blockDim.x) {
    float acc = zl[c];
    for (int i0 = 0; i0 < M; i0 += 16) {  // 16 independent loads in flight per thread
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = i0 + u < M ? ph[(long long)(i0 + u) * q.dphi + c] : 0.f;
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = fmaf(i0 + u < M ? sgam[i0 + u] : 0.f, v[u], acc);
    }
    zl[c] = acc;
    __nv_bfloat16 hi, lo;
    split_bf16(acc, hi, lo);
    zrow[c] = hi; zrow[q.P + c] = lo; zrow[2 * q.P + c] = hi;
  }
}

// ---------------------------------------------------------------- solve
// U = L^{-1} R, R_i = beta_i v_i - coef_i P_i, per 128-column slice; 16-row
// blocks: off-diagonal update from finished rows (L row block read as float4
// broadcasts), then in-block forward substitution in registers. Output U^T as
// the [hi | hi | lo] bf16x3 A operand of GEMM3.
// One column per thread, 256 threads: 8 warps per SM hide the shared-memory
// latency of the substitution (the 2-columns-per-thread, 4-warp form was 73 us at C2).
constexpr int SOLVE_COLS = 256;
__global__ void __launch_bounds__(256) fold_solve_kernel(const float* __restrict__ kvb, long long ld_kvb,
                                                         long long kvb_stride, int v_off, Geom q, Ws w) {
  extern __shared__ __align__(16) float sm[];
  const int Mp = q.Mp, M = q.M;
  constexpr int US = SOLVE_COLS + 1;  // padded row: conflict-free column and row walks
  float* LT = sm;                     // [Mp][Mp]: LT[j][i] = L_ij
  float* us = LT + Mp * Mp;           // [Mp][US]
  const int g = blockIdx.y;
  const int n0 = blockIdx.x * SOLVE_COLS;
  const int c0 = threadIdx.x;
  const bool live0 = n0 + c0 < q.d;
  const float4* Lg = reinterpret_cast<const float4*>(w.L + (long long)g * Mp * Mp);  // already LT layout
  for (int e = threadIdx.x; e < Mp * Mp / 4; e += blockDim.x) reinterpret_cast<float4*>(LT)[e] = Lg[e];
  const float* beta = w.beta + (long long)g * Mp;
  const float* coef = w.coef + (long long)g * Mp;
  const float* Pf = w.Pf + (long long)g * M * q.NP1;
  const float* kv = kvb + (long long)g * kvb_stride;
  for (int i0 = 0; i0 < Mp; i0 += 16) {  // 32 independent loads in flight per thread
    float v0[16], p0[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int i = i0 + t;
      const bool ok = i < M && live0;
      v0[t] = ok ? kv[(long long)i * ld_kvb + v_off + n0 + c0] : 0.f;
      p0[t] = ok ? Pf[(long long)i * q.NP1 + n0 + c0] : 0.f;
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) us[(i0 + t) * US + c0] = beta[i0 + t] * v0[t] - coef[i0 + t] * p0[t];
  }
  __syncthreads();
  for (int b = 0; b < Mp; b += 16) {
    float x[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) x[t] = us[(b + t) * US + c0];
    for (int j = 0; j < b; ++j) {
      const float u0 = us[j * US + c0];
      const float4* lrow = reinterpret_cast<const float4*>(LT + j * Mp + b);
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        const float4 l = lrow[t4];
        x[4 * t4 + 0] = fmaf(-l.x, u0, x[4 * t4 + 0]);
        x[4 * t4 + 1] = fmaf(-l.y, u0, x[4 * t4 + 1]);
        x[4 * t4 + 2] = fmaf(-l.z, u0, x[4 * t4 + 2]);
        x[4 * t4 + 3] = fmaf(-l.w, u0, x[4 * t4 + 3]);
      }
    }
#pragma unroll
    for (int t = 1; t < 16; ++t)
#pragma unroll
      for (int s = 0; s < t; ++s) x[t] = fmaf(-LT[(b + s) * Mp + b + t], x[s], x[t]);
#pragma unroll
    for (int t = 0; t < 16; ++t) us[(b + t) * US + c0] = x[t];
  }
  __syncthreads();
  // U^T rows [hi | hi | lo]: warp w writes rows n0 + w, n0 + w + 8, ...; lanes walk tokens
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rr = warp; rr < SOLVE_COLS; rr += 8) {
    if (n0 + rr >= q.d) break;
    __nv_bfloat16* out = w.UTs + ((long long)g * q.d + n0 + rr) * 3 * Mp;
    for (int i = 2 * lane; i < Mp; i += 64) {
      __nv_bfloat16 h0, l0, h1, l1;
      split_bf16(us[i * US + rr], h0, l0);
      split_bf16(us[(i + 1) * US + rr], h1, l1);
      const __nv_bfloat162 hh = __halves2bfloat162(h0, h1), ll = __halves2bfloat162(l0, l1);
      *reinterpret_cast<__nv_bfloat162*>(out + i) = hh;
      *reinterpret_cast<__nv_bfloat162*>(out + Mp + i) = hh;
      *reinterpret_cast<__nv_bfloat162*>(out + 2 * Mp + i) = ll;
    }
  }
}

}  // namespace foldtc
}  // namespace armt

using namespace armt;

extern "C" long long armt_fold_tc_workspace_bytes(int G, int n_mem, int d, int d_phi) {
  long long total = 0;
  foldtc::carve(nullptr, foldtc::geom(G, n_mem, d, d_phi), &total);
  return total + 256;
}

extern "C" long long armt_memop_rows(int d, int n_mem) { return foldtc::geom(1, n_mem, d, 8).NB; }

extern "C" int armt_mem_fold_tc(const ArmtMembers* mem, const float* kvb, long long ld_kvb, long long kvb_stride,
                                int v_off, int k_off, int b_off, float* A, float* z, void* memop, int d, int n_mem,
                                int d_mem, int nu, float eps, void* ws, void* stream) {
  using namespace armt::foldtc;
  ARMT_REQUIRE(mem && mem->G >= 1 && mem->G <= ARMT_MAX_MEMBERS, ARMT_ERR_DIM, "fold_tc: bad member count");
  ARMT_REQUIRE(kvb && A && z && memop && ws, ARMT_ERR_INPUT, "fold_tc: null pointer");
  ARMT_REQUIRE(nu >= 1 && d_mem >= 1 && d >= 8 && d % 8 == 0, ARMT_ERR_DIM, "fold_tc: bad sizes");
  ARMT_REQUIRE(n_mem <= 32 * QMAX, ARMT_ERR_UNSUPPORTED, "fold_tc: M=%d > %d", n_mem, 32 * QMAX);
  if (n_mem == 0) return ARMT_OK;
  for (int g = 0; g < mem->G; ++g)
    for (int h = g + 1; h < mem->G; ++h)
      ARMT_REQUIRE(mem->layer[g] != mem->layer[h], ARMT_ERR_INPUT, "fold_tc: duplicate layer %d in one group",
                   mem->layer[g]);
  const int dphi = 2 * nu * d_mem;
  const Geom q = geom(mem->G, n_mem, d, dphi);
  cudaStream_t s = as_stream(stream);
  Ws w = carve(ws, q);
  auto* mo = reinterpret_cast<__nv_bfloat16*>(memop);

  const size_t phi_smem = sizeof(float) * ((size_t)PT * 2 * d_mem + (size_t)PT * (q.P + 1));
  ARMT_REQUIRE(phi_smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold_tc: d_phi too large");
  cudaFuncSetAttribute(fold_phi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)phi_smem);
  fold_phi_kernel<<<dim3(q.Mp / PT, mem->G), 256, phi_smem, s>>>(*mem, kvb, ld_kvb, kvb_stride, k_off, b_off, z, mo,
                                                                  d_mem, nu, q, w);
  ARMT_CHECK_LAUNCH("fold_phi");

  // GEMM1: [P | c' | K] (M x (d + 8 + M)) = Phi_s . memop[layer]^T, K = 3P
  {
    ArmtGemmArgs a;
    memset(&a, 0, sizeof(a));
    a.G = mem->G; a.M = n_mem; a.N = d + 8 + n_mem; a.K = 3 * q.P; a.ab_dtype = ARMT_BF16;
    a.A = w.Phis; a.lda = 3 * q.P; a.a_stride = (long long)n_mem * 3 * q.P;
    a.B = mo; a.ldb = 3 * q.P; a.b_stride = (long long)q.NB * 3 * q.P;
    a.C = w.Pf; a.ldc = q.NP1; a.c_stride = (long long)n_mem * q.NP1; a.c_dtype = ARMT_F32;
    a.epilogue = ARMT_EPI_STORE;
    for (int g = 0; g < mem->G; ++g) { a.a_slot[g] = g; a.b_index[g] = mem->layer[g]; a.c_slot[g] = g; }
    int rc = gemm_tc(a, s);
    if (rc) return rc;
  }
  const size_t chain_smem = sizeof(float) * ((size_t)std::max(q.Mp * q.Mp, 4 * dphi) + 3 * (size_t)q.Mp);
  if (n_mem <= 128) {
    cudaFuncSetAttribute(fold_chain_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem);
    fold_chain_kernel<4><<<mem->G, 512, chain_smem, s>>>(*mem, z, mo, eps, q, w);
  } else {
    cudaFuncSetAttribute(fold_chain_kernel<QMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem);
    fold_chain_kernel<QMAX><<<mem->G, 512, chain_smem, s>>>(*mem, z, mo, eps, q, w);
  }
  ARMT_CHECK_LAUNCH("fold_chain");

  const size_t solve_smem = sizeof(float) * ((size_t)q.Mp * q.Mp + (size_t)q.Mp * (SOLVE_COLS + 1));
  ARMT_REQUIRE(solve_smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold_tc: M too large for the solve");
  cudaFuncSetAttribute(fold_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem);
  dim3 grid((d + SOLVE_COLS - 1) / SOLVE_COLS, mem->G);
  fold_solve_kernel<<<grid, SOLVE_COLS, solve_smem, s>>>(kvb, ld_kvb, kvb_stride, v_off, q, w);
  ARMT_CHECK_LAUNCH("fold_solve");

  // GEMM3: A[layer] = A[layer] + U^T Phi (d x dphi, K = 3Mp); memop rows [0, d) <- split(A)
  {
    ArmtGemmArgs a;
    memset(&a, 0, sizeof(a));
    a.G = mem->G; a.M = d; a.N = dphi; a.K = 3 * q.Mp; a.ab_dtype = ARMT_BF16;
    a.A = w.UTs; a.lda = 3 * q.Mp; a.a_stride = (long long)d * 3 * q.Mp;
    a.B = w.PhiTs; a.ldb = 3 * q.Mp; a.b_stride = (long long)q.P * 3 * q.Mp;
    a.C = A; a.ldc = dphi; a.c_stride = (long long)d * dphi; a.c_dtype = ARMT_F32;
    a.epilogue = ARMT_EPI_RESIDUAL;
    a.R = A; a.ldr = dphi; a.r_stride = (long long)d * dphi;
    a.C2 = mo; a.ldc2 = 3 * q.P; a.c2_stride = (long long)q.NB * 3 * q.P; a.c2_split = q.P;
    for (int g = 0; g < mem->G; ++g) { a.a_slot[g] = g; a.b_index[g] = g; a.c_slot[g] = mem->layer[g]; }
    return gemm_tc(a, s);
  }
}
