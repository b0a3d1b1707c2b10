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
#include <cstdlib>
#include <cstring>
#include <mutex>
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
  g.P = (dphi + 31) / 32 * 32;   // 2P % 64 == 0: the [hi | lo] memory operand wraps at 2P
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
  // row layouts (token-major): phi32, Phi_s [hi|hi|lo], memop Phi' rows [hi|lo]
  __nv_bfloat16* mrow = memop + ((long long)layer * q.NB + q.d + 8) * 2 * P;
  for (int e = threadIdx.x; e < PT * P; e += blockDim.x) {
    const int t = e / P, c = e - t * P, i = i0 + t;
    if (i >= q.M) continue;
    const float v = sp[t * (P + 1) + c];
    if (c < q.dphi) w.phi32[((long long)g * q.M + i) * q.dphi + c] = v;
    __nv_bfloat16 hi, lo;
    split_bf16(v, hi, lo);
    __nv_bfloat16* a = w.Phis + ((long long)g * q.M + i) * 3 * P;
    a[c] = hi; a[P + c] = hi; a[2 * P + c] = lo;
    __nv_bfloat16* b = mrow + (long long)i * 2 * P;
    b[c] = hi; b[P + c] = lo;
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
  __nv_bfloat16* zrow = memop + ((long long)layer * q.NB + q.d) * 2 * q.P;
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
    zrow[c] = hi; zrow[q.P + c] = lo;
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


// ============================================================================
// Fold v2 (n_mem <= 128): no sequential substitution over the d value columns.
//
// With W = L^{-T} Phi (M x P), the update is A_M = A0 + U^T Phi = A0 + R^T W and
// R^T = V^T diag(beta) - P^T diag(coef), P^T = A0 Phi^T, so
//   A_M = A0 + [V^T | P^T] . [Y ; Z],   Y = diag(beta) W,  Z = -diag(coef) W.
// Everything that depends on the sequential chain is a small M x M or M x P
// matrix; the d-wide work is two tensor-core GEMMs, the first of which never
// waits on the chain:
//   fold_prep   phi (fp32 + bf16x3 split), beta, c_i = z0.phi_i, K = Phi Phi^T (fp32)
//   GEMM-R      [V^T | P^T] as a bf16 [hi | lo] operand (FOLDR epilogue); needs only phi
//   fold_w      per 32 features of a member: the z/gamma chain -> zq, gamma, coef (redone
//               by each of the member's CTAs: one warp, no extra launch or round trip); the
//               16 x 16 diagonal blocks of L = I + diag(coef) tril(K,-1) inverted; W = L^{-T} Phi
//               by blocked back substitution -> [Y | Z] bf16x3 rows; z_M = z0 + sum gamma_i phi_i
//   GEMM3       A += [V^T | P^T] [Y ; Z]^T (RESIDUAL epilogue, memop rows re-split)
// GEMM-R runs on a forked stream concurrently with fold_w.
// ============================================================================

constexpr int TB2 = 32;   // tokens per K block in fold_prep

struct Ws2 {
  float *phi32, *K, *c, *nrm, *beta;
  __nv_bfloat16 *Phis, *YZ, *VP;
};

__host__ __device__ inline Ws2 carve2(void* base, const Geom& q, long long* total_bytes = nullptr) {
  float* f = reinterpret_cast<float*>(base);
  Ws2 w;
  long long o = 0;
  auto take = [&](long long n) { float* p = f + o; o += align256(n); return p; };
  w.phi32 = take((long long)q.G * q.M * q.dphi);
  w.K = take((long long)q.G * q.Mp * q.Mp);
  w.c = take((long long)q.G * q.Mp);
  w.nrm = take((long long)q.G * q.Mp);
  w.beta = take((long long)q.G * q.Mp);
  w.Phis = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.M * 3 * q.P + 1) / 2));
  w.YZ = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.dphi * 6 * q.Mp + 1) / 2));
  w.VP = reinterpret_cast<__nv_bfloat16*>(take(((long long)q.G * q.d * 4 * q.Mp + 1) / 2));
  if (total_bytes) *total_bytes = o * 4;
  return w;
}

// global -> shared copies that hold no registers (the kernels below are latency-bound:
// every input is in flight at once, then one wait)
__device__ __forceinline__ void cpa4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ unsigned long long f2u(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float2 u2f(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}

// grid (nbt (nbt + 1) / 2, G): CTA (bi, bj), bi >= bj, owns the 32 x 32 block K[bi][bj]
// (and writes its mirror, so K is exactly symmetric); diagonal CTAs also emit the
// per-token quantities of their 32 tokens. phi_i = DPFP_nu(k_i) (armt/memory.py:34-45):
// feature c = (j-1)*2m + a is r[a] * r[(a + j) mod 2m], r = [relu(k), relu(-k)]; the
// (a, (a + j) mod 2m) pairs come from a per-CTA table (no division in the loops).
constexpr int PS2 = 4;   // phi row padding (floats): rows stay 16-byte aligned for float4 reads
__global__ void __launch_bounds__(256) fold_prep_kernel(const __grid_constant__ ArmtMembers mem,
                                                        const float* __restrict__ kvb, long long ld_kvb,
                                                        long long kvb_stride, int k_off, int b_off,
                                                        const float* __restrict__ z, int d_mem, Geom q, Ws2 w,
                                                        bool phi_only) {
  extern __shared__ __align__(16) float sm[];
  const int two_m = 2 * d_mem, P = q.P, PS = P + PS2, M = q.M, Mp = q.Mp;
  const int RS = two_m + 1;
  float* sp = sm;                      // [2][TB2][PS]   phi rows (float4-aligned)
  float* sk = sp + 2 * TB2 * PS;       // [2][TB2][d_mem] raw k
  float* sr = sk + 2 * TB2 * d_mem;    // [2][TB2][RS]   r = [relu(k), relu(-k)]
  float* sz = sr + 2 * TB2 * RS;       // [P] z0 of the member's layer
  float* sb = sz + P;                  // [TB2] raw beta logits
  int* ta = reinterpret_cast<int*>(sb + TB2);   // [P] first factor index (-1: zero feature)
  int* tb = ta + P;                              // [P] second factor index
  int t = blockIdx.x, bi = 0;
  if (phi_only) {   // grid (nbt, G): the per-token outputs of token block blockIdx.x only
    bi = t;
    t = bi;
  } else {
    while (t > bi) { t -= bi + 1; ++bi; }
  }
  const int bj = t;
  const int g = blockIdx.y, layer = mem.layer[g];
  const float* kv = kvb + (long long)g * kvb_stride;
  const int nsrc = bi == bj ? 1 : 2;
  const int tid = threadIdx.x;
  for (int s = 0; s < nsrc; ++s) {
    const int i0 = (s == 0 ? bi : bj) * TB2;
    for (int e = tid; e < TB2 * d_mem; e += 256) {
      const int tt = e / d_mem, c = e - tt * d_mem;
      const bool ok = i0 + tt < M;
      cpa4(sk + (s * TB2 + tt) * d_mem + c, kv + (ok ? (long long)(i0 + tt) * ld_kvb + k_off + c : 0), ok);
    }
  }
  const float* zl = z + (long long)layer * q.dphi;
  for (int c = tid; c < P; c += 256) cpa4(sz + c, zl + (c < q.dphi ? c : 0), c < q.dphi);
  if (bi == bj && tid < TB2) {
    const bool ok = bi * TB2 + tid < M;
    cpa4(sb + tid, kv + (ok ? (long long)(bi * TB2 + tid) * ld_kvb + b_off : 0), ok);
  }
  for (int c = tid; c < P; c += 256) {
    if (c < q.dphi) {
      const int j = c / two_m + 1, a = c - (j - 1) * two_m;
      ta[c] = a;
      tb[c] = (a + j) % two_m;
    } else {
      ta[c] = -1;
      tb[c] = 0;
    }
  }
  cpa_wait_all();
  __syncthreads();
  for (int e = tid; e < nsrc * TB2 * d_mem; e += 256) {
    const int st = e / d_mem, c = e - st * d_mem;
    const float k = sk[e];
    sr[st * RS + c] = fmaxf(k, 0.f);
    sr[st * RS + d_mem + c] = fmaxf(-k, 0.f);
  }
  __syncthreads();
  // phi rows: thread = feature, loop over tokens
  for (int c = tid; c < PS; c += 256) {
    const int a = c < P ? ta[c] : -1, b = c < P ? tb[c] : 0;
    for (int s = 0; s < nsrc; ++s) {
      const int i0 = (s == 0 ? bi : bj) * TB2;
#pragma unroll 8
      for (int tt = 0; tt < TB2; ++tt) {
        const float* r = sr + (s * TB2 + tt) * RS;
        sp[(s * TB2 + tt) * PS + c] = (a >= 0 && i0 + tt < M) ? r[a] * r[b] : 0.f;
      }
    }
  }
  __syncthreads();
  if (!phi_only) {
  const float* pr = sp;
  const float* pc = sp + (nsrc - 1) * TB2 * PS;
  // K block: thread (ty, tx) -> rows {ty, ty+16} x cols {tx, tx+16}; 4 features per step
  // (float4 reads, packed f32x2 FMAs: even / odd features in the two lanes of each pair,
  // combined at the end). K[a][b] and K[b][a] run the identical sequence, so K is symmetric.
  const int tx = tid & 15, ty = tid >> 4;
  unsigned long long k2[4] = {0ull, 0ull, 0ull, 0ull};
  const float4* ra0 = reinterpret_cast<const float4*>(pr + ty * PS);
  const float4* ra1 = reinterpret_cast<const float4*>(pr + (ty + 16) * PS);
  const float4* rb0 = reinterpret_cast<const float4*>(pc + tx * PS);
  const float4* rb1 = reinterpret_cast<const float4*>(pc + (tx + 16) * PS);
#pragma unroll 4
  for (int c4 = 0; c4 < P / 4; ++c4) {
    const float4 a0 = ra0[c4], a1 = ra1[c4], b0 = rb0[c4], b1 = rb1[c4];
    k2[0] = ffma2(f2u(a0.x, a0.y), f2u(b0.x, b0.y), k2[0]);
    k2[0] = ffma2(f2u(a0.z, a0.w), f2u(b0.z, b0.w), k2[0]);
    k2[1] = ffma2(f2u(a0.x, a0.y), f2u(b1.x, b1.y), k2[1]);
    k2[1] = ffma2(f2u(a0.z, a0.w), f2u(b1.z, b1.w), k2[1]);
    k2[2] = ffma2(f2u(a1.x, a1.y), f2u(b0.x, b0.y), k2[2]);
    k2[2] = ffma2(f2u(a1.z, a1.w), f2u(b0.z, b0.w), k2[2]);
    k2[3] = ffma2(f2u(a1.x, a1.y), f2u(b1.x, b1.y), k2[3]);
    k2[3] = ffma2(f2u(a1.z, a1.w), f2u(b1.z, b1.w), k2[3]);
  }
  float* Kg = w.K + (long long)g * Mp * Mp;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const float2 kv2 = u2f(k2[2 * u + v]);
      const float kk = kv2.x + kv2.y;
      const int i = bi * TB2 + ty + 16 * u, j = bj * TB2 + tx + 16 * v;
      if (i < Mp && j < Mp) {
        Kg[(long long)i * Mp + j] = kk;
        Kg[(long long)j * Mp + i] = kk;
        if (i == j) w.nrm[(long long)g * Mp + i] = kk;
      }
    }
  }
  if (bi != bj) return;
  // per-token outputs of the diagonal block: thread = feature
  const int i0 = bi * TB2;
  for (int c = tid; c < P; c += 256) {
#pragma unroll 4
    for (int tt = 0; tt < TB2; ++tt) {
      const int i = i0 + tt;
      if (i >= M) break;
      const float v = sp[tt * PS + c];
      if (c < q.dphi) w.phi32[((long long)g * M + i) * q.dphi + c] = v;
      __nv_bfloat16 hi, lo;
      split_bf16(v, hi, lo);
      __nv_bfloat16* a = w.Phis + ((long long)g * M + i) * 3 * P;   // [hi | hi | lo]: GEMM-R B operand
      a[c] = hi; a[P + c] = hi; a[2 * P + c] = lo;
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
  for (int tt = warp; tt < TB2; tt += 8) {
    const int i = i0 + tt;
    if (i >= Mp) break;
    float cz = 0.f;
    for (int c = lane; c < q.dphi; c += 32) cz = fmaf(sp[tt * PS + c], sz[c], cz);
    cz = warp_sum(cz);
    if (lane == 0) {
      w.c[(long long)g * Mp + i] = cz;
      w.beta[(long long)g * Mp + i] = i < M ? sigmoid_ref(sb[tt]) : 0.f;
    }
  }
}

// grid (nbt (nbt + 1) / 2, G), 256 threads, two CTAs per SM: CTA (bi, bj), bi >= bj, computes
// the fp32 block K[bi][bj] = Phi_bi Phi_bj^T (and its mirror; diagonal blocks also nrm) from
// the phi rows fold_prep (phi-only mode) wrote — one wave at C2 instead of fold_prep's two.
// 4 feature quarters x 64 threads, thread (ty, tx) -> rows {ty + 8u} x cols {tx + 8v}, 4
// features per step (float4 reads, packed f32x2 FMAs), partial blocks summed in a fixed order
// through shared memory, so K[a][b] and K[b][a] are the identical sum and K is symmetric.
__global__ void __launch_bounds__(256, 2) fold_k_kernel(Geom q, Ws2 w) {
  extern __shared__ __align__(16) float sm[];
  const int P = q.P, PS = P + PS2, M = q.M, Mp = q.Mp, dphi = q.dphi;
  float* sp = sm;   // [2][TB2][PS]
  int t = blockIdx.x, bi = 0;
  while (t > bi) { t -= bi + 1; ++bi; }
  const int bj = t, g = blockIdx.y, tid = threadIdx.x;
  const int nsrc = bi == bj ? 1 : 2;
  const float* ph = w.phi32 + (long long)g * M * dphi;
  const bool vec = (dphi & 3) == 0;
  for (int s2 = 0; s2 < nsrc; ++s2) {
    const int i0 = (s2 == 0 ? bi : bj) * TB2;
    float* dst = sp + s2 * TB2 * PS;
    if (vec) {
      const int c4n = P / 4;
      for (int e = tid; e < TB2 * c4n; e += 256) {
        const int tt = e / c4n, c4 = e - tt * c4n;
        float* d4 = dst + tt * PS + 4 * c4;
        if (i0 + tt < M && 4 * c4 < dphi) cpa16(d4, ph + (long long)(i0 + tt) * dphi + 4 * c4);
        else *reinterpret_cast<float4*>(d4) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      for (int e = tid; e < TB2 * P; e += 256) {
        const int tt = e / P, c = e - tt * P;
        const bool ok = i0 + tt < M && c < dphi;
        cpa4(dst + tt * PS + c, ph + (ok ? (long long)(i0 + tt) * dphi + c : 0), ok);
      }
    }
  }
  cpa_wait_all();
  __syncthreads();
  const float* pr = sp;
  const float* pc = sp + (nsrc - 1) * TB2 * PS;
  const int qf = tid >> 6, t64 = tid & 63, tx = t64 & 7, ty = t64 >> 3;
  const int c4_0 = qf * (P / 16), c4_1 = c4_0 + P / 16;   // P is a multiple of 32
  unsigned long long k2[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) k2[u][v] = 0ull;
#pragma unroll 2
  for (int c4 = c4_0; c4 < c4_1; ++c4) {
    float4 ra[4], rb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ra[u] = reinterpret_cast<const float4*>(pr + (ty + 8 * u) * PS)[c4];
      rb[u] = reinterpret_cast<const float4*>(pc + (tx + 8 * u) * PS)[c4];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        k2[u][v] = ffma2(f2u(ra[u].x, ra[u].y), f2u(rb[v].x, rb[v].y), k2[u][v]);
        k2[u][v] = ffma2(f2u(ra[u].z, ra[u].w), f2u(rb[v].z, rb[v].w), k2[u][v]);
      }
  }
  __syncthreads();   // sp is free: every thread is past its reads
  constexpr int RW = TB2 + 1;
  float* red = sp;   // [4][TB2][RW]
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float2 kv2 = u2f(k2[u][v]);
      red[(qf * TB2 + ty + 8 * u) * RW + tx + 8 * v] = kv2.x + kv2.y;
    }
  __syncthreads();
  float* Kg = w.K + (long long)g * Mp * Mp;
  for (int e = tid; e < TB2 * TB2; e += 256) {
    const int ii = e / TB2, jj = e - ii * TB2;
    const float kk = ((red[ii * RW + jj] + red[(TB2 + ii) * RW + jj]) + red[(2 * TB2 + ii) * RW + jj]) +
                     red[(3 * TB2 + ii) * RW + jj];
    const int i = bi * TB2 + ii, j = bj * TB2 + jj;
    if (i < Mp && j < Mp) {
      Kg[(long long)i * Mp + j] = kk;
      Kg[(long long)j * Mp + i] = kk;
      if (i == j) w.nrm[(long long)g * Mp + i] = kk;
    }
  }
}

// grid (ceil(dphi / 32), G), 256 threads. Each CTA redoes its member's (one-warp) chain —
// zq_i = c_i + sum_{j<i} gamma_j K_ij, gamma_i = nrm_i <= eps ? 0 : 1 - zq_i / nrm_i
// (armt/memory.py:101-106,116-119), coef_i = |zq_i| <= eps ? 0 : beta_i / zq_i — inverts the
// 16 x 16 diagonal blocks of L = I + diag(coef) tril(K,-1), then computes W = L^{-T} Phi for its
// 32 features by blocked back substitution, W_b = L_bb^{-T} (Phi_b - sum_{k>b} L_kb^T W_k), and
// writes [Y hi | Z hi | Y hi | Z hi | Y lo | Z lo] (Y = beta_i W[i][p], Z = -coef_i W[i][p]) — the
// bf16x3 B operand of GEMM3 — and z_M[p] = z0[p] + sum_i gamma_i phi_i[p] (+ its memop row).
__global__ void __launch_bounds__(256, 2) fold_w_kernel(const __grid_constant__ ArmtMembers mem, float eps,
                                                        float* __restrict__ z, __nv_bfloat16* __restrict__ memop,
                                                        Geom q, Ws2 w) {
  extern __shared__ __align__(16) float sm[];
  const int Mp = q.Mp, M = q.M, nb = Mp / 16;
  constexpr int WS = 33;
  float* sL = sm;                  // [Mp][Mp]: K, then L's strict lower part
  float* sW = sL + Mp * Mp;        // [Mp][WS]: Phi slice, overwritten by W block by block
  float* sD = sW + Mp * WS;        // [Mp][16]: diagonal-block inverses
  float* sR = sD + Mp * 16;        // [16][WS]: block right-hand side
  float* sc = sR + 16 * WS;        // [Mp] c = z0 . phi
  float* snrm = sc + Mp;           // [Mp]
  float* sbt = snrm + Mp;          // [Mp] beta
  float* szq = sbt + Mp;           // [Mp]
  float* sg = szq + Mp;            // [Mp] gamma
  float* scf = sg + Mp;            // [Mp] coef
  const int p0 = blockIdx.x * 32, g = blockIdx.y, layer = mem.layer[g];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float* Kg = w.K + (long long)g * Mp * Mp;
    for (int e = tid; e < Mp * Mp / 4; e += 256) cpa16(sL + 4 * e, Kg + 4 * e);
    const float* ph = w.phi32 + (long long)g * M * q.dphi;
    for (int e = tid; e < Mp * 32; e += 256) {
      const int i = e >> 5, c = e & 31;
      const bool ok = i < M && p0 + c < q.dphi;
      cpa4(sW + i * WS + c, ph + (ok ? (long long)i * q.dphi + p0 + c : 0), ok);
    }
    if (tid < Mp) {
      cpa4(sc + tid, w.c + (long long)g * Mp + tid, true);
      cpa4(snrm + tid, w.nrm + (long long)g * Mp + tid, true);
      cpa4(sbt + tid, w.beta + (long long)g * Mp + tid, true);
    }
    cpa_wait_all();
  }
  __syncthreads();
  if (warp == 0) {
    // ---- the chain, blocks of 4 tokens (lane t owns tokens t, t+32, t+64, t+96)
    float e[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int tt = lane + 32 * r;
      e[r] = tt < M ? sc[tt] : 0.f;
    }
    const int rmax = (M + 31) / 32;
    for (int i0 = 0; i0 < M; i0 += 4) {
      const int qi = i0 >> 5, l0 = i0 & 31;
      float mine = 0.f;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r == qi) mine = e[r];
      float zq[4], gam[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) zq[u] = __shfl_sync(0xffffffffu, mine, l0 + u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
#pragma unroll
        for (int v = 0; v < u; ++v) zq[u] = fmaf(gam[v], sL[(i0 + v) * Mp + i], zq[u]);
        const float nrm = i < M ? snrm[i] : 0.f;
        gam[u] = (i < M && nrm > eps) ? 1.f - __fdividef(zq[u], nrm) : 0.f;
      }
      if (lane < 4 && i0 + lane < M) {
        szq[i0 + lane] = lane == 0 ? zq[0] : lane == 1 ? zq[1] : lane == 2 ? zq[2] : zq[3];
        sg[i0 + lane] = lane == 0 ? gam[0] : lane == 1 ? gam[1] : lane == 2 ? gam[2] : gam[3];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r < rmax) {
          const int tt = lane + 32 * r;
          if (tt >= i0 + 4 && tt < M) {
            float acc = e[r];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = fmaf(gam[u], sL[(i0 + u) * Mp + tt], acc);
            e[r] = acc;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < Mp; i += 256) {
    float cf = 0.f;
    if (i < M) {
      const float zq = szq[i];
      cf = fabsf(zq) <= eps ? 0.f : sbt[i] / zq;
    } else {
      sg[i] = 0.f;
    }
    scf[i] = cf;
  }
  __syncthreads();
  // L strict lower part in place: row j = warp + 8k, columns = lanes
  for (int j = warp; j < Mp; j += 8) {
    const float cj = scf[j];
    for (int i = lane; i < Mp; i += 32) sL[j * Mp + i] = i < j ? cj * sL[j * Mp + i] : 0.f;
  }
  __syncthreads();
  // diagonal blocks: sD[(r0 + t) * 16 + col] = (L_bb^{-1})[t][col], one column per thread
  if (tid < nb * 16) {
    const int b = tid >> 4, col = tid & 15, r0 = 16 * b;
    float x[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      float acc = t == col ? 1.f : 0.f;
#pragma unroll
      for (int s2 = 0; s2 < t; ++s2) acc = fmaf(-sL[(r0 + t) * Mp + r0 + s2], x[s2], acc);
      x[t] = acc;
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) sD[(r0 + t) * 16 + col] = x[t];
  }
  // z_M (4 partial chains, fixed order) while the Phi slice is intact
  if (warp == 7) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int i = 0;
    for (; i + 4 <= M; i += 4) {
      a0 = fmaf(sg[i], sW[i * WS + lane], a0);
      a1 = fmaf(sg[i + 1], sW[(i + 1) * WS + lane], a1);
      a2 = fmaf(sg[i + 2], sW[(i + 2) * WS + lane], a2);
      a3 = fmaf(sg[i + 3], sW[(i + 3) * WS + lane], a3);
    }
    for (; i < M; ++i) a0 = fmaf(sg[i], sW[i * WS + lane], a0);
    const int pp = p0 + lane;
    if (pp < q.dphi) {
      const float acc = z[(long long)layer * q.dphi + pp] + ((a0 + a1) + (a2 + a3));
      z[(long long)layer * q.dphi + pp] = acc;
      __nv_bfloat16 hi, lo;
      split_bf16(acc, hi, lo);
      __nv_bfloat16* zrow = memop + ((long long)layer * q.NB + q.d) * 2 * q.P;
      zrow[pp] = hi; zrow[q.P + pp] = lo;
    }
  }
  __syncthreads();
  // blocked back substitution; thread (r = tid / 16, columns cp, cp + 16), cp = tid % 16
  const int r = tid >> 4, cp = tid & 15;
  for (int b = nb - 1; b >= 0; --b) {
    const int r0 = 16 * b, i = r0 + r;
    float s0 = sW[i * WS + cp], s1 = sW[i * WS + cp + 16];
    float t0 = 0.f, t1 = 0.f;
#pragma unroll 2
    for (int j = r0 + 16; j < Mp; j += 2) {   // rows of later blocks are final
      const float l0 = sL[j * Mp + i], l1 = sL[(j + 1) * Mp + i];
      s0 = fmaf(-l0, sW[j * WS + cp], s0);
      s1 = fmaf(-l0, sW[j * WS + cp + 16], s1);
      t0 = fmaf(-l1, sW[(j + 1) * WS + cp], t0);
      t1 = fmaf(-l1, sW[(j + 1) * WS + cp + 16], t1);
    }
    sR[r * WS + cp] = s0 + t0;
    sR[r * WS + cp + 16] = s1 + t1;
    __syncthreads();
    // W_i = sum_t (L_bb^{-1})[t][r] R_t (lower triangular: t >= r)
    float w0 = 0.f, w1 = 0.f;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const float dv = sD[(r0 + t) * 16 + r];
      w0 = fmaf(dv, sR[t * WS + cp], w0);
      w1 = fmaf(dv, sR[t * WS + cp + 16], w1);
    }
    sW[i * WS + cp] = w0;
    sW[i * WS + cp + 16] = w1;
    __syncthreads();
  }
  // [Y | Z] rows: thread = (feature c = warp + 8k, token pair 2 * lane + 64 m)
  for (int c = warp; c < 32; c += 8) {
    const int pp = p0 + c;
    if (pp >= q.dphi) break;
    __nv_bfloat16* o = w.YZ + ((long long)g * q.dphi + pp) * 6 * Mp;
    for (int i = 2 * lane; i < Mp; i += 64) {
      const float w0 = sW[i * WS + c], w1 = sW[(i + 1) * WS + c];
      __nv_bfloat16 yh0, yl0, yh1, yl1, zh0, zl0, zh1, zl1;
      split_bf16(sbt[i] * w0, yh0, yl0);
      split_bf16(sbt[i + 1] * w1, yh1, yl1);
      split_bf16(-scf[i] * w0, zh0, zl0);
      split_bf16(-scf[i + 1] * w1, zh1, zl1);
      const __nv_bfloat162 yh = __halves2bfloat162(yh0, yh1), zh = __halves2bfloat162(zh0, zh1);
      *reinterpret_cast<__nv_bfloat162*>(o + i) = yh;
      *reinterpret_cast<__nv_bfloat162*>(o + Mp + i) = zh;
      *reinterpret_cast<__nv_bfloat162*>(o + 2 * Mp + i) = yh;
      *reinterpret_cast<__nv_bfloat162*>(o + 3 * Mp + i) = zh;
      *reinterpret_cast<__nv_bfloat162*>(o + 4 * Mp + i) = __halves2bfloat162(yl0, yl1);
      *reinterpret_cast<__nv_bfloat162*>(o + 5 * Mp + i) = __halves2bfloat162(zl0, zl1);
    }
  }
}

}  // namespace foldtc
}  // namespace armt

using namespace armt;

extern "C" long long armt_fold_tc_workspace_bytes(int G, int n_mem, int d, int d_phi) {
  long long t1 = 0, t2 = 0;
  foldtc::carve(nullptr, foldtc::geom(G, n_mem, d, d_phi), &t1);
  foldtc::carve2(nullptr, foldtc::geom(G, n_mem, d, d_phi), &t2);
  return (t1 > t2 ? t1 : t2) + 256;
}

namespace {

// Fold v2 host sequence (see the block comment above fold_prep_kernel).
int fold_v2(const ArmtMembers* mem, const float* kvb, long long ld_kvb, long long kvb_stride, int v_off,
            int k_off, int b_off, float* A, float* z, __nv_bfloat16* mo, int d, int n_mem, int d_mem, float eps,
            const armt::foldtc::Geom& q, void* ws, cudaStream_t s) {
  using namespace armt::foldtc;
  const int G = mem->G;
  Ws2 w = carve2(ws, q);
  const int nbt = (q.Mp + TB2 - 1) / TB2;
  const size_t prep_smem = sizeof(float) * ((size_t)2 * TB2 * (q.P + PS2) + (size_t)2 * TB2 * d_mem +
                                            (size_t)2 * TB2 * (2 * d_mem + 1) + 3 * (size_t)q.P + TB2);
  ARMT_REQUIRE(prep_smem <= 227 * 1024, ARMT_ERR_UNSUPPORTED, "fold_tc: d_phi too large");
  cudaFuncSetAttribute(fold_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prep_smem);
  const int kblocks = nbt * (nbt + 1) / 2 * G;
  if (kblocks <= armt::num_sms()) {
    // one wave: phi and the K blocks in one kernel (one CTA per SM, 153 KB of phi rows)
    fold_prep_kernel<<<dim3(nbt * (nbt + 1) / 2, G), 256, prep_smem, s>>>(*mem, kvb, ld_kvb, kvb_stride, k_off,
                                                                          b_off, z, d_mem, q, w, false);
    ARMT_CHECK_LAUNCH("fold_prep");
  } else {
    // more K blocks than SMs (C2, G = 16: 160): phi, c, beta and the GEMM-R operand per token
    // block first, then K = Phi Phi^T from those rows at two CTAs per SM — one wave instead of
    // two (G = 16: 29 vs 35 us; at G = 1 the extra launch would cost 4 us, hence the switch)
    fold_prep_kernel<<<dim3(nbt, G), 256, prep_smem, s>>>(*mem, kvb, ld_kvb, kvb_stride, k_off, b_off, z, d_mem,
                                                           q, w, true);
    ARMT_CHECK_LAUNCH("fold_prep");
    const size_t k_smem = sizeof(float) * std::max((size_t)2 * TB2 * (q.P + PS2), (size_t)4 * TB2 * (TB2 + 1));
    cudaFuncSetAttribute(fold_k_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k_smem);
    fold_k_kernel<<<dim3(nbt * (nbt + 1) / 2, G), 256, k_smem, s>>>(q, w);
    ARMT_CHECK_LAUNCH("fold_k");
  }

  // GEMM-R on a forked stream: [V^T | P^T] needs only phi, so it overlaps the chain
  ForkedStream* fk = forked_stream(s);
  cudaStream_t sr = s;
  if (fk != nullptr) {
    const int rc = fk->fork();
    if (rc) return rc;
    sr = fk->side;
  }
  {
    ArmtGemmArgs a;
    memset(&a, 0, sizeof(a));
    a.G = G; a.M = d; a.N = n_mem; a.K = 3 * q.P; a.ab_dtype = ARMT_BF16;
    a.A = mo; a.lda = 2 * q.P; a.a_stride = (long long)q.NB * 2 * q.P; a.a_kwrap = 2 * q.P;
    a.B = w.Phis; a.ldb = 3 * q.P; a.b_stride = (long long)n_mem * 3 * q.P;
    a.C = w.VP; a.ldc = 4 * q.Mp; a.c_stride = (long long)d * 4 * q.Mp; a.c_dtype = ARMT_BF16;
    a.R = kvb + v_off; a.ldr = ld_kvb; a.r_stride = kvb_stride; a.c2_split = q.Mp;
    a.epilogue = ARMT_EPI_FOLDR;
    // leave SMs for the chain kernel running beside it
    a.max_ctas = fk != nullptr ? std::max(2, armt::num_sms() - std::min(G, 32) - 4) : 0;
    for (int g = 0; g < G; ++g) { a.a_slot[g] = mem->layer[g]; a.b_index[g] = g; a.c_slot[g] = g; }
    int rc = gemm_tc(a, sr);
    if (rc) return rc;
  }
  const size_t w_smem = sizeof(float) * ((size_t)q.Mp * q.Mp + (33 + 16 + 6) * (size_t)q.Mp + 16 * 33);
  cudaFuncSetAttribute(fold_w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w_smem);
  fold_w_kernel<<<dim3((q.dphi + 31) / 32, G), 256, w_smem, s>>>(*mem, eps, z, mo, q, w);
  ARMT_CHECK_LAUNCH("fold_w");
  if (fk != nullptr) {
    const int rc = fk->join();
    if (rc) return rc;
  }
  // GEMM3: A[layer] += [V^T | P^T] [Y ; Z]^T (K = 6 Mp over a 4 Mp operand); memop rows [0, d) <- split(A)
  ArmtGemmArgs a;
  memset(&a, 0, sizeof(a));
  a.G = G; a.M = d; a.N = q.dphi; a.K = 6 * q.Mp; a.ab_dtype = ARMT_BF16;
  a.A = w.VP; a.lda = 4 * q.Mp; a.a_stride = (long long)d * 4 * q.Mp; a.a_kwrap = 4 * q.Mp;
  a.B = w.YZ; a.ldb = 6 * q.Mp; a.b_stride = (long long)q.dphi * 6 * q.Mp;
  a.C = A; a.ldc = q.dphi; a.c_stride = (long long)d * q.dphi; a.c_dtype = ARMT_F32;
  a.epilogue = ARMT_EPI_RESIDUAL;
  a.R = A; a.ldr = q.dphi; a.r_stride = (long long)d * q.dphi;
  a.C2 = mo; a.ldc2 = 2 * q.P; a.c2_stride = (long long)q.NB * 2 * q.P; a.c2_split = q.P;
  for (int g = 0; g < G; ++g) { a.a_slot[g] = g; a.b_index[g] = g; a.c_slot[g] = mem->layer[g]; }
  return gemm_tc(a, s);
}

}  // namespace

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
  auto* mo = reinterpret_cast<__nv_bfloat16*>(memop);
  // v2 (no substitution over the value columns) for n_mem <= 128; ARMT_FOLD_V1=1 keeps v1 (A/B)
  static const bool v1 = getenv("ARMT_FOLD_V1") && getenv("ARMT_FOLD_V1")[0] == '1';
  if (q.Mp <= 128 && d_mem <= 64 && q.P <= 512 && !v1)
    return fold_v2(mem, kvb, ld_kvb, kvb_stride, v_off, k_off, b_off, A, z, mo, d, n_mem, d_mem, eps, q, ws, s);
  Ws w = carve(ws, q);

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
    a.B = mo; a.ldb = 2 * q.P; a.b_stride = (long long)q.NB * 2 * q.P; a.b_kwrap = 2 * q.P;
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
    a.C2 = mo; a.ldc2 = 2 * q.P; a.c2_stride = (long long)q.NB * 2 * q.P; a.c2_split = q.P;
    for (int g = 0; g < mem->G; ++g) { a.a_slot[g] = g; a.b_index[g] = g; a.c_slot[g] = mem->layer[g]; }
    return gemm_tc(a, s);
  }
}
