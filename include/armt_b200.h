/*
 * armt_b200.h — C-ABI of the B200-native ARMT segment-recurrent forward.
 *
 * Drop-in boundary for the reference's stacked cores. The reference has no
 * FFI: its operator boundary is the three Python functions its executors
 * call once per schedule step (armt/executors.py:139-141, 200-203) plus the
 * grouped GEMM they are built from. Each entry point below names the
 * reference interface it replaces. The Python package
 * paper_2506_05229_b200 binds these with ctypes and
 * keeps the reference's Python signatures on top.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer (owned by the caller, e.g. torch);
 *     every call enqueues work on `stream` (a cudaStream_t passed as void*)
 *     and returns immediately. No entry point allocates device memory.
 *   - Strides are in ELEMENTS. "slot" tables index per-segment activation
 *     buffers, "layer" tables index layer-stacked weights/state; member g of
 *     a grouped call is (slot[g], layer[g]) — the per-layer pointer arrays of
 *     the diagonal wavefront.
 *   - Return value: ARMT_OK or an ArmtStatus; armt_last_error() gives text.
 *     The Python boundary maps ARMT_ERR_DIM -> DimensionError,
 *     ARMT_ERR_INPUT -> InputError, others -> DeviceError.
 */
#ifndef ARMT_B200_H
#define ARMT_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define ARMT_MAX_MEMBERS 128

typedef enum {
  ARMT_OK = 0,
  ARMT_ERR_DIM = 1,          /* shapes/strides/alignment violate the contract */
  ARMT_ERR_INPUT = 2,        /* bad values (ids, eps, sizes) */
  ARMT_ERR_UNSUPPORTED = 3,  /* legal but not implemented on this path */
  ARMT_ERR_CUDA = 4          /* CUDA runtime / launch error */
} ArmtStatus;

typedef enum { ARMT_F32 = 0, ARMT_BF16 = 1 } ArmtDtype;

/* Fused GEMM epilogues. */
typedef enum {
  ARMT_EPI_STORE = 0,     /* C = acc                                                  */
  ARMT_EPI_RESIDUAL = 1,  /* C = R + acc (f32); optional C2 = bf16(C)                 */
  ARMT_EPI_RETRIEVE = 2,  /* C = R + (|den| <= eps ? 0 : acc/den)  armt/memory.py:149-152 */
  ARMT_EPI_SWIGLU = 3,    /* C[:, j] = silu(acc_gate) * acc_up     armt/layers.py:228-232 */
  ARMT_EPI_ROPE = 4,      /* C = rope(acc) on cols < rope_cols     armt/layers.py:169-176 */
  ARMT_EPI_LSE = 5,       /* no C: per row and N-tile (max, sum exp) of acc in base-2 units into
                             lse_part[row*lse_ld + nb] (float2), and acc[row][targets[row]] into
                             lse_tgt[row] -- the fused next-token NLL of the LM head */
  ARMT_EPI_DPFP = 6,      /* acc = q (M x N, N = d_mem <= 64): C = bf16 DPFP_nu(q) (ldc >= 2*nu*N) and
                             den[g*den_stride + m] = DPFP(q) . z[e_index[g]] (z rows of 2*nu*N floats)
                             armt/memory.py:34-45,137-147 -- retrieval's feature map fused into q-proj */
  ARMT_EPI_FOLDR = 7      /* fold-internal (armt_mem_fold_tc): acc = P^T = A0 Phi^T (M = d rows, N = n_mem
                             token columns); C row r = bf16 [V hi | P hi | V lo | P lo],
                             c2_split = segment width, V[r][i] = R[i*ldr + r] (value rows, token-major) */
} ArmtEpilogue;

/* Members of one grouped launch: member g runs slot[g] against layer[g]. */
typedef struct {
  int G;
  int slot[ARMT_MAX_MEMBERS];
  int layer[ARMT_MAX_MEMBERS];
} ArmtMembers;

/*
 * Grouped GEMM: for g < G,  C[c_slot[g]] (M x N) = epi( A[a_slot[g]] (M x K) . B[b_index[g]]^T )
 * A is K-major (row m contiguous over k), B is K-major (row n contiguous over k,
 * i.e. the weight stored (out, in)). Operand dtype selects the engine:
 * ARMT_BF16 -> tcgen05/TMEM/TMA kernel; ARMT_F32 -> SIMT fp32 kernel (parity mode).
 */
typedef struct {
  int G, M, N, K;
  int ab_dtype;                         /* ArmtDtype of A and B */
  const void* A; long long lda, a_stride;
  const void* B; long long ldb, b_stride;
  void* C; long long ldc, c_stride; int c_dtype;
  int epilogue;                         /* ArmtEpilogue */
  const float* R; long long ldr, r_stride;     /* RESIDUAL/RETRIEVE input, indexed by c_slot */
  void* C2; long long ldc2, c2_stride;         /* RESIDUAL: optional bf16 copy, indexed by c_slot */
  int c2_split;                         /* >0: C2 gets the [hi | lo] bf16 split of C at cols n, n+s */
  /* fused RMSNorm (bf16 path): RESIDUAL/RETRIEVE epilogues write sum(C^2) of each row per
   * 64-column block to ssq_out[g*ssq_stride + m*ssq_np + n/64]; ROPE/SWIGLU epilogues scale
   * the accumulator row by 1/sqrt(sum_p ssq_in[g*ssq_stride + m*ssq_np + p]/norm_d + norm_eps),
   * summing the ssq_np partials in order (deterministic: no atomics). */
  float* ssq_out; const float* ssq_in; long long ssq_stride; int ssq_np;
  int norm_d; float norm_eps;
  float* lse_part; long long lse_ld; const long long* targets; float* lse_tgt; int lse_rows;
  const float* den; long long den_stride;      /* RETRIEVE: den[g*den_stride + m] */
  float eps;
  const float* rope_cos; const float* rope_sin;  /* ROPE: (head_dim/2, M) tables, position-contiguous */
  int head_dim; int rope_cols;
  int swiglu_block;                     /* SWIGLU: cols [t*2b, t*2b+b) gate, [t*2b+b, (t+1)*2b) up */
  int max_ctas;                         /* bf16 engine: cap on resident CTAs (0 = one per SM); lets a
                                           launch leave SMs free for a concurrent stream */
  const float* z; int nu;               /* DPFP: memory normaliser rows and feature-map order */
  int a_kwrap, b_kwrap;                 /* >0: operand K columns [w, K) are read from [0, K - w) (a bf16x3
                                           operand stores [hi | lo] once and reuses hi as its third part);
                                           multiples of 64; 0 = plain */
  int a_slot[ARMT_MAX_MEMBERS];
  int b_index[ARMT_MAX_MEMBERS];
  int c_slot[ARMT_MAX_MEMBERS];
  int e_index[ARMT_MAX_MEMBERS];        /* DPFP: memory-state row of member g's z */
} ArmtGemmArgs;

/* Replaces grouped_gemm / gemm / _project (armt/tensor_ops.py:204-264,
 * armt/layers.py:183-188) with the fused epilogues of the callers. */
int armt_gemm(const ArmtGemmArgs* args, void* stream);

/* Replaces embed_segment (armt/layers.py:306-318): x[slot] = [emb[ids]; mem_emb].
 * ids are int64 [seg], validated by the caller; emb/mem_emb dtype = w_dtype.
 * Writes f32 x (T x d, row stride d) and, if x_bf != NULL, a bf16 copy. */
int armt_embed(const long long* ids, const void* emb, const void* mem_emb, int w_dtype,
               float* x, void* x_bf, int seg, int n_mem, int d, int vocab, void* stream);

/* Ids outside [0, vocab) seen by armt_embed since the last reset (their rows
 * are written as zeros, never gathered). Synchronous; -1 on a CUDA error. */
long long armt_embed_bad_ids(int reset);

/* Replaces rms_norm_stacked (armt/tensor_ops.py:267-281):
 * out[g] = x[slot[g]] / sqrt(mean(x^2) + eps) * gain[layer[g]]. */
int armt_rmsnorm(const ArmtMembers* mem, const float* x, long long x_stride,
                 const float* gain, void* out, int out_dtype, long long out_stride,
                 int rows, int d, float eps, void* stream);

/* Replaces the DPFP feature map + denominator of retrieve_stack
 * (armt/memory.py:34-45, 139-147): phi[g] = DPFP_nu(q[g]); den[g] = phi[g].z[layer[g]]. */
int armt_dpfp_den(const ArmtMembers* mem, const float* q, long long q_stride,
                  const float* z, void* phi, int phi_dtype, long long ld_phi,
                  long long phi_stride, float* den, long long den_stride,
                  int rows, int d_mem, int nu, void* stream);

/* Replaces QK^T / softmax / PV / head merge of _attention_stack
 * (armt/layers.py:211-223): causal attention over T rows per member and head.
 * qkv rows hold [q | k | v] (3*d cols, q/k already rotated); ctx rows hold d cols. */
int armt_attention(int G, const void* qkv, long long ld_qkv, long long qkv_stride,
                   void* ctx, long long ld_ctx, long long ctx_stride, int dtype,
                   int T, int n_heads, int d_head, float scale, void* stream);

/* Stand-alone RoPE on the q|k columns of qkv (armt/layers.py:169-176, 207-208);
 * the bf16 path fuses this into the QKV GEMM epilogue instead. */
int armt_rope(int G, void* qkv, long long ld_qkv, long long qkv_stride, int dtype, int T,
              int n_heads, int d_head, const float* cos_t, const float* sin_t, void* stream);

/* Stand-alone SwiGLU over block-interleaved [gate | up] columns (armt/layers.py:228-232);
 * the bf16 path fuses this into the gate/up GEMM epilogue instead. */
int armt_swiglu(int G, const void* gu, long long ld_gu, long long gu_stride, void* out,
                long long ld_out, long long out_stride, int dtype, int rows, int d_ff,
                int block, void* stream);

/* Replaces update_stack's fold (armt/memory.py:94-125, 155-180): for each member,
 * fold its M memory tokens in order into A[layer], z[layer] (fp32, in place).
 * kvb[g] rows hold v (cols v_off..v_off+d), k (k_off..k_off+d_mem), beta logit (b_off).
 * If A_shadow != NULL, also refreshes the bf16 copy (L, d, ld_shadow) used by retrieval.
 * ws: device workspace of armt_fold_workspace_bytes(G, M, d_phi) bytes. */
int armt_mem_fold(const ArmtMembers* mem, const float* kvb, long long ld_kvb,
                  long long kvb_stride, int v_off, int k_off, int b_off, float* A, float* z,
                  void* A_shadow, long long ld_shadow, int d, int n_mem, int d_mem, int nu,
                  float eps, void* ws, void* stream);
long long armt_fold_workspace_bytes(int G, int n_mem, int d_phi);

/* Tensor-core form of the same fold for the bf16 path (chunked delta rule: with
 * L = I + diag(c) tril(Phi Phi^T, -1) and W = L^{-T} Phi, A += [V^T | (A Phi^T)^T-rows] [diag(beta) W ;
 * -diag(c) W]; grouped tcgen05 GEMMs on bf16x3-split operands, the chain and L^{-1} in smem).
 * `memop` (L, armt_memop_rows(d, M), 2*P) bf16, P = d_phi rounded up to 32, holds per layer
 * the [hi|lo] split of A (rows 0..d-1) and of z (row d); retrieval reads its hi part.
 * ws: armt_fold_tc_workspace_bytes(G, M, d, d_phi) bytes, zero-initialised once. */
int armt_mem_fold_tc(const ArmtMembers* mem, const float* kvb, long long ld_kvb,
                     long long kvb_stride, int v_off, int k_off, int b_off, float* A, float* z,
                     void* memop, int d, int n_mem, int d_mem, int nu, float eps, void* ws,
                     void* stream);
long long armt_fold_tc_workspace_bytes(int G, int n_mem, int d, int d_phi);
long long armt_memop_rows(int d, int n_mem);

/* Elementwise copy/cast between f32 and bf16 buffers (n elements). */
int armt_cast(const void* src, int src_dtype, void* dst, int dst_dtype, long long n, void* stream);

/* Next-token negative log-likelihood per row: nll[r] = logsumexp(logits[r]) - logits[r][target[r]].
 * Used by the end-to-end API to return a scalar result to the host. */
int armt_logits_nll(const void* logits, int dtype, long long ld, const long long* targets,
                    float* nll, long long rows, int vocab, void* stream);

/* Finalize the fused LM-head NLL: nll[r] = ln2 * (M + log2(sum_t s_t 2^(m_t - M))) - tgt[r],
 * M = max_t m_t over the n_tiles (max, sum) partials of row r (rows with target < 0 -> 0). */
int armt_lse_finalize(const float* lse_part, long long lse_ld, int n_tiles, const float* tgt,
                      const long long* targets, float* nll, long long rows, void* stream);

/* Reduce each row's n_tiles (max, sum) partials to one (max, sum) pair: out[r] (float2).
 * Vocab-parallel LM head: per-rank reduction before the cross-rank all-gather, whose
 * (rows, ranks) result armt_lse_finalize then turns into the NLL. */
int armt_lse_reduce(const float* lse_part, long long lse_ld, int n_tiles, float* out, long long rows,
                    void* stream);

/* Diagnostics: with ARMT_GEMM_PROF set at load, the tcgen05 GEMM accumulates wait cycles
 * ([0] MMA waiting for a full stage, [1] MMA waiting for a free accumulator, [2] MMA loop
 * cycles, [3] producer waiting for an empty stage, [4] tiles, [5] epilogue waiting). */
int armt_gemm_prof(unsigned long long* out8, int reset);

/* Introspection. */
const char* armt_last_error(void);
const char* armt_version(void);
int armt_num_sms(void);
int armt_kernel_count(void);   /* device kernels launched by this library since load */
/* ABI self-check for bindings: 0 -> sizeof(ArmtGemmArgs), 1 -> sizeof(ArmtMembers),
 * 2 -> offsetof(ArmtGemmArgs, a_slot). */
long long armt_abi_sizeof(int which);

#ifdef __cplusplus
}
#endif
#endif /* ARMT_B200_H */
