/*
 * b200moe -- C ABI of the B200-native MoE-layer hot path.
 *
 * The reference (moefold, /root/reference/pkg/src/moefold) is a pure
 * Python/numpy simulator: it has no FFI.  Its drop-in boundary is the Python
 * API re-exported by moefold/__init__.py:7-69; the package
 * paper_2504_14960_b200 mirrors that API and binds the entry points below with
 * ctypes.  Each entry point names the reference function
 * whose arithmetic it replaces.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *   - `stream` is a cudaStream_t passed as void*; nothing here synchronises
 *     the device or allocates memory (callers pass workspaces);
 *   - return value: B200MOE_OK or an error code; b200moe_last_error() gives a
 *     message.  Shape/argument validation happens before any launch.
 *   - dtype codes: B200MOE_F32 (float32) / B200MOE_BF16 (bfloat16).
 */
#ifndef B200MOE_H_
#define B200MOE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define B200MOE_API __attribute__((visibility("default")))
#else
#define B200MOE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define B200MOE_OK 0
#define B200MOE_EINVAL 1        /* bad argument / shape (ValidationError) */
#define B200MOE_ELAUNCH 2       /* CUDA launch or runtime failure        */
#define B200MOE_EUNSUPPORTED 3  /* configuration not supported by a kernel */
#define B200MOE_ENODEV 4        /* no sm_100 device                       */

#define B200MOE_F32 0
#define B200MOE_BF16 1

#define B200MOE_GATE_SOFTMAX 0 /* router.py:146-147 */
#define B200MOE_GATE_SIGMOID 1 /* router.py:148-149 */

#define B200MOE_ACT_RELU 0   /* experts.py:24-25 */
#define B200MOE_ACT_GELU 1   /* experts.py:26-28 (tanh approximation) */
#define B200MOE_ACT_SWIGLU 2 /* builder-defined: silu(x Wg) * (x Wu) */

#define B200MOE_MAJOR_K 0
#define B200MOE_MAJOR_MN 1

B200MOE_API const char* b200moe_version(void);
B200MOE_API const char* b200moe_last_error(void);
/* 0 when the current device is sm_100 (B200); B200MOE_ENODEV otherwise. */
B200MOE_API int b200moe_device_check(void);
/* let kernels on the current device dereference device `peer`'s memory (the
 * in-process multi-GPU world; already-enabled is not an error) */
B200MOE_API int b200moe_enable_peer_access(int peer);

/* ---------------------------------------------------------------- router */

/* logits[T,E] (fp32) = x[T,H] @ w_g[H,E]                -- router.py:145 */
B200MOE_API int b200moe_router_logits(const void* x, int x_dtype, const float* w_g, int64_t T, int64_t H,
                          int E, float* logits, void* stream);

/* scores = softmax/sigmoid(logits) (fp64 internally, stored fp32),
 * topk_idx[T,k] best first with ties to the lower expert id, gates[T,k] raw
 * or renormalised over the k winners.  gates_f64 (nullable) receives the
 * float64 gates, used as the probability-priority key.  A token with a
 * non-finite logit sets bit 0 of *status (nullable) and gets the placeholder
 * routing 0..k-1 (the host raises NumericError, router.py:141-144).
 *                                                       -- router.py:112-162 */
B200MOE_API int b200moe_router_topk(const float* logits, int64_t T, int E, int k, int gate_fn, int renorm,
                        float* scores, int32_t* topk_idx, float* gates, double* gates_f64,
                        int32_t* status, void* stream);

/* Fused router forward for bf16 tokens on the tensor cores: logits = x @ W_g
 * (tcgen05, x read once by TMA), then the b200moe_router_topk arithmetic in
 * the same kernel for E <= 32 (a second launch for 32 < E <= 64).  w_parts
 * is bf16 [NP, H], rows p*EP + e holding the exact three-way split
 * hi + mid + lo of W_g^T (EP = E rounded up to 8/16/32/64, NP =
 * b200moe_router_fwd_tc_np(E), zero padded).  status is required.
 *                                        -- router.py:141-162 (compute_gates) */
B200MOE_API int b200moe_router_fwd_tc_np(int E);
B200MOE_API int b200moe_router_fwd_tc(const void* x, int64_t T, int64_t H, const void* w_parts, int E, int k,
                                      int gate_fn, int renorm, float* logits, float* scores,
                                      int32_t* topk_idx, float* gates, double* gates_f64, int32_t* status,
                                      void* stream);

/* Workspace bytes needed by b200moe_dispatch_plan for T tokens, E experts. */
B200MOE_API size_t b200moe_dispatch_plan_ws(int64_t T, int E);

/* Capacity dropping + dispatch plan as one stable counting sort by expert.
 *   router.py:165-206 (apply_capacity, position priority) and
 *   dispatcher.py:96-131 (build_dispatch_plan).
 * kept_in   [T*k] u8, nullable: pairs with 0 are treated as already dropped.
 * order     [T] i32, nullable: token admission order for capacity (identity
 *           when positions are increasing in row order).
 * cap       per-expert capacity; <= 0 means dropless.
 * align     > 0: each expert segment of the padded (GEMM) layout is rounded up
 *           to a multiple of align rows; < 0: pad-to-capacity, every segment
 *           has exactly -align rows (requires 0 < cap <= -align), so all
 *           exchange sizes are static.
 * Outputs: kept_out[T*k] u8; expert_counts[E] (kept pairs);
 *   expert_offsets[E+1] (unpadded, send order); padded_offsets[E+1];
 *   send_row[T*k] (row of the pair in reference permutation order, -1 when
 *   dropped); gemm_row[T*k] (row in the padded expert-major layout, -1);
 *   perm[T*k] i64: perm[send_row] = token*k + slot (DispatchPlan.permutation);
 *   perm_gates[T*k] f32 nullable: gate of each send row (DispatchPlan.gates). */
B200MOE_API int b200moe_dispatch_plan(const int32_t* topk_idx, const float* gates, const uint8_t* kept_in,
                          const int32_t* order, int64_t T, int k, int E, int64_t cap, int align,
                          void* workspace, size_t workspace_bytes, uint8_t* kept_out,
                          int32_t* expert_counts, int32_t* expert_offsets, int32_t* padded_offsets,
                          int32_t* send_row, int32_t* gemm_row, int64_t* perm, float* perm_gates,
                          void* stream);

/* Probability-priority capacity (router.py:195): pair (t,s) of expert e is
 * kept iff fewer than `cap` pairs of e precede it in (-gate, position, slot)
 * order.  The pairs are given expert-segmented by a dropless plan
 * (perm0 / offsets0 from b200moe_dispatch_plan with cap <= 0);
 * gates_f64 [T*k]; positions[T] i64 nullable (identity). */
B200MOE_API int b200moe_capacity_by_gate(const int64_t* perm0, const int32_t* offsets0, const double* gates_f64,
                             const int64_t* positions, int64_t T, int k, int E, int64_t cap,
                             uint8_t* kept_out, void* stream);

/* dz[T,E] = d(gates)/d(logits)^T dgates                 -- dispatcher.py:470-488
 * dz_parts (nullable, bf16 [T, b200moe_router_parts_cols(E)]): also the exact
 * split hi + mid + lo of dz, cols p * EPW + e (EPW = E rounded up to
 * 8/16/32/64), zero padded -- the B operand of b200moe_router_wgrad_tc. */
B200MOE_API int b200moe_router_bwd(const float* dgates, const float* scores, const int32_t* topk_idx,
                       const float* gates, int64_t T, int E, int k, int gate_fn, int renorm,
                       float* dz, void* dz_parts, void* stream);
B200MOE_API int b200moe_router_parts_cols(int E);
/* dW_g[H,E] = x^T dz on the tensor cores (bf16 x [T,H], the dz parts of
 * b200moe_router_bwd), split over tokens and folded in fixed order; H % 64
 * == 0, E <= 64.                                          -- dispatcher.py:489 */
B200MOE_API size_t b200moe_router_wgrad_tc_ws(int64_t T, int64_t H, int E);
B200MOE_API int b200moe_router_wgrad_tc(const void* x, const void* dz_parts, int64_t T, int64_t H, int E,
                                        float* dw_g, void* workspace, size_t workspace_bytes, void* stream);

/* dw_g[H,E] (fp32, overwritten) = x^T dz, split over token chunks and
 * reduced in a fixed order (deterministic).  workspace: >=
 * b200moe_router_wgrad_ws(T, H, E) bytes.                -- dispatcher.py:489 */
B200MOE_API size_t b200moe_router_wgrad_ws(int64_t T, int64_t H, int E);
B200MOE_API int b200moe_router_wgrad(const void* x, int x_dtype, const float* dz, int64_t T, int64_t H, int E,
                         float* dw_g, void* workspace, size_t workspace_bytes, void* stream);

/* Full-sequence capacity over the TP x CP group (router.py:209-269).  The
 * group's pairs, all-gathered into fixed member slots, sorted on the device in
 * admission order: seg_sorted[N] = (pos / seq_len) * E + expert (INT64_MAX for
 * empty slots, sorted ascending; ties in priority order), order[N] = slot of
 * each sorted pair.  kept_slot[slot] = rank inside its segment < cap.
 * pos_by_pos (nullable): all pairs' positions sorted ascending; a position
 * shared by more than k pairs (two tokens) sets bit 3 of *status. */
B200MOE_API int b200moe_fullseq_capacity(const int64_t* seg_sorted, const int64_t* order, int64_t N,
                                         int64_t cap, uint8_t* kept_slot, const int64_t* pos_by_pos, int k,
                                         int32_t* status, void* stream);

/* load statistics (router.py:279-301): counts[e] = kept pairs routed to e,
 * top1[e] = tokens whose best expert is e, score_sum[e] = sum over tokens of
 * scores[t, e] / sum_e' scores[t, e'] (fp64; scores may be NULL).  kept may
 * be NULL (all kept).  Deterministic: per-chunk partials folded in order. */
B200MOE_API size_t b200moe_router_stats_ws(int64_t T, int E);
B200MOE_API int b200moe_router_stats(const int32_t* topk_idx, const uint8_t* kept, const float* scores,
                                     int64_t T, int k, int E, int64_t* counts, int64_t* top1,
                                     double* score_sum, void* workspace, size_t workspace_bytes,
                                     void* stream);

/* fp32 router GEMMs on the bf16 tensor cores (router.py:145, dispatcher.py:
 * 489-490 for bf16 tokens): an fp32 matrix is split into three bf16 parts
 * hi + mid + lo that sum to it exactly; with Ep = E rounded up to 8,
 * out3 [rows, 3 Ep] = (hi | mid | lo) and out6 [rows, 6 Ep] =
 * (hi | hi | hi | mid | mid | lo) (either may be NULL).  x . W_g then runs
 * as one b200moe_gemm_tc launch against the W_g parts, dz . W_g^T as one
 * launch over K = 6 Ep, x^T dz as one split-K launch. */
B200MOE_API int b200moe_split_bf16x3(const float* src, int64_t rows, int E, void* out3, void* out6,
                                     void* stream);
/* out[r, e] = sum over g ascending of ((p[g,r,e] + p[g,r,Ep+e]) + p[g,r,2Ep+e]),
 * parts [G, rows, 3 Ep] fp32: folds the three part products (and split-K groups). */
B200MOE_API int b200moe_sum_parts(const float* parts, int64_t G, int64_t rows, int E, float* out,
                                  void* stream);

/* ------------------------------------------------------- permute/combine */

/* out[row_of(t,s)] = x[t] (* scale[t,s] when scale != NULL) for every kept
 * pair (pair_row >= 0).                                 -- dispatcher.py:134-142
 * When padded_offsets/expert_counts are given, rows
 * [padded_offsets[e]+expert_counts[e], padded_offsets[e+1]) are zeroed
 * (align: the plan's align; at most align-1, or -align when negative, pad
 * rows per segment). */
B200MOE_API int b200moe_permute(const void* x, int dtype, int64_t T, int64_t H, int k, const int32_t* pair_row,
                    const float* scale, void* out, const int32_t* padded_offsets,
                    const int32_t* expert_counts, int E, int align, void* stream);

/* Backward dispatch (dispatcher.py:426-428): dy_rows[row] = gate * u[t] and
 * dgates[t*k+s] = <u[t], y_rows[row]> (0 for dropped pairs). */
B200MOE_API int b200moe_permute_bwd(const void* u, int dtype, int64_t T, int64_t H, int k,
                        const int32_t* pair_row, const float* gates, const void* y_rows,
                        void* dy_rows, float* dgates, const int32_t* padded_offsets,
                        const int32_t* expert_counts, int E, int align, void* stream);

/* out[t] = sum_s w[t,s] * rows[row_of(t,s)] (+ dz[t] @ w_g^T when dz != NULL)
 * with w = gates (or 1 when gates == NULL); tokens with no kept pair get 0.
 * w_gT is the TRANSPOSED gating matrix [E, H] fp32.  accumulate: out += ...
 *                       -- dispatcher.py:145-157 (fwd), :467-468,490 (bwd) */
B200MOE_API int b200moe_combine(const void* rows, int dtype, int64_t T, int64_t H, int k,
                    const int32_t* pair_row, const float* gates, const float* dz,
                    const float* w_gT, int E, void* out, int out_dtype, int accumulate,
                    void* stream);
/* b200moe_combine (bf16) over ETP partial rows: rows r of the combine are
 * bf16(sum over p = 0..nparts-1 ascending, fp32, of parts[p * part_stride +
 * r * H ..]) -- the ETP reduce-scatter fold (dispatcher.py:349-361,
 * collectives.py:386-388; b200moe_ep_reduce_parts) fused into the
 * combine's row loads.  rows_out (nullable, [rows, H] bf16, forward only)
 * receives every reduced pair row (the forward's saved y_perm,
 * dispatcher.py:374).  With dz (backward): E <= 8, no gates. */
B200MOE_API int b200moe_combine_parts(const void* parts, int nparts, int64_t part_stride, void* rows_out,
                                      int64_t T, int64_t H, int k, const int32_t* pair_row,
                                      const float* gates, const float* dz, const float* w_gT, int E,
                                      void* out, int accumulate, void* stream);

/* ------------------------------------------------------------ expert GEMM */

/* Grouped GEMM, fp32 accumulation:  C_g = A_g · B_g  for g < G.
 *   A(m,k) = A[(m_base+m)*a_sm + (k_base+k)*a_sk]
 *   B(k,n) = B[b_group*b_sg + (k_base+k)*b_sk + n*b_sn]
 *   C(m,n) = C[c_group*c_sg + (m_base+m)*ldc + n]
 * grouped_dim = 0 ("M"): m_base = group_off[g], M_g = group_off[g+1]-group_off[g],
 *   k_base = 0, K fixed, b_group = group_expert[g] (identity when NULL), c_group = 0.
 * grouped_dim = 1 ("K"): k_base = group_off[g], K_g likewise, m_base = 0,
 *   M fixed, b_group = 0, c_group = g.
 * group_off is a DEVICE array [G+1]; group sizes never leave the device. */
typedef struct {
  int dtype_in;      /* B200MOE_F32 | B200MOE_BF16 (A and B) */
  int dtype_out;     /* B200MOE_F32 | B200MOE_BF16 */
  int grouped_dim;   /* 0 = M, 1 = K */
  int accumulate;    /* C += A·B (fp32 out only) */
  int G;
  int64_t M, N, K;   /* the fixed extents (M ignored for grouped M, K for grouped K) */
  const void* A; int64_t a_sm, a_sk;
  const void* B; int64_t b_sg, b_sk, b_sn;
  void* C; int64_t c_sg, ldc;
  const int32_t* group_off;
  const int32_t* group_expert;
  int64_t max_rows;  /* upper bound of group_off[G] (buffer capacity) */
  int dtype_b;       /* dtype of B (may differ from A's dtype_in) */
  const int32_t* group_end; /* nullable: group g = [group_off[g], group_end[g]) (gaps allowed) */
} b200moe_gemm_args;

/* Portable SIMT implementation (fp32 parity mode and cross-check) of the
 * expert GEMMs, experts.py:130-172 batched over groups. */
B200MOE_API int b200moe_gemm_simt(const b200moe_gemm_args* args, void* stream);

/* Tensor-core grouped GEMM (tcgen05 + TMEM + TMA, bf16 in, fp32 accumulate):
 * the expert FFN GEMMs of experts.py:130-172 batched over groups,
 * with fused expert epilogues.  Operands:
 *   A K-major  [a_rows, lda]      (row = token, K contiguous)
 *   A MN-major [a_rows, lda]      (row = K index = token, M contiguous; grouped K)
 *   B K-major  [b_batch, N, ldb]  (weights, K contiguous)
 *   B MN-major [b_batch, K, ldb]  (N contiguous); grouped K: [a_rows, ldb]
 * grouped_dim 0 (M): group g owns rows [group_off[g], group_off[g+1]) of A and
 *   C, uses weight batch group_expert[g] (identity when NULL).
 * grouped_dim 1 (K): group g reduces over rows [group_off[g], group_off[g+1])
 *   (multiples of 64), C_g = C + g*c_sg.
 * epilogue: 0 store (bf16/fp32, accumulate), 1 SwiGLU fwd (C=pre, H=h),
 *   2 SwiGLU bwd (acc=dh [.,N=F], PRE=pre, C=dpre), 3 act fwd, 4 act bwd,
 *   5 scatter to peers (see row_origin).
 * num_ctas: persistent grid size (<= 0: one CTA per SM). */
typedef struct {
  int G;
  int grouped_dim;
  int64_t M, N, K;
  const void* A; int a_major; int64_t lda; int64_t a_rows;
  const void* B; int b_major; int64_t ldb; int64_t b_batch; int64_t b_batch_stride;
  void* C; int64_t ldc; int64_t c_sg; int out_dtype; int accumulate;
  const int32_t* group_off;
  const int32_t* group_expert;
  int epilogue; int act;
  void* H; int64_t ldh;
  const void* PRE; int64_t ldpre;
  int num_ctas;
  const int32_t* group_end; /* nullable: group g = [group_off[g], group_end[g]) (gaps allowed) */
  /* epilogue 5 (scatter, bf16, grouped M): C is not written; row r goes to
   * peer_base[row_origin[2r]] + scatter_off + row_origin[2r+1] * ldc * 2 (a
   * peer's buffer over NVLink, or this rank's); rows with row_origin[2r] < 0
   * are skipped.  Replaces the return all_to_all_v of dispatcher.py:355-361
   * (and :462-466 backward), overlapped with the GEMM. */
  const int32_t* row_origin; const uint64_t* peer_base; int64_t scatter_off;
  /* glu_f > 0 (grouped K, fp32 store, M = 2 glu_f): the M rows are packed
   * SwiGLU rows ([32 gate | 32 up] per 64) and are stored de-interleaved as
   * [gate rows | up rows], i.e. C_g^T is the reference's [H, 2F] = [gate | up]
   * dW1 layout (experts.py:168) without a copy. */
  int64_t glu_f;
} b200moe_tc_gemm_args;

B200MOE_API int b200moe_gemm_tc(const b200moe_tc_gemm_args* args, void* stream);

/* ------------------------------------- EP all-to-all over NVLink peer memory
 * Device-side replacement of all_to_all_v + exchange_meta + the grp_order
 * regroup, and of the ETP all-gather-v / reduce-scatter-v
 * (dispatcher.py:309-362, 425-468).  The exchange group is the EP x ETP block
 * of ranks, member m = ep_idx * etp + etp_idx; peer_base[ep*etp] (device
 * array) holds the base address of the same symmetric buffer on every
 * member; regions are addressed by byte offsets.  No call synchronises the
 * host. */

/* row `me` of every member's [members, E] int32 count matrix := counts[E];
 * when *status (nullable) is non-zero -- this rank's step already failed --
 * an abort marker (-1 entries) instead, so that the whole group fails the
 * step together (every rank still completes its barriers and raises). */
B200MOE_API int b200moe_ep_counts_push(const int32_t* counts, int me, int members, int E,
                                       const uint64_t* peer_base, int64_t cnt_off, const int32_t* status,
                                       void* stream);
/* cross-GPU barrier over the members: flag exchange at flag_off with
 * system-scope release/acquire; epoch must increase by one per call (bounded
 * spin, traps if a peer never arrives). */
B200MOE_API int b200moe_ep_barrier(const uint64_t* peer_base, int64_t flag_off, int me, int members,
                                   uint32_t epoch, void* stream);
/* from this rank's copy of the count matrix: seg_off[ep*L] (first row of
 * (me, le) in EP index d's receive buffers -- the same on its etp members),
 * goff[L+1] / gcount[L] (this rank's GEMM groups: one per local expert,
 * senders contiguous in member order, the group padded to align rows).
 * Marker rows count as empty and set bit 1 of *status (nullable).  A layout
 * that exceeds cap_rows sets bit 4 (this rank's groups become empty) or,
 * without a status word, traps. */
B200MOE_API int b200moe_ep_layout(const int32_t* cnt_local, int me, int ep, int etp, int L, int align,
                                  int64_t cap_rows, int32_t* seg_off, int32_t* goff, int32_t* gcount,
                                  int32_t* status, void* stream);
/* zero the pad rows of this rank's receive buffer (bf16 [rows, H]); with
 * origin (int32 [rows, 2]) also mark them "no origin" for the scatter epilogue */
B200MOE_API int b200moe_ep_zero_pads(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount,
                                     int G, int align, int32_t* origin, void* stream);
/* fused permute + push: x[t] (bwd: gates*u[t]) -> row rr = seg_off[d,le] +
 * (gemm_row - poff[e]) of the buffers at dst_off of all etp members of EP
 * index d = e / L.  Forward also writes (me, gemm_row) into their int32
 * [rows, 2] origin tables at origin_off, so their GEMM epilogues
 * (b200moe_gemm_tc epilogue 5) return the expert outputs straight to this
 * rank's padded layout.  Backward reads the returned (ETP-reduced) rows
 * (y_rows, local, padded layout) for dgates = <u[t], y>.  dup_off >= 0: the
 * pairs of a token bound for the same EP index send the row once; the others
 * record their leader row in the receivers' int32 [rows, 2] dup tables at
 * dup_off, resolved by b200moe_ep_expand after the barrier (dup_off < 0: every
 * pair pushes its own row).  Nothing is pushed when *status (nullable) is
 * non-zero (a failed step). */
B200MOE_API int b200moe_ep_dispatch(const void* x, int64_t T, int64_t H, int k, int L,
                                    const int32_t* topk_idx, const int32_t* gemm_row,
                                    const int32_t* poff, const int32_t* seg_off,
                                    const uint64_t* peer_base, int me, int etp, int64_t dst_off,
                                    int64_t origin_off, int64_t dup_off, const void* y_rows,
                                    const float* gates, float* dgates, int bwd, const int32_t* status,
                                    void* stream);
/* b200moe_ep_dispatch split in two for overlapping the exchange with the
 * first expert GEMM: part 1 performs only the stores into this rank's own
 * buffers (the rows its experts take from itself), part 2 only those into
 * the other members' (NVLink); part 0 = both (b200moe_ep_dispatch).  Each
 * pair's dgate (backward) is written by exactly one part: part 1 for pairs
 * routed to this rank's EP index, part 2 for the rest.  Part 2 launches one
 * small block per SM whose register budget fits beside a resident
 * b200moe_gemm_tc CTA, so it runs concurrently with a GEMM on another
 * stream. */
B200MOE_API int b200moe_ep_dispatch_part(const void* x, int64_t T, int64_t H, int k, int L,
                                         const int32_t* topk_idx, const int32_t* gemm_row,
                                         const int32_t* poff, const int32_t* seg_off,
                                         const uint64_t* peer_base, int me, int etp, int64_t dst_off,
                                         int64_t origin_off, int64_t dup_off, const void* y_rows,
                                         const float* gates, float* dgates, int bwd, int part,
                                         const int32_t* status, void* stream);
/* GEMM groups of the split first GEMM, from the layout of b200moe_ep_layout:
 * per local expert, the rows this rank sent itself (available before the
 * barrier) and the rest (two groups: before and after them, pads included).
 * split (int32, 8L + 2) = loc_off[L+1] | loc_end[L] | rem_off[2L+1] |
 * rem_end[2L] | rem_exp[2L] -- b200moe_gemm_tc group_off / group_end /
 * group_expert arrays; loc_off[L] = rem_off[2L] = goff[L]. */
B200MOE_API int b200moe_ep_split_groups(const int32_t* cnt_local, int me, int ep, int etp, int L,
                                        const int32_t* seg_off, const int32_t* goff, const int32_t* gcount,
                                        int32_t* split, void* stream);
/* Receiver side of the deduplicated push (dispatcher.py:317-323's regroup
 * has no counterpart: the reference moves every pair): over the real rows
 * goff[g] .. goff[g] + gcount[g] of the bf16 [rows, H] receive buffer, with
 * the dup table written by the senders: phase 0 (forward) copies leader rows
 * into their duplicates; phase 1 (backward) writes bf16(gate * leader) into
 * the duplicates; phase 2 scales the raw leaders in place. */
B200MOE_API int b200moe_ep_expand(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount,
                                  int G, const int32_t* dup, int phase, void* stream);
/* out[i] = bf16(sum over p ascending of parts[p * part_stride + i]), fp32
 * accumulation: the ETP reduce of the members' partial expert outputs that
 * their scatter epilogues returned (collectives.py:386-388 fold order). */
B200MOE_API int b200moe_ep_reduce_parts(const void* parts, int nparts, int64_t part_stride, int64_t n,
                                        void* out, void* stream);

/* Elementwise expert activations (experts.py:23-37) in the padded row layout, rows < group_off[G].
 * SwiGLU layout: pre has 2F columns, 64-column blocks of [32 gate | 32 up]. */
B200MOE_API int b200moe_act_fwd(const void* pre, int dtype, int act, const int32_t* group_off, int G,
                    int64_t max_rows, int64_t F, void* h, void* stream);
B200MOE_API int b200moe_act_bwd(const void* dh, const void* pre, int dtype, int act, const int32_t* group_off,
                    int G, int64_t max_rows, int64_t F, void* dpre, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200MOE_H_ */
