// extern "C" entry points of libb200moe.so: argument validation, error
// reporting, dispatch to the kernels.  See include/b200moe.h.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace b200moe {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// kernels (defined in the other translation units)
int router_logits(const void*, int, const float*, int64_t, int64_t, int, float*, cudaStream_t);
int router_topk(const float*, int64_t, int, int, int, int, float*, int32_t*, float*, double*,
                int32_t*, cudaStream_t);
int router_fwd_tc_np(int);
int router_fwd_tc(const void*, int64_t, int64_t, const void*, int, int, int, int, float*, float*,
                  int32_t*, float*, double*, int32_t*, cudaStream_t);
size_t plan_ws_bytes(int64_t, int);
int fullseq_capacity(const int64_t*, const int64_t*, int64_t, int64_t, uint8_t*, const int64_t*, int,
                     int32_t*, cudaStream_t);
int dispatch_plan(const int32_t*, const float*, const uint8_t*, const int32_t*, int64_t, int, int,
                  int64_t, int, void*, uint8_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*,
                  int64_t*, float*, cudaStream_t);
int capacity_by_gate(const int64_t*, const int32_t*, const double*, const int64_t*, int64_t, int,
                     int, int64_t, uint8_t*, cudaStream_t);
int router_bwd(const float*, const float*, const int32_t*, const float*, int64_t, int, int, int,
               int, float*, void*, int, int, cudaStream_t);
int router_parts_layout(int, int*, int*);
size_t router_wgrad_tc_ws_bytes(int64_t, int64_t, int);
int router_wgrad_tc(const void*, const void*, int64_t, int64_t, int, float*, void*, size_t, cudaStream_t);
size_t router_wgrad_ws_bytes(int64_t, int64_t, int);
int router_wgrad(const void*, int, const float*, int64_t, int64_t, int, float*, void*, cudaStream_t);
int permute(const void*, int, int64_t, int64_t, int, const int32_t*, const float*, void*,
            const int32_t*, const int32_t*, int, int64_t, cudaStream_t);
int permute_bwd(const void*, int, int64_t, int64_t, int, const int32_t*, const float*, const void*,
                void*, float*, const int32_t*, const int32_t*, int, int64_t, cudaStream_t);
int combine(const void*, int, int64_t, int64_t, int, const int32_t*, const float*, const float*,
            const float*, int, void*, int, int, cudaStream_t);
int gemm_simt(const b200moe_gemm_args*, cudaStream_t);
int gemm_tc(const b200moe_tc_gemm_args*, cudaStream_t);
int ep_barrier(const uint64_t*, int64_t, int, int, uint32_t, cudaStream_t);
int ep_counts_push(const int32_t*, int, int, int, const uint64_t*, int64_t, const int32_t*, cudaStream_t);
int ep_layout(const int32_t*, int, int, int, int, int, int64_t, int32_t*, int32_t*, int32_t*, int32_t*,
              cudaStream_t);
int ep_reduce_parts(const void*, int, int64_t, int64_t, void*, cudaStream_t);
int ep_zero_pads(void*, int64_t, const int32_t*, const int32_t*, int, int, int32_t*, cudaStream_t);
int ep_dispatch(const void*, int64_t, int64_t, int, int, const int32_t*, const int32_t*,
                const int32_t*, const int32_t*, const uint64_t*, int, int, int64_t, int64_t, int64_t,
                const void*, const float*, float*, int, int, const int32_t*, cudaStream_t);
int combine_parts(const void*, int, int64_t, void*, int64_t, int64_t, int, const int32_t*, const float*,
                  const float*, const float*, int, void*, int, cudaStream_t);
int ep_split_groups(const int32_t*, int, int, int, int, const int32_t*, const int32_t*, const int32_t*,
                    int32_t*, cudaStream_t);
int ep_expand(void*, int64_t, const int32_t*, const int32_t*, int, const void*, int, cudaStream_t);
int split_bf16x3(const float*, int64_t, int, void*, void*, cudaStream_t);
size_t router_stats_ws_bytes(int64_t, int);
int router_stats(const int32_t*, const uint8_t*, const float*, int64_t, int, int, int64_t*, int64_t*,
                 double*, void*, cudaStream_t);
int sum_parts(const float*, int64_t, int64_t, int, float*, cudaStream_t);
int act_fwd(const void*, int, int, const int32_t*, int, int64_t, int64_t, void*, cudaStream_t);
int act_bwd(const void*, const void*, int, int, const int32_t*, int, int64_t, int64_t, void*,
            cudaStream_t);

}  // namespace b200moe

using namespace b200moe;

#define REQUIRE(cond, ...)          \
  do {                              \
    if (!(cond)) {                  \
      set_error(__VA_ARGS__);       \
      return B200MOE_EINVAL;        \
    }                               \
  } while (0)

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
static inline bool dt_ok(int d) { return d == B200MOE_F32 || d == B200MOE_BF16; }

extern "C" {

const char* b200moe_version(void) { return "b200moe 0.1.0 (sm_100a)"; }
const char* b200moe_last_error(void) { return g_err; }

int b200moe_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    set_error("no CUDA device");
    return B200MOE_ENODEV;
  }
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    set_error("device %d is sm_%d%d; this library is built for sm_100a only", dev, major, minor);
    return B200MOE_ENODEV;
  }
  return B200MOE_OK;
}

int b200moe_router_logits(const void* x, int x_dtype, const float* w_g, int64_t T, int64_t H, int E,
                          float* logits, void* stream) {
  REQUIRE(dt_ok(x_dtype), "router_logits: bad dtype %d", x_dtype);
  REQUIRE(T >= 0 && H >= 1 && E >= 1, "router_logits: bad shape T=%lld H=%lld E=%d", (long long)T,
          (long long)H, E);
  if (T == 0) return B200MOE_OK;
  REQUIRE(x && w_g && logits, "router_logits: null pointer");
  return router_logits(x, x_dtype, w_g, T, H, E, logits, S(stream));
}

int b200moe_router_topk(const float* logits, int64_t T, int E, int k, int gate_fn, int renorm,
                        float* scores, int32_t* topk_idx, float* gates, double* gates_f64,
                        int32_t* status, void* stream) {
  REQUIRE(E >= 1 && k >= 1 && k <= E, "1<=k<=E violated (k=%d, E=%d)", k, E);
  REQUIRE(k <= 32, "router_topk: k=%d > 32 unsupported", k);
  REQUIRE(gate_fn == B200MOE_GATE_SOFTMAX || gate_fn == B200MOE_GATE_SIGMOID,
          "unknown gate_fn %d", gate_fn);
  if (T == 0) return B200MOE_OK;
  REQUIRE(logits && scores && topk_idx && gates, "router_topk: null pointer");
  return router_topk(logits, T, E, k, gate_fn, renorm, scores, topk_idx, gates, gates_f64, status,
                     S(stream));
}

int b200moe_router_fwd_tc_np(int E) { return router_fwd_tc_np(E); }

int b200moe_router_fwd_tc(const void* x, int64_t T, int64_t H, const void* w_parts, int E, int k,
                          int gate_fn, int renorm, float* logits, float* scores, int32_t* topk_idx,
                          float* gates, double* gates_f64, int32_t* status, void* stream) {
  REQUIRE(E >= 1 && k >= 1 && k <= E, "1<=k<=E violated (k=%d, E=%d)", k, E);
  REQUIRE(router_fwd_tc_np(E) > 0, "router_fwd_tc: E=%d > 64 unsupported", E);
  REQUIRE(k <= 32, "router_fwd_tc: k=%d > 32 unsupported", k);
  REQUIRE(gate_fn == B200MOE_GATE_SOFTMAX || gate_fn == B200MOE_GATE_SIGMOID,
          "unknown gate_fn %d", gate_fn);
  REQUIRE(T >= 0 && H >= 64 && H % 8 == 0, "router_fwd_tc: bad shape T=%lld H=%lld", (long long)T,
          (long long)H);
  if (T == 0) return B200MOE_OK;
  REQUIRE(x && w_parts && logits && scores && topk_idx && gates && status,
          "router_fwd_tc: null pointer");
  REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)w_parts & 15) == 0, "router_fwd_tc: misaligned operand");
  return router_fwd_tc(x, T, H, w_parts, E, k, gate_fn, renorm, logits, scores, topk_idx, gates,
                       gates_f64, status, S(stream));
}

int b200moe_enable_peer_access(int peer) {
  int dev = 0, can = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess) {
    cudaGetLastError();
    set_error("enable_peer_access: cannot query device %d -> %d", dev, peer);
    return B200MOE_ENODEV;
  }
  if (!can) {
    set_error("enable_peer_access: device %d cannot access device %d", dev, peer);
    return B200MOE_EUNSUPPORTED;
  }
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
    set_error("enable_peer_access: %s", cudaGetErrorString(e));
    return B200MOE_ELAUNCH;
  }
  cudaGetLastError();  // clear "already enabled"
  return B200MOE_OK;
}

size_t b200moe_dispatch_plan_ws(int64_t T, int E) { return plan_ws_bytes(T, E); }

int b200moe_dispatch_plan(const int32_t* topk_idx, const float* gates, const uint8_t* kept_in,
                          const int32_t* order, int64_t T, int k, int E, int64_t cap, int align,
                          void* workspace, size_t workspace_bytes, uint8_t* kept_out,
                          int32_t* expert_counts, int32_t* expert_offsets, int32_t* padded_offsets,
                          int32_t* send_row, int32_t* gemm_row, int64_t* perm, float* perm_gates,
                          void* stream) {
  REQUIRE(E >= 1 && E <= 4096 && k >= 1 && k <= 16 && k <= E, "dispatch_plan: bad E=%d k=%d", E, k);
  REQUIRE(align != 0, "dispatch_plan: align must be non-zero");
  REQUIRE(align > 0 || (cap > 0 && cap <= -(int64_t)align),
          "dispatch_plan: pad-to-capacity (align < 0) needs 0 < cap <= -align");
  REQUIRE(T >= 0 && T * k < (int64_t)INT32_MAX, "dispatch_plan: T*k must fit int32");
  REQUIRE(workspace_bytes >= plan_ws_bytes(T, E), "dispatch_plan: workspace too small");
  REQUIRE(expert_counts && expert_offsets && padded_offsets && workspace,
          "dispatch_plan: null pointer");
  if (T > 0) REQUIRE(topk_idx && kept_out && send_row && gemm_row && perm, "dispatch_plan: null pointer");
  REQUIRE(T == 0 || !perm_gates || gates, "dispatch_plan: perm_gates needs gates");
  return dispatch_plan(topk_idx, gates, kept_in, order, T, k, E, cap, align, workspace, kept_out,
                       expert_counts, expert_offsets, padded_offsets, send_row, gemm_row, perm,
                       perm_gates, S(stream));
}

int b200moe_capacity_by_gate(const int64_t* perm0, const int32_t* offsets0, const double* gates_f64,
                             const int64_t* positions, int64_t T, int k, int E, int64_t cap,
                             uint8_t* kept_out, void* stream) {
  REQUIRE(cap >= 1, "capacity_by_gate: cap must be >= 1");
  REQUIRE(E >= 1 && k >= 1, "capacity_by_gate: bad E/k");
  if (T == 0) return B200MOE_OK;
  REQUIRE(perm0 && offsets0 && gates_f64 && kept_out, "capacity_by_gate: null pointer");
  return capacity_by_gate(perm0, offsets0, gates_f64, positions, T, k, E, cap, kept_out, S(stream));
}

int b200moe_router_bwd(const float* dgates, const float* scores, const int32_t* topk_idx,
                       const float* gates, int64_t T, int E, int k, int gate_fn, int renorm,
                       float* dz, void* dz_parts, void* stream) {
  REQUIRE(E >= 1 && k >= 1 && k <= E, "router_bwd: bad E=%d k=%d", E, k);
  int epw = 0, nb = 0;
  REQUIRE(!dz_parts || router_parts_layout(E, &epw, &nb), "router_bwd: dz parts need E <= 64 (E=%d)", E);
  if (T == 0) return B200MOE_OK;
  REQUIRE(dgates && scores && topk_idx && gates && dz, "router_bwd: null pointer");
  return router_bwd(dgates, scores, topk_idx, gates, T, E, k, gate_fn, renorm, dz, dz_parts, epw, nb,
                    S(stream));
}

int b200moe_fullseq_capacity(const int64_t* seg_sorted, const int64_t* order, int64_t N, int64_t cap,
                             uint8_t* kept_slot, const int64_t* pos_by_pos, int k, int32_t* status,
                             void* stream) {
  REQUIRE(N >= 0 && cap >= 0 && k >= 1, "fullseq_capacity: bad args");
  if (N == 0) return B200MOE_OK;
  REQUIRE(seg_sorted && order && kept_slot, "fullseq_capacity: null pointer");
  return fullseq_capacity(seg_sorted, order, N, cap, kept_slot, pos_by_pos, k, status, S(stream));
}

int b200moe_router_parts_cols(int E) {
  int epw = 0, nb = 0;
  return router_parts_layout(E, &epw, &nb) ? nb : 0;
}

size_t b200moe_router_wgrad_tc_ws(int64_t T, int64_t H, int E) { return router_wgrad_tc_ws_bytes(T, H, E); }

int b200moe_router_wgrad_tc(const void* x, const void* dz_parts, int64_t T, int64_t H, int E, float* dw_g,
                            void* workspace, size_t workspace_bytes, void* stream) {
  int epw = 0, nb = 0;
  REQUIRE(router_parts_layout(E, &epw, &nb), "router_wgrad_tc: E=%d > 64 unsupported", E);
  REQUIRE(T >= 0 && H >= 128 && H % 64 == 0, "router_wgrad_tc: H=%lld must be a multiple of 64 (>= 128)",
          (long long)H);
  REQUIRE(dw_g && (T == 0 || (x && dz_parts && workspace)), "router_wgrad_tc: null pointer");
  REQUIRE(workspace_bytes >= router_wgrad_tc_ws_bytes(T, H, E), "router_wgrad_tc: workspace too small");
  return router_wgrad_tc(x, dz_parts, T, H, E, dw_g, workspace, workspace_bytes, S(stream));
}

size_t b200moe_router_wgrad_ws(int64_t T, int64_t H, int E) { return router_wgrad_ws_bytes(T, H, E); }

int b200moe_router_wgrad(const void* x, int x_dtype, const float* dz, int64_t T, int64_t H, int E,
                         float* dw_g, void* workspace, size_t workspace_bytes, void* stream) {
  REQUIRE(dt_ok(x_dtype) && H >= 1 && E >= 1 && T >= 0, "router_wgrad: bad args");
  REQUIRE(dw_g, "router_wgrad: null pointer");
  if (T == 0) return cudaMemsetAsync(dw_g, 0, H * E * sizeof(float), S(stream)) == cudaSuccess
                         ? B200MOE_OK : B200MOE_ELAUNCH;
  REQUIRE(x && dz && workspace, "router_wgrad: null pointer");
  REQUIRE(workspace_bytes >= router_wgrad_ws_bytes(T, H, E), "router_wgrad: workspace too small");
  return router_wgrad(x, x_dtype, dz, T, H, E, dw_g, workspace, S(stream));
}

int b200moe_permute(const void* x, int dtype, int64_t T, int64_t H, int k, const int32_t* pair_row,
                    const float* scale, void* out, const int32_t* padded_offsets,
                    const int32_t* expert_counts, int E, int align, void* stream) {
  REQUIRE(dt_ok(dtype) && H >= 1 && k >= 1 && T >= 0, "permute: bad args");
  REQUIRE(out, "permute: null output");
  if (T > 0) REQUIRE(x && pair_row, "permute: null pointer");
  // align > 0: at most align-1 pad rows per segment; align < 0: fixed segments
  // of -align rows (pad-to-capacity), up to -align pad rows
  const int64_t max_pad = (padded_offsets && expert_counts) ? (align > 1 ? align - 1 : (align < 0 ? -(int64_t)align : 0)) : 0;
  return permute(x, dtype, T, H, k, pair_row, scale, out, padded_offsets, expert_counts, E,
                 max_pad, S(stream));
}

int b200moe_permute_bwd(const void* u, int dtype, int64_t T, int64_t H, int k,
                        const int32_t* pair_row, const float* gates, const void* y_rows,
                        void* dy_rows, float* dgates, const int32_t* padded_offsets,
                        const int32_t* expert_counts, int E, int align, void* stream) {
  REQUIRE(dt_ok(dtype) && H >= 1 && k >= 1 && T >= 0, "permute_bwd: bad args");
  if (T > 0) REQUIRE(u && pair_row && gates && y_rows && dy_rows && dgates, "permute_bwd: null pointer");
  // align > 0: at most align-1 pad rows per segment; align < 0: fixed segments
  // of -align rows (pad-to-capacity), up to -align pad rows
  const int64_t max_pad = (padded_offsets && expert_counts) ? (align > 1 ? align - 1 : (align < 0 ? -(int64_t)align : 0)) : 0;
  return permute_bwd(u, dtype, T, H, k, pair_row, gates, y_rows, dy_rows, dgates, padded_offsets,
                     expert_counts, E, max_pad, S(stream));
}

int b200moe_combine(const void* rows, int dtype, int64_t T, int64_t H, int k,
                    const int32_t* pair_row, const float* gates, const float* dz,
                    const float* w_gT, int E, void* out, int out_dtype, int accumulate,
                    void* stream) {
  REQUIRE(dt_ok(dtype) && dt_ok(out_dtype) && H >= 1 && k >= 1 && T >= 0, "combine: bad args");
  REQUIRE(!dz || (w_gT && E >= 1), "combine: dz needs w_gT and E");
  if (T > 0) REQUIRE(rows && pair_row && out, "combine: null pointer");
  return combine(rows, dtype, T, H, k, pair_row, gates, dz, w_gT, E, out, out_dtype, accumulate,
                 S(stream));
}

int b200moe_combine_parts(const void* parts, int nparts, int64_t part_stride, void* rows_out, int64_t T,
                          int64_t H, int k, const int32_t* pair_row, const float* gates, const float* dz,
                          const float* w_gT, int E, void* out, int accumulate, void* stream) {
  REQUIRE(nparts >= 1 && nparts <= 32 && part_stride >= 0 && H % 8 == 0 && k >= 1 && k <= 8 && T >= 0,
          "combine_parts: 1 <= nparts <= 32, H %% 8 == 0, 1 <= k <= 8 required");
  REQUIRE(!dz || (w_gT && E >= 1 && E <= 8 && !gates), "combine_parts: dz needs w_gT, E <= 8 and no gates");
  REQUIRE(!rows_out || !dz, "combine_parts: rows_out only without dz");
  if (T > 0) REQUIRE(parts && pair_row && out, "combine_parts: null pointer");
  if (T == 0) return B200MOE_OK;
  return combine_parts(parts, nparts, part_stride, rows_out, T, H, k, pair_row, gates, dz, w_gT, E, out,
                       accumulate, S(stream));
}

int b200moe_gemm_simt(const b200moe_gemm_args* a, void* stream) {
  REQUIRE(a, "gemm_simt: null args");
  REQUIRE(dt_ok(a->dtype_in) && dt_ok(a->dtype_out) && dt_ok(a->dtype_b), "gemm_simt: bad dtype");
  REQUIRE(a->grouped_dim == 0 || a->grouped_dim == 1, "gemm_simt: bad grouped_dim");
  REQUIRE(a->G >= 1 && a->N >= 1, "gemm_simt: bad G/N");
  REQUIRE(a->A && a->B && a->C && a->group_off, "gemm_simt: null pointer");
  if (a->grouped_dim == 0) REQUIRE(a->K >= 1 && a->max_rows >= 0, "gemm_simt: bad K/max_rows");
  else REQUIRE(a->M >= 1, "gemm_simt: bad M");
  return gemm_simt(a, S(stream));
}

int b200moe_gemm_tc(const b200moe_tc_gemm_args* a, void* stream) {
  REQUIRE(a, "gemm_tc: null args");
  REQUIRE(a->grouped_dim == 0 || a->grouped_dim == 1, "gemm_tc: bad grouped_dim");
  REQUIRE(a->N >= 1 && a->a_rows >= 0 && a->b_batch >= 1, "gemm_tc: bad shape");
  REQUIRE(a->grouped_dim == 1 || a->K >= 1, "gemm_tc: bad K");
  REQUIRE(a->grouped_dim == 0 || a->M >= 1, "gemm_tc: bad M");
  REQUIRE(a->A && a->B && (a->C || a->epilogue == 5) && a->group_off, "gemm_tc: null pointer");
  REQUIRE(a->epilogue >= 0 && a->epilogue <= 5, "gemm_tc: bad epilogue %d", a->epilogue);
  REQUIRE(a->epilogue != 5 || (a->row_origin && a->peer_base), "gemm_tc: scatter needs row_origin, peer_base");
  REQUIRE(a->epilogue == 0 || a->grouped_dim == 0, "gemm_tc: fused epilogues need grouped M");
  REQUIRE(a->epilogue == 0 || a->out_dtype == B200MOE_BF16, "gemm_tc: fused epilogues write bf16");
  REQUIRE(!a->accumulate || a->epilogue == 0, "gemm_tc: accumulate only with the plain store epilogue");
  REQUIRE((a->epilogue != 1 && a->epilogue != 3) || a->H, "gemm_tc: epilogue needs H");
  REQUIRE((a->epilogue != 2 && a->epilogue != 4) || a->PRE, "gemm_tc: epilogue needs PRE");
  REQUIRE(a->epilogue != 1 || a->N % 64 == 0, "gemm_tc: SwiGLU fwd needs N %% 64 == 0");
  REQUIRE(a->epilogue != 2 || a->N % 32 == 0, "gemm_tc: SwiGLU bwd needs N %% 32 == 0");
  if (a->a_rows == 0) return B200MOE_OK;
  return gemm_tc(a, S(stream));
}

int b200moe_ep_counts_push(const int32_t* counts, int me, int ep, int E, const uint64_t* peer_base,
                           int64_t cnt_off, const int32_t* status, void* stream) {
  REQUIRE(counts && peer_base && ep >= 1 && ep <= 32 && me >= 0 && me < ep && E >= 1,
          "ep_counts_push: bad args");
  return ep_counts_push(counts, me, ep, E, peer_base, cnt_off, status, S(stream));
}

int b200moe_ep_barrier(const uint64_t* peer_base, int64_t flag_off, int me, int ep, uint32_t epoch,
                       void* stream) {
  REQUIRE(peer_base && ep >= 1 && ep <= 32 && me >= 0 && me < ep, "ep_barrier: bad args");
  return ep_barrier(peer_base, flag_off, me, ep, epoch, S(stream));
}

int b200moe_ep_layout(const int32_t* cnt_local, int me, int ep, int etp, int L, int align, int64_t cap_rows,
                      int32_t* seg_off, int32_t* goff, int32_t* gcount, int32_t* status, void* stream) {
  REQUIRE(cnt_local && seg_off && goff && gcount && ep >= 1 && etp >= 1 && ep * etp <= 32 && L >= 1 &&
              align >= 1 && me >= 0 && me < ep * etp && cap_rows >= 0 && cap_rows < (1ll << 31),
          "ep_layout: bad args");
  return ep_layout(cnt_local, me, ep, etp, L, align, cap_rows, seg_off, goff, gcount, status, S(stream));
}

int b200moe_ep_zero_pads(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount, int G,
                         int align, int32_t* origin, void* stream) {
  REQUIRE(buf && goff && gcount && H >= 1, "ep_zero_pads: bad args");
  return ep_zero_pads(buf, H, goff, gcount, G, align, origin, S(stream));
}

int b200moe_ep_dispatch_part(const void* x, int64_t T, int64_t H, int k, int L, const int32_t* topk_idx,
                             const int32_t* gemm_row, const int32_t* poff, const int32_t* seg_off,
                             const uint64_t* peer_base, int me, int etp, int64_t dst_off,
                             int64_t origin_off, int64_t dup_off, const void* y_rows, const float* gates,
                             float* dgates, int bwd, int part, const int32_t* status, void* stream) {
  REQUIRE(H % 8 == 0 && k >= 1 && L >= 1 && me >= 0 && etp >= 1 && etp <= 32 && part >= 0 && part <= 2,
          "ep_dispatch: H %% 8, k >= 1, me >= 0, 1 <= etp <= 32, part in [0, 2] required");
  if (T == 0) return B200MOE_OK;
  REQUIRE(x && topk_idx && gemm_row && poff && seg_off && peer_base, "ep_dispatch: null pointer");
  REQUIRE(!bwd || (gates && dgates && y_rows), "ep_dispatch: backward needs gates, dgates, y_rows");
  return ep_dispatch(x, T, H, k, L, topk_idx, gemm_row, poff, seg_off, peer_base, me, etp, dst_off,
                     origin_off, dup_off, y_rows, gates, dgates, bwd, part, status, S(stream));
}

int b200moe_ep_dispatch(const void* x, int64_t T, int64_t H, int k, int L, const int32_t* topk_idx,
                        const int32_t* gemm_row, const int32_t* poff, const int32_t* seg_off,
                        const uint64_t* peer_base, int me, int etp, int64_t dst_off, int64_t origin_off,
                        int64_t dup_off, const void* y_rows, const float* gates, float* dgates, int bwd,
                        const int32_t* status, void* stream) {
  return b200moe_ep_dispatch_part(x, T, H, k, L, topk_idx, gemm_row, poff, seg_off, peer_base, me, etp,
                                  dst_off, origin_off, dup_off, y_rows, gates, dgates, bwd, 0, status,
                                  stream);
}

int b200moe_ep_split_groups(const int32_t* cnt_local, int me, int ep, int etp, int L, const int32_t* seg_off,
                            const int32_t* goff, const int32_t* gcount, int32_t* split, void* stream) {
  REQUIRE(cnt_local && seg_off && goff && gcount && split && ep >= 1 && etp >= 1 && ep * etp <= 32 &&
              L >= 1 && me >= 0 && me < ep * etp,
          "ep_split_groups: bad args");
  return ep_split_groups(cnt_local, me, ep, etp, L, seg_off, goff, gcount, split, S(stream));
}

int b200moe_ep_expand(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount, int G,
                      const int32_t* dup, int phase, void* stream) {
  REQUIRE(buf && goff && gcount && dup && H % 8 == 0 && phase >= 0 && phase <= 2,
          "ep_expand: bad args");
  return ep_expand(buf, H, goff, gcount, G, dup, phase, S(stream));
}

int b200moe_ep_reduce_parts(const void* parts, int nparts, int64_t part_stride, int64_t n, void* out,
                            void* stream) {
  REQUIRE(nparts >= 1 && n >= 0 && n % 8 == 0 && part_stride % 8 == 0 && part_stride >= n,
          "ep_reduce_parts: bad args");
  if (n == 0) return B200MOE_OK;
  REQUIRE(parts && out, "ep_reduce_parts: null pointer");
  return ep_reduce_parts(parts, nparts, part_stride, n, out, S(stream));
}

size_t b200moe_router_stats_ws(int64_t T, int E) { return router_stats_ws_bytes(T, E); }

int b200moe_router_stats(const int32_t* topk_idx, const uint8_t* kept, const float* scores, int64_t T, int k,
                         int E, int64_t* counts, int64_t* top1, double* score_sum, void* workspace,
                         size_t workspace_bytes, void* stream) {
  REQUIRE(T >= 0 && k >= 1 && E >= 1 && k <= E, "router_stats: bad shape");
  REQUIRE(workspace_bytes >= router_stats_ws_bytes(T, E), "router_stats: workspace too small");
  REQUIRE(counts && top1 && score_sum && workspace && (T == 0 || topk_idx), "router_stats: null pointer");
  return router_stats(topk_idx, kept, scores, T, k, E, counts, top1, score_sum, workspace, S(stream));
}

int b200moe_split_bf16x3(const float* src, int64_t rows, int E, void* out3, void* out6, void* stream) {
  REQUIRE(rows >= 0 && E >= 1 && (out3 || out6), "split_bf16x3: bad args");
  if (rows == 0) return B200MOE_OK;
  REQUIRE(src, "split_bf16x3: null pointer");
  return split_bf16x3(src, rows, E, out3, out6, S(stream));
}

int b200moe_sum_parts(const float* parts, int64_t G, int64_t rows, int E, float* out, void* stream) {
  REQUIRE(G >= 1 && rows >= 0 && E >= 1, "sum_parts: bad args");
  if (rows == 0) return B200MOE_OK;
  REQUIRE(parts && out, "sum_parts: null pointer");
  return sum_parts(parts, G, rows, E, out, S(stream));
}

int b200moe_act_fwd(const void* pre, int dtype, int act, const int32_t* group_off, int G,
                    int64_t max_rows, int64_t F, void* h, void* stream) {
  REQUIRE(dt_ok(dtype) && G >= 1 && F >= 1, "act_fwd: bad args");
  REQUIRE(act == B200MOE_ACT_RELU || act == B200MOE_ACT_GELU || act == B200MOE_ACT_SWIGLU,
          "act_fwd: unknown activation %d", act);
  REQUIRE(act != B200MOE_ACT_SWIGLU || F % 32 == 0, "act_fwd: swiglu needs F %% 32 == 0");
  REQUIRE(pre && h && group_off, "act_fwd: null pointer");
  return act_fwd(pre, dtype, act, group_off, G, max_rows, F, h, S(stream));
}

int b200moe_act_bwd(const void* dh, const void* pre, int dtype, int act, const int32_t* group_off,
                    int G, int64_t max_rows, int64_t F, void* dpre, void* stream) {
  REQUIRE(dt_ok(dtype) && G >= 1 && F >= 1, "act_bwd: bad args");
  REQUIRE(act == B200MOE_ACT_RELU || act == B200MOE_ACT_GELU || act == B200MOE_ACT_SWIGLU,
          "act_bwd: unknown activation %d", act);
  REQUIRE(act != B200MOE_ACT_SWIGLU || F % 32 == 0, "act_bwd: swiglu needs F %% 32 == 0");
  REQUIRE(dh && pre && dpre && group_off, "act_bwd: null pointer");
  return act_bwd(dh, pre, dtype, act, group_off, G, max_rows, F, dpre, S(stream));
}

}  // extern "C"
