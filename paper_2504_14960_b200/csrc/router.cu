// K1: router -- gating logits, softmax/sigmoid + top-k, capacity + dispatch
// plan (stable counting sort by expert), router backward.
//
// Reference semantics: /root/reference/pkg/src/moefold/router.py:112-206 and
// dispatcher.py:96-131, 470-490.  All integer outputs are deterministic (no
// atomics whose order could leak into a result).
#include <float.h>

#include "common.cuh"

namespace b200moe {

// ---------------------------------------------------------------------------
// logits = x @ w_g                                            (router.py:145)
// ---------------------------------------------------------------------------
// E <= 32: lanes split the hidden dim, each lane keeps TPW x E partial sums,
// one butterfly reduction at the end.  W_g rows (E contiguous floats) are read
// once per h and reused for the TPW tokens of the warp.
template <typename T, int EP, int TPW>
__global__ void __launch_bounds__(256) logits_lane_h_kernel(const T* __restrict__ x,
                                                            const float* __restrict__ wg,
                                                            int64_t Tn, int64_t H, int E,
                                                            float* __restrict__ logits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t t0 = warp * TPW;
  if (t0 >= Tn) return;
  float acc[TPW][EP];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int e = 0; e < EP; ++e) acc[i][e] = 0.f;
  for (int64_t h = lane; h < H; h += 32) {
    float w[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) w[e] = (e < E) ? __ldg(wg + h * E + e) : 0.f;
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      const float xv = (t < Tn) ? to_f32(x[t * H + h]) : 0.f;
#pragma unroll
      for (int e = 0; e < EP; ++e) acc[i][e] = fmaf(xv, w[e], acc[i][e]);
    }
  }
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int e = 0; e < EP; ++e) acc[i][e] = warp_sum(acc[i][e]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      if (t >= Tn) break;
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (e < E) logits[t * E + e] = acc[i][e];
    }
  }
}

// E in {4, 8} and H % 8 == 0: lanes own 8 consecutive hidden columns per
// step (one 16-byte load per token for bf16), the matching 8 x E block of W_g
// is read as float4 and reused for the warp's TPW tokens.  HBM-bound on x.
template <typename T, int EP, int TPW>
__global__ void __launch_bounds__(256) logits_vec_kernel(const T* __restrict__ x,
                                                         const float* __restrict__ wg, int64_t Tn,
                                                         int64_t H, float* __restrict__ logits) {
  constexpr int V = 8;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t t0 = warp * TPW;
  if (t0 >= Tn) return;
  float acc[TPW][EP];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int e = 0; e < EP; ++e) acc[i][e] = 0.f;
  for (int64_t h = (int64_t)lane * V; h < H; h += 32 * V) {
    float xv[TPW][V];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = min(t0 + i, Tn - 1);
      const T* p = x + t * H + h;
      if (sizeof(T) == 2) {
        Vec16<T> v;
        v.raw = ld_nc_v4(p);
#pragma unroll
        for (int j = 0; j < V; ++j) xv[i][j] = to_f32(v.v[j]);
      } else {
        Vec16<T> a, b;
        a.raw = ld_nc_v4(p);
        b.raw = ld_nc_v4(p + 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          xv[i][j] = to_f32(a.v[j]);
          xv[i][4 + j] = to_f32(b.v[j]);
        }
      }
    }
    const float4* wrow = reinterpret_cast<const float4*>(wg + h * EP);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float w[EP];
#pragma unroll
      for (int q = 0; q < EP / 4; ++q) {
        const float4 f = __ldg(wrow + j * (EP / 4) + q);
        w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int e = 0; e < EP; ++e) acc[i][e] = fmaf(xv[i][j], w[e], acc[i][e]);
    }
  }
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int e = 0; e < EP; ++e) acc[i][e] = warp_sum(acc[i][e]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      if (t >= Tn) break;
#pragma unroll
      for (int e = 0; e < EP; ++e) logits[t * EP + e] = acc[i][e];
    }
  }
}

// E > 32: lanes split the experts (NPL = E/32 per lane), x values are warp
// broadcasts.
template <typename T, int NPL, int TPW>
__global__ void __launch_bounds__(256) logits_lane_e_kernel(const T* __restrict__ x,
                                                            const float* __restrict__ wg,
                                                            int64_t Tn, int64_t H, int E,
                                                            float* __restrict__ logits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t t0 = warp * TPW;
  if (t0 >= Tn) return;
  float acc[TPW][NPL];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int j = 0; j < NPL; ++j) acc[i][j] = 0.f;
  for (int64_t h = 0; h < H; ++h) {
    float w[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int e = lane + 32 * j;
      w[j] = (e < E) ? __ldg(wg + h * E + e) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      const float xv = (t < Tn) ? to_f32(x[t * H + h]) : 0.f;
#pragma unroll
      for (int j = 0; j < NPL; ++j) acc[i][j] = fmaf(xv, w[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    const int64_t t = t0 + i;
    if (t >= Tn) break;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int e = lane + 32 * j;
      if (e < E) logits[t * E + e] = acc[i][j];
    }
  }
}

template <typename T>
static int launch_logits(const T* x, const float* wg, int64_t Tn, int64_t H, int E, float* out,
                         cudaStream_t st) {
  const int threads = 256, wpb = threads / 32;
#define LANE_H(EP, TPW)                                                              \
  {                                                                                  \
    int64_t warps = ceil_div(Tn, TPW);                                               \
    logits_lane_h_kernel<T, EP, TPW><<<(unsigned)ceil_div(warps, wpb), threads, 0, st>>>( \
        x, wg, Tn, H, E, out);                                                       \
  }
#define LANE_E(NPL, TPW)                                                             \
  {                                                                                  \
    int64_t warps = ceil_div(Tn, TPW);                                               \
    logits_lane_e_kernel<T, NPL, TPW><<<(unsigned)ceil_div(warps, wpb), threads, 0, st>>>( \
        x, wg, Tn, H, E, out);                                                       \
  }
  if ((E == 8 || E == 4) && H % 8 == 0) {
    constexpr int TPW = 4;
    const int64_t warps = ceil_div(Tn, TPW);
    if (E == 8)
      logits_vec_kernel<T, 8, TPW><<<(unsigned)ceil_div(warps, wpb), threads, 0, st>>>(x, wg, Tn, H, out);
    else
      logits_vec_kernel<T, 4, TPW><<<(unsigned)ceil_div(warps, wpb), threads, 0, st>>>(x, wg, Tn, H, out);
  }
  else if (E <= 4) LANE_H(4, 8)
  else if (E <= 8) LANE_H(8, 8)
  else if (E <= 16) LANE_H(16, 4)
  else if (E <= 32) LANE_H(32, 2)
  else if (E <= 64) LANE_E(2, 8)
  else if (E <= 128) LANE_E(4, 8)
  else if (E <= 256) LANE_E(8, 4)
  else {
    set_error("router_logits: E=%d > 256 unsupported", E);
    return B200MOE_EUNSUPPORTED;
  }
#undef LANE_H
#undef LANE_E
  B200MOE_CHECK_LAUNCH("router_logits");
  return B200MOE_OK;
}

// ---------------------------------------------------------------------------
// scores + top-k + gates                              (router.py:112-162)
// ---------------------------------------------------------------------------
// One warp per token.  Scores are evaluated in float64 like the reference and
// the selection key is (score desc, expert id asc) -- the stable argsort of
// router.py:123.  Lane l owns experts l, l+32, ... (NPL per lane).
template <int NPL>
__global__ void __launch_bounds__(256) topk_kernel(const float* __restrict__ logits, int64_t Tn,
                                                   int E, int k, int gate_fn, int renorm,
                                                   float* __restrict__ scores,
                                                   int32_t* __restrict__ topk_idx,
                                                   float* __restrict__ gates,
                                                   double* __restrict__ gates64,
                                                   int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= Tn) return;
  double s[NPL];
  const float* row = logits + t * E;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int e = lane + 32 * j;
    s[j] = (e < E) ? (double)row[e] : -DBL_MAX;
    bad |= e < E && !isfinite(row[e]);
  }
  // non-finite logits (router.py:141-144): flag, and a valid placeholder
  // routing 0..k-1 so that nothing downstream indexes out of range
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0 && status) atomicOr(status, 1);
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (lane + 32 * j < E) scores[t * E + lane + 32 * j] = 0.f;
    if (lane < k) {
      topk_idx[t * k + lane] = lane;
      gates[t * k + lane] = 0.f;
      if (gates64) gates64[t * k + lane] = 0.0;
    }
    return;
  }
  if (gate_fn == B200MOE_GATE_SOFTMAX) {
    double m = -DBL_MAX;
#pragma unroll
    for (int j = 0; j < NPL; ++j) m = fmax(m, s[j]);
    m = warp_max(m);
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int e = lane + 32 * j;
      s[j] = (e < E) ? exp(s[j] - m) : 0.0;
      sum += s[j];
    }
    sum = warp_sum(sum);
#pragma unroll
    for (int j = 0; j < NPL; ++j) s[j] = s[j] / sum;
  } else {
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int e = lane + 32 * j;
      s[j] = (e < E) ? 1.0 / (1.0 + exp(-s[j])) : 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int e = lane + 32 * j;
    if (e < E) scores[t * E + e] = (float)s[j];
  }
  // k rounds of warp arg-max; `taken` marks this lane's selected entries.
  unsigned taken = 0;
  double raw_sum = 0.0;
  double my_raw = 0.0;  // lane r keeps the raw score of slot r (k <= 32)
  for (int r = 0; r < k; ++r) {
    double best = -1.0;
    int bid = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int e = lane + 32 * j;
      if (e < E && !((taken >> j) & 1u)) {
        if (s[j] > best || (s[j] == best && e < bid)) {
          best = s[j];
          bid = e;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bid, o);
      if (ob > best || (ob == best && oi < bid)) {
        best = ob;
        bid = oi;
      }
    }
    if ((bid & 31) == lane) taken |= 1u << (bid >> 5);
    if (lane == r) my_raw = best;
    raw_sum += best;  // same order on every lane: slot 0, 1, ...
    if (lane == 0) topk_idx[t * k + r] = bid;
  }
  if (lane < k) {
    const double g = renorm ? my_raw / raw_sum : my_raw;
    gates[t * k + lane] = (float)g;
    if (gates64) gates64[t * k + lane] = g;
  }
}

// ---------------------------------------------------------------------------
// capacity + dispatch plan                (router.py:171-206, dispatcher.py:96-131)
// ---------------------------------------------------------------------------
// Tokens are processed in chunks of PLAN_CHUNK (one per thread).  Pass 1
// counts pairs per (chunk, expert); pass 2 scans chunks per expert (fixed
// order) and lays out expert segments; pass 3 ranks pairs inside the chunk
// with warp ballots and writes rows.  Because a token's k experts are
// distinct, the rank of pair (t, s) in (position, slot) order among pairs of
// expert e equals the number of earlier tokens routed to e.
constexpr int PLAN_CHUNK = 256;

__global__ void __launch_bounds__(PLAN_CHUNK) plan_count_kernel(
    const int32_t* __restrict__ topk, const uint8_t* __restrict__ kept_in,
    const int32_t* __restrict__ order, int64_t Tn, int k, int E, int32_t* __restrict__ chunk_cnt) {
  extern __shared__ int32_t cnt[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * PLAN_CHUNK + threadIdx.x;
  if (i < Tn) {
    const int64_t t = order ? order[i] : i;
    for (int s = 0; s < k; ++s) {
      if (kept_in && !kept_in[t * k + s]) continue;
      atomicAdd(&cnt[topk[t * k + s]], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_cnt[(int64_t)blockIdx.x * E + e] = cnt[e];
}

__global__ void __launch_bounds__(1024) plan_scan_kernel(int32_t* __restrict__ chunk_cnt,
                                                         int64_t nchunks, int E, int64_t cap,
                                                         int align, int32_t* __restrict__ counts,
                                                         int32_t* __restrict__ offsets,
                                                         int32_t* __restrict__ poffsets) {
  extern __shared__ int32_t kept_cnt[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int32_t v = chunk_cnt[c * E + e];
      chunk_cnt[c * E + e] = run;  // becomes the chunk base
      run += v;
    }
    const int32_t kc = (cap > 0 && run > cap) ? (int32_t)cap : run;
    kept_cnt[e] = kc;
    counts[e] = kc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t o = 0, po = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = o;
      poffsets[e] = po;
      o += kept_cnt[e];
      // align < 0: pad-to-capacity, every segment has exactly -align rows
      po += align > 0 ? (kept_cnt[e] + align - 1) / align * align : -align;
    }
    offsets[E] = o;
    poffsets[E] = po;
  }
}

template <int KMAX>
__global__ void __launch_bounds__(PLAN_CHUNK) plan_assign_kernel(
    const int32_t* __restrict__ topk, const float* __restrict__ gates,
    const uint8_t* __restrict__ kept_in, const int32_t* __restrict__ order, int64_t Tn, int k,
    int E, int64_t cap, const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ offsets,
    const int32_t* __restrict__ poffsets, uint8_t* __restrict__ kept_out,
    int32_t* __restrict__ send_row, int32_t* __restrict__ gemm_row, int64_t* __restrict__ perm,
    float* __restrict__ perm_gates) {
  extern __shared__ int32_t wcnt[];  // [nwarps][E]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = PLAN_CHUNK / 32;
  const int64_t i = (int64_t)blockIdx.x * PLAN_CHUNK + threadIdx.x;
  const bool live = i < Tn;
  const int64_t t = live ? (order ? order[i] : i) : 0;
  int ex[KMAX];
  bool val[KMAX];
  int rk[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    ex[s] = -1;
    val[s] = false;
    rk[s] = 0;
    if (s < k && live) {
      ex[s] = topk[t * k + s];
      val[s] = kept_in ? (kept_in[t * k + s] != 0) : true;
    }
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int e = 0; e < E; ++e) {
    bool has = false;
    int slot = -1;
#pragma unroll
    for (int s = 0; s < KMAX; ++s)
      if (val[s] && ex[s] == e) {
        has = true;
        slot = s;
      }
    const unsigned b = __ballot_sync(0xffffffffu, has);
    if (has) {
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (s == slot) rk[s] = __popc(b & lt);
    }
    if (lane == 0) wcnt[w * E + e] = __popc(b);
  }
  __syncthreads();
  // exclusive prefix over warps, per expert (fixed order)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = chunk_base[(int64_t)blockIdx.x * E + e];
    for (int ww = 0; ww < nw; ++ww) {
      const int32_t v = wcnt[ww * E + e];
      wcnt[ww * E + e] = run;
      run += v;
    }
  }
  __syncthreads();
  if (!live) return;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s >= k) break;
    const int64_t p = t * k + s;
    if (!val[s]) {
      kept_out[p] = 0;
      send_row[p] = -1;
      gemm_row[p] = -1;
      continue;
    }
    const int e = ex[s];
    const int32_t r = wcnt[w * E + e] + rk[s];
    const bool keep = cap <= 0 || r < cap;
    kept_out[p] = keep ? 1 : 0;
    if (keep) {
      const int32_t sr = offsets[e] + r;
      send_row[p] = sr;
      gemm_row[p] = poffsets[e] + r;
      perm[sr] = p;
      if (perm_gates) perm_gates[sr] = gates[p];
    } else {
      send_row[p] = -1;
      gemm_row[p] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// probability-priority capacity                              (router.py:195)
// ---------------------------------------------------------------------------
// Pairs are given expert-segmented (perm0/offsets0 of a dropless plan).  The
// rank of a pair inside its segment under (-gate, position, slot) is counted
// against every other pair of the segment, tiled through shared memory:
// O(n_e^2) work per expert, deterministic.
__global__ void __launch_bounds__(256) capacity_by_gate_kernel(
    const int64_t* __restrict__ perm0, const int32_t* __restrict__ off0,
    const double* __restrict__ g64, const int64_t* __restrict__ positions, int k, int64_t cap,
    uint8_t* __restrict__ kept_out) {
  __shared__ double sg[256];
  __shared__ int64_t sp[256];
  __shared__ int32_t ss[256];
  const int e = blockIdx.y;
  const int32_t beg = off0[e], n = off0[e + 1] - beg;
  const int32_t mine = blockIdx.x * 256 + threadIdx.x;
  if ((int32_t)(blockIdx.x * 256) >= n) return;
  double g = 0.0;
  int64_t pos = 0;
  int slot = 0;
  int64_t pair = -1;
  if (mine < n) {
    pair = perm0[beg + mine];
    g = g64[pair];
    pos = positions ? positions[pair / k] : pair / k;
    slot = (int)(pair % k);
  }
  int64_t rank = 0;
  for (int32_t base = 0; base < n; base += 256) {
    __syncthreads();
    const int32_t q = base + threadIdx.x;
    if (q < n) {
      const int64_t pq = perm0[beg + q];
      sg[threadIdx.x] = g64[pq];
      sp[threadIdx.x] = positions ? positions[pq / k] : pq / k;
      ss[threadIdx.x] = (int32_t)(pq % k);
    }
    __syncthreads();
    const int lim = min(256, n - base);
    if (mine < n) {
      for (int j = 0; j < lim; ++j) {
        const double gq = sg[j];
        const bool before = gq > g || (gq == g && (sp[j] < pos || (sp[j] == pos && ss[j] < slot)));
        rank += before ? 1 : 0;
      }
    }
  }
  if (mine < n) kept_out[pair] = rank < cap ? 1 : 0;
}

// ---------------------------------------------------------------------------
// full-sequence capacity                          (router.py:209-269)
// ---------------------------------------------------------------------------
// The (sequence x expert, position) keys of every pair of the TP x CP group
// arrive all-gathered in fixed member slots (padding = INT64_MAX) and sorted
// on the device in admission order: by segment seg = (pos / seq_len) * E + e,
// then (probability priority) by gate descending, then by position.  A pair
// is kept iff its rank inside its segment is below cap -- the rank is its
// index minus the segment's first index, found by binary search in the
// sorted segment array (no scan, no host round trip).  Flags are written
// back to the pairs' original slots.  pos_by_pos (every pair's position,
// sorted) detects duplicate token positions across shards: a token's k pairs
// share a position, so position i equal to position i - k means two tokens
// (status bit 3).
__global__ void __launch_bounds__(256) fullseq_capacity_kernel(
    const int64_t* __restrict__ seg_sorted, const int64_t* __restrict__ order, int64_t N, int64_t cap,
    uint8_t* __restrict__ kept_slot, const int64_t* __restrict__ pos_by_pos, int k,
    int32_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int64_t sg = seg_sorted[i];
  const int64_t slot = order[i];
  if (sg == INT64_MAX) {
    kept_slot[slot] = 0;
  } else {
    int64_t lo = 0, hi = i;  // first index with seg_sorted[idx] == sg
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (seg_sorted[mid] < sg) lo = mid + 1;
      else hi = mid;
    }
    kept_slot[slot] = (i - lo) < cap ? 1 : 0;
  }
  if (pos_by_pos && status && i >= k) {
    const int64_t p = pos_by_pos[i];
    if (p != INT64_MAX && p == pos_by_pos[i - k]) atomicOr(status, 8);
  }
}

int fullseq_capacity(const int64_t* seg_sorted, const int64_t* order, int64_t N, int64_t cap,
                     uint8_t* kept_slot, const int64_t* pos_by_pos, int k, int32_t* status,
                     cudaStream_t st) {
  if (N == 0) return B200MOE_OK;
  fullseq_capacity_kernel<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(seg_sorted, order, N, cap, kept_slot,
                                                                      pos_by_pos, k, status);
  B200MOE_CHECK_LAUNCH("fullseq_capacity");
  return B200MOE_OK;
}

// ---------------------------------------------------------------------------
// router backward                                  (dispatcher.py:470-488)
// ---------------------------------------------------------------------------
// an fp32 value as three bf16 parts hi + mid + lo == v exactly (8 + 8 + 8
// significand bits); see split_bf16x3_kernel below
__device__ __forceinline__ void split3(float v, __nv_bfloat16& hi, __nv_bfloat16& mid, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

template <int NPL>
__global__ void __launch_bounds__(256) router_bwd_kernel(const float* __restrict__ dgates,
                                                         const float* __restrict__ scores,
                                                         const int32_t* __restrict__ topk,
                                                         const float* __restrict__ gates,
                                                         int64_t Tn, int E, int k, int gate_fn,
                                                         int renorm, float* __restrict__ dz,
                                                         __nv_bfloat16* __restrict__ parts, int epw, int nb) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= Tn) return;
  // d_sel per slot, computed redundantly by every lane (k is small)
  double total = 0.0, inner = 0.0;
  if (renorm) {
    for (int s = 0; s < k; ++s) {
      total += (double)scores[t * E + topk[t * k + s]];
      inner += (double)dgates[t * k + s] * (double)gates[t * k + s];
    }
  }
  double ds[NPL], sc[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    ds[j] = 0.0;
    const int e = lane + 32 * j;
    sc[j] = (e < E) ? (double)scores[t * E + e] : 0.0;
  }
  for (int s = 0; s < k; ++s) {
    const int e = topk[t * k + s];
    double d = dgates[t * k + s];
    if (renorm) d = (d - inner) / total;
#pragma unroll
    for (int j = 0; j < NPL; ++j)
      if (lane + 32 * j == e) ds[j] += d;
  }
  if (gate_fn == B200MOE_GATE_SOFTMAX) {
    double dot = 0.0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) dot += ds[j] * sc[j];
    dot = warp_sum(dot);
#pragma unroll
    for (int j = 0; j < NPL; ++j) ds[j] = sc[j] * (ds[j] - dot);
  } else {
#pragma unroll
    for (int j = 0; j < NPL; ++j) ds[j] = ds[j] * sc[j] * (1.0 - sc[j]);
  }
#pragma unroll
  for (int j = 0; j < NPL; ++j) {
    const int e = lane + 32 * j;
    if (e >= E) continue;
    const float v = (float)ds[j];
    dz[t * E + e] = v;
    if (parts) {  // the exact bf16 split hi + mid + lo of dz for the tensor-core x^T dz
      __nv_bfloat16 hi, mid, lo;
      split3(v, hi, mid, lo);
      __nv_bfloat16* row = parts + t * nb;
      row[e] = hi;
      row[epw + e] = mid;
      row[2 * epw + e] = lo;
    }
  }
  if (parts) {
    for (int c = lane; c < nb; c += 32)
      if (c >= 3 * epw || c % epw >= E) parts[t * nb + c] = __float2bfloat16_rn(0.f);
  }
}

// dW_g = x^T dz, split over token chunks for parallelism and reduced in a
// fixed order (deterministic).  Pass 1: CTA (64-wide hidden strip, chunk of
// WG_CHUNK tokens) -> partial[chunk][h][e]; lane owns 2 adjacent h, warps
// stride the chunk's tokens, warps reduce through smem.  Pass 2: sum chunks.
constexpr int WG_CHUNK = 256;
constexpr int WG_EB = 16;

template <typename T>
__global__ void __launch_bounds__(256) router_wgrad_partial_kernel(const T* __restrict__ x,
                                                                   const float* __restrict__ dz,
                                                                   int64_t Tn, int64_t H, int E,
                                                                   float* __restrict__ part) {
  __shared__ float red[8][64][WG_EB + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t h0 = (int64_t)blockIdx.x * 64 + 2 * lane;
  const int64_t tb = (int64_t)blockIdx.y * WG_CHUNK;
  const int64_t te = min(Tn, tb + WG_CHUNK);
  for (int e0 = 0; e0 < E; e0 += WG_EB) {
    float acc0[WG_EB], acc1[WG_EB];
#pragma unroll
    for (int j = 0; j < WG_EB; ++j) acc0[j] = acc1[j] = 0.f;
    for (int64_t t = tb + w; t < te; t += 8) {
      const float x0 = (h0 < H) ? to_f32(x[t * H + h0]) : 0.f;
      const float x1 = (h0 + 1 < H) ? to_f32(x[t * H + h0 + 1]) : 0.f;
      const float* d = dz + t * E + e0;
#pragma unroll
      for (int j = 0; j < WG_EB; ++j) {
        const float dv = (e0 + j < E) ? __ldg(d + j) : 0.f;
        acc0[j] = fmaf(x0, dv, acc0[j]);
        acc1[j] = fmaf(x1, dv, acc1[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < WG_EB; ++j) {
      red[w][2 * lane][j] = acc0[j];
      red[w][2 * lane + 1][j] = acc1[j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * WG_EB; i += 256) {
      const int hh = i / WG_EB, j = i % WG_EB;
      const int64_t h = (int64_t)blockIdx.x * 64 + hh;
      if (h < H && e0 + j < E) {
        float s = 0.f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][hh][j];
        part[((int64_t)blockIdx.y * H + h) * E + e0 + j] = s;
      }
    }
    __syncthreads();
  }
}

__global__ void router_wgrad_reduce_kernel(const float* __restrict__ part, int64_t nchunks,
                                           int64_t HE, float* __restrict__ dwg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < HE;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t c = 0; c < nchunks; ++c) s += part[c * HE + i];
    dwg[i] = s;
  }
}

// ---------------------------------------------------------------------------
// load statistics                                          (router.py:279-301)
// ---------------------------------------------------------------------------
// Per 256-token chunk: kept pairs per expert, top-1 counts, and the sum of
// row-normalised scores per expert (fp64); a second pass folds the chunks in
// order, so the result is deterministic.
constexpr int ST_CHUNK = 256;

__global__ void __launch_bounds__(ST_CHUNK) router_stats_partial_kernel(
    const int32_t* __restrict__ topk, const uint8_t* __restrict__ kept, const float* __restrict__ scores,
    int64_t Tn, int k, int E, int32_t* __restrict__ pc, int32_t* __restrict__ pt, double* __restrict__ pp) {
  __shared__ double rinv[ST_CHUNK];
  const int64_t t0 = (int64_t)blockIdx.x * ST_CHUNK;
  const int nt = (int)(Tn - t0 < ST_CHUNK ? Tn - t0 : ST_CHUNK);
  if (scores && threadIdx.x < nt) {
    const float* row = scores + (t0 + threadIdx.x) * E;
    double s = 0.0;
    for (int e = 0; e < E; ++e) s += row[e];
    rinv[threadIdx.x] = 1.0 / s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += ST_CHUNK) {
    int32_t c = 0, c1 = 0;
    double p = 0.0;
    for (int i = 0; i < nt; ++i) {
      const int64_t t = t0 + i;
      for (int s = 0; s < k; ++s)
        c += (topk[t * k + s] == e && (!kept || kept[t * k + s])) ? 1 : 0;
      c1 += topk[t * k] == e ? 1 : 0;
      if (scores) p += (double)scores[t * E + e] * rinv[i];
    }
    pc[(int64_t)blockIdx.x * E + e] = c;
    pt[(int64_t)blockIdx.x * E + e] = c1;
    pp[(int64_t)blockIdx.x * E + e] = p;
  }
}

__global__ void router_stats_reduce_kernel(const int32_t* __restrict__ pc, const int32_t* __restrict__ pt,
                                           const double* __restrict__ pp, int64_t nch, int E,
                                           int64_t* __restrict__ counts, int64_t* __restrict__ top1,
                                           double* __restrict__ psum) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int64_t c = 0, c1 = 0;
  double p = 0.0;
  for (int64_t i = 0; i < nch; ++i) {
    c += pc[i * E + e];
    c1 += pt[i * E + e];
    p += pp[i * E + e];
  }
  counts[e] = c;
  top1[e] = c1;
  psum[e] = p;
}

size_t router_stats_ws_bytes(int64_t Tn, int E) {
  return (size_t)ceil_div(Tn > 0 ? Tn : 1, ST_CHUNK) * E * (4 + 4 + 8);
}

int router_stats(const int32_t* topk, const uint8_t* kept, const float* scores, int64_t Tn, int k, int E,
                 int64_t* counts, int64_t* top1, double* psum, void* ws, cudaStream_t st) {
  const int64_t nch = ceil_div(Tn > 0 ? Tn : 1, ST_CHUNK);
  double* pp = static_cast<double*>(ws);
  int32_t* pc = reinterpret_cast<int32_t*>(pp + nch * E);
  int32_t* pt = pc + nch * E;
  if (Tn > 0)
    router_stats_partial_kernel<<<(unsigned)nch, ST_CHUNK, 0, st>>>(topk, kept, scores, Tn, k, E, pc, pt, pp);
  else {
    cudaMemsetAsync(pc, 0, (size_t)E * 4, st);
    cudaMemsetAsync(pt, 0, (size_t)E * 4, st);
    cudaMemsetAsync(pp, 0, (size_t)E * 8, st);
  }
  router_stats_reduce_kernel<<<(unsigned)ceil_div(E, 128), 128, 0, st>>>(pc, pt, pp, Tn > 0 ? nch : 1, E, counts,
                                                                          top1, psum);
  B200MOE_CHECK_LAUNCH("router_stats");
  return B200MOE_OK;
}

// ---------------------------------------------------------------------------
// fp32 router GEMMs on the bf16 tensor cores: an fp32 value v is split into
// three bf16 parts hi + mid + lo == v exactly (8 + 8 + 8 significand bits),
// so x(bf16) . W_g = x.hi + x.mid + x.lo with exact products and fp32
// accumulation.  Parts are laid out as column blocks of stride Ep (E rounded
// up to 8, zero padded).
// ---------------------------------------------------------------------------

// src [rows, E] fp32 -> out3 [rows, 3 Ep] = (hi | mid | lo) and/or
// out6 [rows, 6 Ep] = (hi | hi | hi | mid | mid | lo) (the dz side of the
// six-term product dz . W^T)
__global__ void split_bf16x3_kernel(const float* __restrict__ src, int64_t rows, int E, int Ep,
                                    __nv_bfloat16* __restrict__ out3, __nv_bfloat16* __restrict__ out6) {
  const int64_t n = rows * Ep;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / Ep;
    const int e = (int)(i % Ep);
    __nv_bfloat16 hi, mid, lo;
    split3(e < E ? src[r * E + e] : 0.f, hi, mid, lo);
    if (out3) {
      __nv_bfloat16* o = out3 + r * 3 * Ep + e;
      o[0] = hi; o[Ep] = mid; o[2 * Ep] = lo;
    }
    if (out6) {
      __nv_bfloat16* o = out6 + r * 6 * Ep + e;
      o[0] = hi; o[Ep] = hi; o[2 * Ep] = hi; o[3 * Ep] = mid; o[4 * Ep] = mid; o[5 * Ep] = lo;
    }
  }
}

// out[r, e] = sum_g ((p[g, r, e] + p[g, r, Ep + e]) + p[g, r, 2 Ep + e]), g ascending
__global__ void sum_parts_kernel(const float* __restrict__ parts, int64_t G, int64_t rows, int E, int Ep,
                                 float* __restrict__ out) {
  const int64_t n = rows * E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / E;
    const int e = (int)(i % E);
    float s = 0.f;
    for (int64_t g = 0; g < G; ++g) {
      const float* p = parts + (g * rows + r) * 3 * Ep + e;
      s += (p[0] + p[Ep]) + p[2 * Ep];
    }
    out[i] = s;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int split_bf16x3(const float* src, int64_t rows, int E, void* out3, void* out6, cudaStream_t st) {
  const int Ep = (E + 7) / 8 * 8;
  const int64_t n = rows * Ep;
  if (n == 0) return B200MOE_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 16);
  split_bf16x3_kernel<<<grid, 256, 0, st>>>(src, rows, E, Ep, static_cast<__nv_bfloat16*>(out3),
                                            static_cast<__nv_bfloat16*>(out6));
  B200MOE_CHECK_LAUNCH("split_bf16x3");
  return B200MOE_OK;
}

int sum_parts(const float* parts, int64_t G, int64_t rows, int E, float* out, cudaStream_t st) {
  const int Ep = (E + 7) / 8 * 8;
  const int64_t n = rows * E;
  if (n == 0) return B200MOE_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 16);
  sum_parts_kernel<<<grid, 256, 0, st>>>(parts, G, rows, E, Ep, out);
  B200MOE_CHECK_LAUNCH("sum_parts");
  return B200MOE_OK;
}

int router_logits(const void* x, int dt, const float* wg, int64_t Tn, int64_t H, int E,
                  float* out, cudaStream_t st) {
  if (dt == B200MOE_BF16)
    return launch_logits(static_cast<const __nv_bfloat16*>(x), wg, Tn, H, E, out, st);
  return launch_logits(static_cast<const float*>(x), wg, Tn, H, E, out, st);
}

int router_topk(const float* logits, int64_t Tn, int E, int k, int gate_fn, int renorm,
                float* scores, int32_t* idx, float* gates, double* gates64, int32_t* status,
                cudaStream_t st) {
  if (Tn == 0) return B200MOE_OK;
  const unsigned grid = (unsigned)ceil_div(Tn, 8);
#define TK(NPL) topk_kernel<NPL><<<grid, 256, 0, st>>>(logits, Tn, E, k, gate_fn, renorm, scores, idx, gates, gates64, status)
  if (E <= 32) TK(1);
  else if (E <= 64) TK(2);
  else if (E <= 128) TK(4);
  else if (E <= 256) TK(8);
  else {
    set_error("router_topk: E=%d > 256 unsupported", E);
    return B200MOE_EUNSUPPORTED;
  }
#undef TK
  B200MOE_CHECK_LAUNCH("router_topk");
  return B200MOE_OK;
}

size_t plan_ws_bytes(int64_t Tn, int E) {
  const int64_t nch = ceil_div(Tn > 0 ? Tn : 1, PLAN_CHUNK);
  return (size_t)(nch * E) * sizeof(int32_t);
}

int dispatch_plan(const int32_t* topk, const float* gates, const uint8_t* kept_in,
                  const int32_t* order, int64_t Tn, int k, int E, int64_t cap, int align, void* ws,
                  uint8_t* kept_out, int32_t* counts, int32_t* offsets, int32_t* poffsets,
                  int32_t* send_row, int32_t* gemm_row, int64_t* perm, float* perm_gates,
                  cudaStream_t st) {
  const int64_t nch = ceil_div(Tn > 0 ? Tn : 1, PLAN_CHUNK);
  int32_t* cc = static_cast<int32_t*>(ws);
  plan_count_kernel<<<(unsigned)nch, PLAN_CHUNK, E * sizeof(int32_t), st>>>(topk, kept_in, order,
                                                                           Tn, k, E, cc);
  plan_scan_kernel<<<1, 1024, E * sizeof(int32_t), st>>>(cc, nch, E, cap, align, counts, offsets,
                                                         poffsets);
  const size_t smem = (size_t)(PLAN_CHUNK / 32) * E * sizeof(int32_t);
#define PA(KM)                                                                                  \
  plan_assign_kernel<KM><<<(unsigned)nch, PLAN_CHUNK, smem, st>>>(                              \
      topk, gates, kept_in, order, Tn, k, E, cap, cc, offsets, poffsets, kept_out, send_row,    \
      gemm_row, perm, perm_gates)
  if (k <= 2) PA(2);
  else if (k <= 4) PA(4);
  else if (k <= 8) PA(8);
  else if (k <= 16) PA(16);
  else {
    set_error("dispatch_plan: k=%d > 16 unsupported", k);
    return B200MOE_EUNSUPPORTED;
  }
#undef PA
  B200MOE_CHECK_LAUNCH("dispatch_plan");
  return B200MOE_OK;
}

int capacity_by_gate(const int64_t* perm0, const int32_t* off0, const double* g64,
                     const int64_t* positions, int64_t Tn, int k, int E, int64_t cap,
                     uint8_t* kept_out, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(Tn > 0 ? Tn : 1, 256), (unsigned)E);
  capacity_by_gate_kernel<<<grid, 256, 0, st>>>(perm0, off0, g64, positions, k, cap, kept_out);
  B200MOE_CHECK_LAUNCH("capacity_by_gate");
  return B200MOE_OK;
}

int router_bwd(const float* dgates, const float* scores, const int32_t* topk, const float* gates,
               int64_t Tn, int E, int k, int gate_fn, int renorm, float* dz, void* parts, int epw, int nb,
               cudaStream_t st) {
  const unsigned grid = (unsigned)ceil_div(Tn, 8);
  __nv_bfloat16* pb = static_cast<__nv_bfloat16*>(parts);
#define RB(NPL) router_bwd_kernel<NPL><<<grid, 256, 0, st>>>(dgates, scores, topk, gates, Tn, E, k, gate_fn, renorm, dz, pb, epw, nb)
  if (E <= 32) RB(1);
  else if (E <= 64) RB(2);
  else if (E <= 128) RB(4);
  else if (E <= 256) RB(8);
  else {
    set_error("router_bwd: E=%d > 256 unsupported", E);
    return B200MOE_EUNSUPPORTED;
  }
#undef RB
  B200MOE_CHECK_LAUNCH("router_bwd");
  return B200MOE_OK;
}

// bf16 x, E <= 8, H % 8 == 0: thread (h-slice of 8 columns) x (token chunk)
// keeps its 8 x E block of dW_g in registers and streams its chunk's x rows
// once (16-byte loads, a block covers 2048 consecutive columns); dz[t] is a
// uniform (broadcast) load.  The chunks' partial blocks are folded in chunk
// order by router_wgrad_reduce_kernel (deterministic).  HBM-bound on x.
constexpr int WGV_COLS = 2048;  // columns per block: 256 threads x 8
constexpr int WGV_MAX_CHUNKS = 148;

template <int EP, int UT>
__global__ void __launch_bounds__(256, 2) router_wgrad_vec_kernel(const __nv_bfloat16* __restrict__ x,
                                                                 const float* __restrict__ dz, int64_t Tn,
                                                                 int64_t H, int E, int64_t chunk,
                                                                 float* __restrict__ part) {
  const int64_t h0 = (int64_t)blockIdx.y * WGV_COLS + threadIdx.x * 8;
  if (h0 >= H) return;
  const int64_t tb = (int64_t)blockIdx.x * chunk, te = min(Tn, tb + chunk);
  float acc[8][EP];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < EP; ++e) acc[j][e] = 0.f;
  for (int64_t t = tb; t < te; t += UT) {
    Vec16<__nv_bfloat16> v[UT];
#pragma unroll
    for (int u = 0; u < UT; ++u)
      if (t + u < te) v[u].raw = ld_nc_v4(x + (t + u) * H + h0);
#pragma unroll
    for (int u = 0; u < UT; ++u) {
      if (t + u >= te) break;
      float d[EP];
      const float* dr = dz + (t + u) * E;
#pragma unroll
      for (int e = 0; e < EP; ++e) d[e] = e < E ? __ldg(dr + e) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xv = __bfloat162float(v[u].v[j]);
#pragma unroll
        for (int e = 0; e < EP; ++e) acc[j][e] = fmaf(xv, d[e], acc[j][e]);
      }
    }
  }
  float* o = part + ((int64_t)blockIdx.x * H + h0) * E;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int e = 0; e < EP; ++e)
      if (e < E) o[j * E + e] = acc[j][e];
}

size_t router_wgrad_ws_bytes(int64_t Tn, int64_t H, int E) {
  const int64_t nch = std::max<int64_t>(ceil_div(Tn > 0 ? Tn : 1, WG_CHUNK), WGV_MAX_CHUNKS);
  return (size_t)nch * H * E * sizeof(float);
}

int router_wgrad(const void* x, int dt, const float* dz, int64_t Tn, int64_t H, int E, float* dwg,
                 void* ws, cudaStream_t st) {
  float* part = static_cast<float*>(ws);
  const int64_t HE = H * E;
  if (dt == B200MOE_BF16 && E <= 8 && H % 8 == 0 && Tn > 0) {
    constexpr int UT = 4;
    int64_t chunk = ceil_div(Tn, WGV_MAX_CHUNKS);
    chunk = std::max<int64_t>(ceil_div(chunk, UT) * UT, 32);
    const int64_t nch = ceil_div(Tn, chunk);
    dim3 grid((unsigned)nch, (unsigned)ceil_div(H, WGV_COLS));
    const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
    if (E <= 4)
      router_wgrad_vec_kernel<4, UT><<<grid, 256, 0, st>>>(xb, dz, Tn, H, E, chunk, part);
    else
      router_wgrad_vec_kernel<8, UT><<<grid, 256, 0, st>>>(xb, dz, Tn, H, E, chunk, part);
    router_wgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(HE, 256), 148 * 8), 256, 0, st>>>(
        part, nch, HE, dwg);
    B200MOE_CHECK_LAUNCH("router_wgrad");
    return B200MOE_OK;
  }
  const int64_t nch = ceil_div(Tn, WG_CHUNK);
  dim3 grid((unsigned)ceil_div(H, 64), (unsigned)nch);
  if (dt == B200MOE_BF16)
    router_wgrad_partial_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), dz, Tn, H, E, part);
  else
    router_wgrad_partial_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), dz, Tn,
                                                             H, E, part);
  router_wgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(HE, 256), 148 * 8), 256, 0, st>>>(
      part, nch, HE, dwg);
  B200MOE_CHECK_LAUNCH("router_wgrad");
  return B200MOE_OK;
}

}  // namespace b200moe
