// K2: token permute / unpermute-combine (forward and backward).
//
// Reference semantics: dispatcher.py:134-157 (permute, unpermute_combine),
// :426-428 (backward dispatch rows + dgate), :467-468 + :490 (backward
// combine + router term).  Token-major: each token row is read once with
// 16-byte vector loads and written to (or gathered from) its k pair rows, so
// the kernels are HBM-bound at  T*H*b + P*H*b  bytes.
#include "common.cuh"

namespace b200moe {

template <typename T>
__device__ __forceinline__ void scale_vec(Vec16<T>& v, float s) {
#pragma unroll
  for (int i = 0; i < Vec16<T>::N; ++i) v.v[i] = from_f32<T>(to_f32(v.v[i]) * s);
}

// ------------------------------------------------------------------ permute
template <typename T, int KMAX, bool VEC>
__global__ void __launch_bounds__(256) permute_kernel(const T* __restrict__ x, int64_t Tn, int64_t H,
                                                      int k, const int32_t* __restrict__ pair_row,
                                                      const float* __restrict__ scale,
                                                      T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= Tn) return;
  int32_t rows[KMAX];
  float sc[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    rows[s] = (s < k) ? pair_row[t * k + s] : -1;
    sc[s] = (s < k && scale) ? scale[t * k + s] : 1.f;
  }
  const T* src = x + t * H;
  if (VEC) {
    constexpr int N = Vec16<T>::N;
    const int64_t nv = H / N;
    for (int64_t c = lane; c < nv; c += 32) {
      Vec16<T> v;
      v.raw = ld_nc_v4(src + c * N);
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (rows[s] < 0) continue;
        Vec16<T> o = v;
        if (scale) scale_vec(o, sc[s]);
        st_v4(out + (int64_t)rows[s] * H + c * N, o.raw);
      }
    }
  } else {
    for (int64_t c = lane; c < H; c += 32) {
      const float v = to_f32(src[c]);
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (rows[s] >= 0) out[(int64_t)rows[s] * H + c] = from_f32<T>(v * sc[s]);
    }
  }
}

// Zero the alignment padding of every expert segment.
template <typename T>
__global__ void zero_pad_kernel(T* __restrict__ buf, int64_t H, const int32_t* __restrict__ poff,
                                const int32_t* __restrict__ cnt) {
  const int e = blockIdx.y;
  const int64_t row = (int64_t)poff[e] + cnt[e] + blockIdx.x;
  if (row >= poff[e + 1]) return;
  T* p = buf + row * H;
  for (int64_t c = threadIdx.x; c < H; c += blockDim.x) p[c] = from_f32<T>(0.f);
}

// ------------------------------------------------------------- permute bwd
template <typename T, int KMAX, bool VEC>
__global__ void __launch_bounds__(256) permute_bwd_kernel(
    const T* __restrict__ u, int64_t Tn, int64_t H, int k, const int32_t* __restrict__ pair_row,
    const float* __restrict__ gates, const T* __restrict__ y_rows, T* __restrict__ dy_rows,
    float* __restrict__ dgates) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= Tn) return;
  int32_t rows[KMAX];
  float g[KMAX], dot[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    rows[s] = (s < k) ? pair_row[t * k + s] : -1;
    g[s] = (s < k) ? gates[t * k + s] : 0.f;
    dot[s] = 0.f;
  }
  const T* src = u + t * H;
  if (VEC) {
    constexpr int N = Vec16<T>::N;
    const int64_t nv = H / N;
    for (int64_t c = lane; c < nv; c += 32) {
      Vec16<T> v;
      v.raw = ld_nc_v4(src + c * N);
      // all k expert rows in flight before the first use
      Vec16<T> y[KMAX];
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (rows[s] >= 0) y[s].raw = ld_nc_v4(y_rows + (int64_t)rows[s] * H + c * N);
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (rows[s] < 0) continue;
        Vec16<T> o;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const float uv = to_f32(v.v[i]);
          dot[s] = fmaf(uv, to_f32(y[s].v[i]), dot[s]);
          o.v[i] = from_f32<T>(uv * g[s]);
        }
        st_v4(dy_rows + (int64_t)rows[s] * H + c * N, o.raw);
      }
    }
  } else {
    for (int64_t c = lane; c < H; c += 32) {
      const float uv = to_f32(src[c]);
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (rows[s] < 0) continue;
        const int64_t off = (int64_t)rows[s] * H + c;
        dot[s] = fmaf(uv, to_f32(y_rows[off]), dot[s]);
        dy_rows[off] = from_f32<T>(uv * g[s]);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s >= k) break;
    const float d = warp_sum(dot[s]);
    if (lane == 0) dgates[t * k + s] = rows[s] >= 0 ? d : 0.f;
  }
}

// ------------------------------------------------------------------ combine
// bf16(sum over p ascending of parts[p][r][h..h+8)) in fp32, part 0 already
// loaded -- the ETP reduce-scatter fold (ep_peer.cu ep_reduce_parts) fused
// into the combines' row loads
template <typename T>
__device__ __forceinline__ Vec16<T> reduce_parts_row(const T* __restrict__ rows, int32_t r, int64_t H,
                                                     int64_t h, int nparts, int64_t pstride, Vec16<T> p0) {
  static_assert(sizeof(T) == 2, "bf16 rows");
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = to_f32(p0.v[j]);
  for (int p = 1; p < nparts; ++p) {
    Vec16<T> q;
    q.raw = ld_nc_v4(rows + p * pstride + (int64_t)r * H + h);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += to_f32(q.v[j]);
  }
  Vec16<T> o;
#pragma unroll
  for (int j = 0; j < 8; ++j) o.v[j] = from_f32<T>(acc[j]);
  return o;
}

// TPW tokens per warp so the optional router term (dz[t] @ w_g^T, w_g^T given
// as [E, H]) reuses each w_g^T chunk across the warp's tokens.
template <typename Tin, typename Tout, int KMAX, int TPW>
__global__ void __launch_bounds__(256) combine_kernel(
    const Tin* __restrict__ rows, int64_t Tn, int64_t H, int k, const int32_t* __restrict__ pair_row,
    const float* __restrict__ gates, const float* __restrict__ dz, const float* __restrict__ wgT,
    int E, Tout* __restrict__ out, int accumulate) {
  constexpr int N = 4;  // 4 elements per lane per step (8 B bf16 / 16 B fp32)
  const int lane = threadIdx.x & 31;
  const int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TPW;
  if (t0 >= Tn) return;
  int32_t r[TPW][KMAX];
  float w[TPW][KMAX];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      const int64_t t = t0 + i;
      const bool ok = t < Tn && s < k;
      r[i][s] = ok ? pair_row[t * k + s] : -1;
      w[i][s] = (ok && gates) ? gates[t * k + s] : 1.f;
    }
  for (int64_t h = (int64_t)lane * N; h < H; h += 32 * N) {
    const int nh = (int)min((int64_t)N, H - h);
    float acc[TPW][N];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) acc[i][j] = 0.f;
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (r[i][s] < 0) continue;
        const Tin* p = rows + (int64_t)r[i][s] * H + h;
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (j < nh) acc[i][j] = fmaf(w[i][s], to_f32(p[j]), acc[i][j]);
      }
    }
    if (dz) {
      for (int e = 0; e < E; ++e) {
        float wv[N];
#pragma unroll
        for (int j = 0; j < N; ++j) wv[j] = (j < nh) ? __ldg(wgT + (int64_t)e * H + h + j) : 0.f;
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int64_t t = t0 + i;
          if (t >= Tn) break;
          const float d = __ldg(dz + t * E + e);
#pragma unroll
          for (int j = 0; j < N; ++j) acc[i][j] = fmaf(d, wv[j], acc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      if (t >= Tn) break;
      Tout* o = out + t * H + h;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (j >= nh) break;
        float v = acc[i][j];
        if (accumulate) v += to_f32(o[j]);
        o[j] = from_f32<Tout>(v);
      }
    }
  }
}

// Vectorised combine (H % 8 == 0): each lane owns 8 consecutive columns per
// step; the TPW x k row loads of a step are independent 16-byte loads (bf16)
// so every warp keeps TPW*k requests in flight.
template <typename Tin, typename Tout, int KMAX, int TPW>
__global__ void __launch_bounds__(256) combine_vec_kernel(
    const Tin* __restrict__ rows, int64_t Tn, int64_t H, int k, const int32_t* __restrict__ pair_row,
    const float* __restrict__ gates, const float* __restrict__ dz, const float* __restrict__ wgT,
    int E, Tout* __restrict__ out, int accumulate) {
  constexpr int V = 8;
  const int lane = threadIdx.x & 31;
  const int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TPW;
  if (t0 >= Tn) return;
  int32_t r[TPW][KMAX];
  float w[TPW][KMAX];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      const int64_t t = t0 + i;
      const bool ok = t < Tn && s < k;
      r[i][s] = ok ? pair_row[t * k + s] : -1;
      w[i][s] = (ok && gates) ? gates[t * k + s] : 1.f;
    }
  for (int64_t h = (int64_t)lane * V; h < H; h += 32 * V) {
    float acc[TPW][V];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int j = 0; j < V; ++j) acc[i][j] = 0.f;
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (r[i][s] < 0) continue;
        const Tin* p = rows + (int64_t)r[i][s] * H + h;
        float v[V];
        if (sizeof(Tin) == 2) {
          Vec16<Tin> a;
          a.raw = ld_nc_v4(p);
#pragma unroll
          for (int j = 0; j < V; ++j) v[j] = to_f32(a.v[j]);
        } else {
          Vec16<Tin> a, b;
          a.raw = ld_nc_v4(p);
          b.raw = ld_nc_v4(p + 4);
#pragma unroll
          for (int j = 0; j < 4; ++j) { v[j] = to_f32(a.v[j]); v[4 + j] = to_f32(b.v[j]); }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) acc[i][j] = fmaf(w[i][s], v[j], acc[i][j]);
      }
    }
    if (dz) {
      for (int e = 0; e < E; ++e) {
        const float4* wp = reinterpret_cast<const float4*>(wgT + (int64_t)e * H + h);
        const float4 wa = __ldg(wp), wb = __ldg(wp + 1);
        const float wv[V] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int64_t t = min(t0 + i, Tn - 1);
          const float d = __ldg(dz + t * E + e);
#pragma unroll
          for (int j = 0; j < V; ++j) acc[i][j] = fmaf(d, wv[j], acc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int64_t t = t0 + i;
      if (t >= Tn) break;
      Tout* o = out + t * H + h;
      if (accumulate) {
#pragma unroll
        for (int j = 0; j < V; ++j) acc[i][j] += to_f32(o[j]);
      }
      if (sizeof(Tout) == 2) {
        Vec16<Tout> q;
#pragma unroll
        for (int j = 0; j < V; ++j) q.v[j] = from_f32<Tout>(acc[i][j]);
        st_v4(o, q.raw);
      } else {
        Vec16<Tout> a, b;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a.v[j] = from_f32<Tout>(acc[i][j]);
          b.v[j] = from_f32<Tout>(acc[i][4 + j]);
        }
        st_v4(o, a.raw);
        st_v4(o + 4, b.raw);
      }
    }
  }
}

// Backward combine with the router term (dispatcher.py:480-490 for bf16,
// E <= 8, H % 8 == 0):  dx[t] = sum_s rows[pair_row[t, s]] + dz[t] @ W_g^T
// (+ out[t] when accumulating).  A block covers 2048 consecutive columns,
// each thread 8 of them with its 8 x E slice of W_g^T in registers for the
// whole kernel, and walks a chunk of tokens: per token k 16-byte row loads,
// one 16-byte store, dz[t] and the pair rows as uniform loads -- the FMAs of
// the router term hide under the row traffic (HBM-bound like the plain
// gather).  fp32 sum order: slots in order, then the router term.
constexpr int CR_COLS = 2048;

template <int KMAX, int EP, int UT>
__global__ void __launch_bounds__(256, 2) combine_router_kernel(
    const __nv_bfloat16* __restrict__ rows, int64_t Tn, int64_t H, int k, const int32_t* __restrict__ pair_row,
    const float* __restrict__ dz, const float* __restrict__ wgT, int E, __nv_bfloat16* __restrict__ out,
    int accumulate, int64_t chunk, int nparts, int64_t pstride) {
  const int64_t h0 = (int64_t)blockIdx.y * CR_COLS + threadIdx.x * 8;
  if (h0 >= H) return;
  float w[EP][8];
#pragma unroll
  for (int e = 0; e < EP; ++e) {
    if (e < E) {
      const float4* wp = reinterpret_cast<const float4*>(wgT + (int64_t)e * H + h0);
      const float4 a = __ldg(wp), b = __ldg(wp + 1);
      w[e][0] = a.x; w[e][1] = a.y; w[e][2] = a.z; w[e][3] = a.w;
      w[e][4] = b.x; w[e][5] = b.y; w[e][6] = b.z; w[e][7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) w[e][j] = 0.f;
    }
  }
  const int64_t tb = (int64_t)blockIdx.x * chunk, te = min(Tn, tb + chunk);
  for (int64_t t = tb; t < te; t += UT) {
    Vec16<__nv_bfloat16> v[UT][KMAX];
    bool has[UT][KMAX];
#pragma unroll
    for (int u = 0; u < UT; ++u)
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        const int32_t r = (t + u < te && s < k) ? __ldg(pair_row + (t + u) * k + s) : -1;
        has[u][s] = r >= 0;
        if (r >= 0) v[u][s].raw = ld_nc_v4(rows + (int64_t)r * H + h0);
      }
    if (nparts > 1) {
      // ETP partial rows (one block per member, pstride apart): the row is
      // bf16(sum over members ascending, fp32) -- ep_reduce_parts' value
#pragma unroll
      for (int u = 0; u < UT; ++u)
#pragma unroll
        for (int s = 0; s < KMAX; ++s) {
          if (!has[u][s]) continue;
          const int32_t r = __ldg(pair_row + (t + u) * k + s);
          v[u][s] = reduce_parts_row(rows, r, H, h0, nparts, pstride, v[u][s]);
        }
    }
#pragma unroll
    for (int u = 0; u < UT; ++u) {
      if (t + u >= te) break;
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (has[u][s]) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v[u][s].v[j]);
        }
      const float* dr = dz + (t + u) * E;
#pragma unroll
      for (int e = 0; e < EP; ++e) {
        const float d = e < E ? __ldg(dr + e) : 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(d, w[e][j], acc[j]);
      }
      __nv_bfloat16* o = out + (t + u) * H + h0;
      Vec16<__nv_bfloat16> q;
      if (accumulate) {
        q.raw = ld_v4(o);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(q.v[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) q.v[j] = __float2bfloat16_rn(acc[j]);
      st_v4(o, q.raw);
    }
  }
}

// Gather-sum without the router term: one warp per token (high occupancy),
// each lane owns 8 columns per step and keeps UNR steps x k row loads in
// flight.
template <typename Tin, typename Tout, int KMAX, int UNR>
__global__ void __launch_bounds__(256) combine_gather_kernel(
    const Tin* __restrict__ rows, int64_t Tn, int64_t H, int k, const int32_t* __restrict__ pair_row,
    const float* __restrict__ gates, Tout* __restrict__ out, int accumulate, int nparts, int64_t pstride,
    Tin* __restrict__ rows_out) {
  static_assert(sizeof(Tin) == 2, "bf16 rows");
  constexpr int V = 8;
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= Tn) return;
  int32_t r[KMAX];
  float w[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    r[s] = s < k ? pair_row[t * k + s] : -1;
    w[s] = (s < k && gates) ? gates[t * k + s] : 1.f;
  }
  for (int64_t h0 = (int64_t)lane * V; h0 < H; h0 += 32 * V * UNR) {
    Vec16<Tin> v[UNR][KMAX];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t h = h0 + (int64_t)u * 32 * V;
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (r[s] >= 0 && h < H) v[u][s].raw = ld_nc_v4(rows + (int64_t)r[s] * H + h);
    }
    if (nparts > 1 || rows_out) {  // ETP partial rows: reduce (ep_reduce_parts' value), keep the row
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t h = h0 + (int64_t)u * 32 * V;
#pragma unroll
        for (int s = 0; s < KMAX; ++s)
          if (r[s] >= 0 && h < H) {
            v[u][s] = reduce_parts_row(rows, r[s], H, h, nparts, pstride, v[u][s]);
            if (rows_out) st_v4(rows_out + (int64_t)r[s] * H + h, v[u][s].raw);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t h = h0 + (int64_t)u * 32 * V;
      if (h >= H) break;
      float acc[V];
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = 0.f;
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (r[s] < 0) continue;
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = fmaf(w[s], to_f32(v[u][s].v[j]), acc[j]);
      }
      Tout* o = out + t * H + h;
      if (accumulate) {
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += to_f32(o[j]);
      }
      if (sizeof(Tout) == 2) {
        Vec16<Tout> q;
#pragma unroll
        for (int j = 0; j < V; ++j) q.v[j] = from_f32<Tout>(acc[j]);
        st_v4(o, q.raw);
      } else {
        Vec16<Tout> a, b;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a.v[j] = from_f32<Tout>(acc[j]);
          b.v[j] = from_f32<Tout>(acc[4 + j]);
        }
        st_v4(o, a.raw);
        st_v4(o + 4, b.raw);
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
#define KDISPATCH(k, MACRO)            \
  if (k <= 1) { MACRO(1); }            \
  else if (k <= 2) { MACRO(2); }       \
  else if (k <= 4) { MACRO(4); }       \
  else if (k <= 8) { MACRO(8); }       \
  else if (k <= 16) { MACRO(16); }     \
  else {                               \
    set_error("k=%d > 16 unsupported", k); \
    return B200MOE_EUNSUPPORTED;       \
  }

template <typename T>
static int launch_permute(const T* x, int64_t Tn, int64_t H, int k, const int32_t* pr,
                          const float* scale, T* out, const int32_t* poff, const int32_t* cnt,
                          int E, int64_t max_pad, cudaStream_t st) {
  const unsigned grid = (unsigned)ceil_div(Tn, 8);
  const bool vec = (H % Vec16<T>::N) == 0;
#define PK(KM)                                                                                   \
  {                                                                                              \
    if (vec) permute_kernel<T, KM, true><<<grid, 256, 0, st>>>(x, Tn, H, k, pr, scale, out);     \
    else permute_kernel<T, KM, false><<<grid, 256, 0, st>>>(x, Tn, H, k, pr, scale, out);        \
  }
  if (Tn > 0) { KDISPATCH(k, PK) }
#undef PK
  if (poff && cnt && max_pad > 0) {
    dim3 g((unsigned)max_pad, (unsigned)E);
    zero_pad_kernel<T><<<g, 128, 0, st>>>(out, H, poff, cnt);
  }
  B200MOE_CHECK_LAUNCH("permute");
  return B200MOE_OK;
}

int permute(const void* x, int dt, int64_t Tn, int64_t H, int k, const int32_t* pr,
            const float* scale, void* out, const int32_t* poff, const int32_t* cnt, int E,
            int64_t max_pad, cudaStream_t st) {
  if (dt == B200MOE_BF16)
    return launch_permute(static_cast<const __nv_bfloat16*>(x), Tn, H, k, pr, scale,
                          static_cast<__nv_bfloat16*>(out), poff, cnt, E, max_pad, st);
  return launch_permute(static_cast<const float*>(x), Tn, H, k, pr, scale,
                        static_cast<float*>(out), poff, cnt, E, max_pad, st);
}

template <typename T>
static int launch_permute_bwd(const T* u, int64_t Tn, int64_t H, int k, const int32_t* pr,
                              const float* gates, const T* y, T* dy, float* dg,
                              const int32_t* poff, const int32_t* cnt, int E, int64_t max_pad,
                              cudaStream_t st) {
  const unsigned grid = (unsigned)ceil_div(Tn, 8);
  const bool vec = (H % Vec16<T>::N) == 0;
#define PB(KM)                                                                                 \
  {                                                                                            \
    if (vec) permute_bwd_kernel<T, KM, true><<<grid, 256, 0, st>>>(u, Tn, H, k, pr, gates, y, dy, dg); \
    else permute_bwd_kernel<T, KM, false><<<grid, 256, 0, st>>>(u, Tn, H, k, pr, gates, y, dy, dg); \
  }
  if (Tn > 0) { KDISPATCH(k, PB) }
#undef PB
  if (poff && cnt && max_pad > 0) {
    dim3 g((unsigned)max_pad, (unsigned)E);
    zero_pad_kernel<T><<<g, 128, 0, st>>>(dy, H, poff, cnt);
  }
  B200MOE_CHECK_LAUNCH("permute_bwd");
  return B200MOE_OK;
}

int permute_bwd(const void* u, int dt, int64_t Tn, int64_t H, int k, const int32_t* pr,
                const float* gates, const void* y, void* dy, float* dg, const int32_t* poff,
                const int32_t* cnt, int E, int64_t max_pad, cudaStream_t st) {
  if (dt == B200MOE_BF16)
    return launch_permute_bwd(static_cast<const __nv_bfloat16*>(u), Tn, H, k, pr, gates,
                              static_cast<const __nv_bfloat16*>(y),
                              static_cast<__nv_bfloat16*>(dy), dg, poff, cnt, E, max_pad, st);
  return launch_permute_bwd(static_cast<const float*>(u), Tn, H, k, pr, gates,
                            static_cast<const float*>(y), static_cast<float*>(dy), dg, poff, cnt,
                            E, max_pad, st);
}

template <typename Tin, typename Tout>
static int launch_combine(const Tin* rows, int64_t Tn, int64_t H, int k, const int32_t* pr,
                          const float* gates, const float* dz, const float* wgT, int E, Tout* out,
                          int acc, cudaStream_t st, int nparts = 1, int64_t pstride = 0,
                          Tin* rows_out = nullptr) {
  constexpr int TPW = 4;
  const unsigned grid = (unsigned)ceil_div(ceil_div(Tn, TPW), 8);
  bool done = false;
  if constexpr (sizeof(Tin) == 2 && sizeof(Tout) == 2) {
    if (dz && !gates && E <= 8 && H % 8 == 0 && k <= 8 && Tn > 0) {  // (k > 8: combine_vec below)
      // two tokens (2k 16-byte row loads) in flight per thread
      int64_t chunk = std::max<int64_t>(ceil_div(ceil_div(Tn, 148), 8) * 8, 16);
      dim3 g2((unsigned)ceil_div(Tn, chunk), (unsigned)ceil_div(H, CR_COLS));
      auto* ob = reinterpret_cast<__nv_bfloat16*>(out);
      auto* rb = reinterpret_cast<const __nv_bfloat16*>(rows);
#define CR(KM) if (E <= 4) combine_router_kernel<KM, 4, 2><<<g2, 256, 0, st>>>(rb, Tn, H, k, pr, dz, wgT, E, ob, acc, chunk, nparts, pstride); \
               else combine_router_kernel<KM, 8, 2><<<g2, 256, 0, st>>>(rb, Tn, H, k, pr, dz, wgT, E, ob, acc, chunk, nparts, pstride)
      KDISPATCH(k, CR)
#undef CR
      done = true;
    }
  }
  if constexpr (sizeof(Tin) == 2) {
    if (!done && !dz && H % 8 == 0) {
      const unsigned g1 = (unsigned)ceil_div(Tn, 8);
#define CG1(KM) combine_gather_kernel<Tin, Tout, KM, (KM <= 2 ? 4 : (KM <= 4 ? 2 : 1))><<<g1, 256, 0, st>>>(rows, Tn, H, k, pr, gates, out, acc, nparts, pstride, rows_out)
      if (Tn > 0) { KDISPATCH(k, CG1) }
#undef CG1
      done = true;
    }
  }
  if (!done && nparts > 1) {
    set_error("combine: ETP partial rows need bf16 rows, H %% 8 == 0 and (with dz) E <= 8, k <= 8");
    return B200MOE_EUNSUPPORTED;
  }
  if (done) {
  } else if (H % 8 == 0) {
#define CV(KM) combine_vec_kernel<Tin, Tout, KM, TPW><<<grid, 256, 0, st>>>(rows, Tn, H, k, pr, gates, dz, wgT, E, out, acc)
    if (Tn > 0) { KDISPATCH(k, CV) }
#undef CV
  } else {
#define CB(KM) combine_kernel<Tin, Tout, KM, TPW><<<grid, 256, 0, st>>>(rows, Tn, H, k, pr, gates, dz, wgT, E, out, acc)
    if (Tn > 0) { KDISPATCH(k, CB) }
#undef CB
  }
  B200MOE_CHECK_LAUNCH("combine");
  return B200MOE_OK;
}

int combine_parts(const void* rows, int nparts, int64_t pstride, void* rows_out, int64_t Tn, int64_t H, int k,
                  const int32_t* pr, const float* gates, const float* dz, const float* wgT, int E, void* out,
                  int acc, cudaStream_t st) {
  return launch_combine(static_cast<const __nv_bfloat16*>(rows), Tn, H, k, pr, gates, dz, wgT, E,
                        static_cast<__nv_bfloat16*>(out), acc, st, nparts, pstride,
                        static_cast<__nv_bfloat16*>(rows_out));
}

int combine(const void* rows, int dt, int64_t Tn, int64_t H, int k, const int32_t* pr,
            const float* gates, const float* dz, const float* wgT, int E, void* out, int odt,
            int acc, cudaStream_t st) {
  if (dt == B200MOE_BF16) {
    auto r = static_cast<const __nv_bfloat16*>(rows);
    if (odt == B200MOE_BF16)
      return launch_combine(r, Tn, H, k, pr, gates, dz, wgT, E, static_cast<__nv_bfloat16*>(out), acc, st);
    return launch_combine(r, Tn, H, k, pr, gates, dz, wgT, E, static_cast<float*>(out), acc, st);
  }
  auto r = static_cast<const float*>(rows);
  if (odt == B200MOE_BF16)
    return launch_combine(r, Tn, H, k, pr, gates, dz, wgT, E, static_cast<__nv_bfloat16*>(out), acc, st);
  return launch_combine(r, Tn, H, k, pr, gates, dz, wgT, E, static_cast<float*>(out), acc, st);
}

}  // namespace b200moe
