// Portable grouped GEMM (CUDA cores, fp32 accumulation) and the elementwise
// expert activations.  Used for the fp32 parity mode (the reference's float64
// tolerances cannot be met with tensor-core TF32/BF16 inputs) and as the
// on-device cross-check of the tcgen05 kernel.  Reference arithmetic:
// experts.py:130-172.
#include "common.cuh"

namespace b200moe {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename Tin, typename TinB, typename Tout>
__global__ void __launch_bounds__(256) gemm_simt_kernel(b200moe_gemm_args a) {
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const Tin* A = static_cast<const Tin*>(a.A);
  const TinB* B = static_cast<const TinB*>(a.B);
  Tout* C = static_cast<Tout*>(a.C);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t n0 = (int64_t)blockIdx.x * SB_N;

  // Work items: grouped-M -> the row block may intersect several groups;
  // grouped-K -> blockIdx.z is the group.
  int g_begin, g_end;
  int64_t m_lo, m_hi;
  if (a.grouped_dim == 0) {
    m_lo = (int64_t)blockIdx.y * SB_M;
    m_hi = m_lo + SB_M;
    if (a.group_end) {  // explicit [begin, end) per group, possibly with gaps
      g_begin = 0;
      g_end = a.G;
    } else {
      if (m_lo >= a.group_off[a.G]) return;
      g_begin = 0;
      while (g_begin < a.G && a.group_off[g_begin + 1] <= m_lo) ++g_begin;
      g_end = g_begin;
      while (g_end < a.G && a.group_off[g_end] < m_hi) ++g_end;
    }
  } else {
    g_begin = blockIdx.z;
    g_end = g_begin + 1;
    m_lo = (int64_t)blockIdx.y * SB_M;
    m_hi = m_lo + SB_M;
    if (m_lo >= a.M) return;
  }
  for (int g = g_begin; g < g_end; ++g) {
    int64_t mbase, mcount, kbase, K, b_off, c_off;
    const int64_t gend = a.group_end ? a.group_end[g] : a.group_off[g + 1];
    if (a.grouped_dim == 0) {
      const int64_t lo = max(m_lo, (int64_t)a.group_off[g]);
      const int64_t hi = min(m_hi, gend);
      if (hi <= lo) continue;
      mbase = lo;
      mcount = hi - lo;
      kbase = 0;
      K = a.K;
      const int64_t bg = a.group_expert ? a.group_expert[g] : g;
      b_off = bg * a.b_sg;
      c_off = 0;
    } else {
      mbase = m_lo;
      mcount = min((int64_t)SB_M, a.M - m_lo);
      kbase = a.group_off[g];
      K = gend - kbase;
      b_off = 0;
      c_off = (int64_t)g * a.c_sg;
    }
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int64_t k0 = 0; k0 < K; k0 += SB_K) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = tid + i * 256;
        int m, kk;
        if (a.a_sk == 1) { kk = e % SB_K; m = e / SB_K; }
        else { m = e % SB_M; kk = e / SB_M; }
        float v = 0.f;
        if (m < mcount && k0 + kk < K)
          v = to_f32(A[(mbase + m) * a.a_sm + (kbase + k0 + kk) * a.a_sk]);
        As[kk][m] = v;
        int n;
        if (a.b_sn == 1) { n = e % SB_N; kk = e / SB_N; }
        else { kk = e % SB_K; n = e / SB_K; }
        float w = 0.f;
        if (n0 + n < a.N && k0 + kk < K)
          w = to_f32(B[b_off + (kbase + k0 + kk) * a.b_sk + (n0 + n) * a.b_sn]);
        Bs[kk][n] = w;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < SB_K; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = ty * 4 + i;
      if (m >= mcount) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = n0 + tx * 4 + j;
        if (n >= a.N) continue;
        Tout* p = C + c_off + (mbase + m) * a.ldc + n;
        float v = acc[i][j];
        if (a.accumulate) v += to_f32(*p);
        *p = from_f32<Tout>(v);
      }
    }
  }
}

int gemm_simt(const b200moe_gemm_args* a, cudaStream_t st) {
  dim3 grid;
  grid.x = (unsigned)ceil_div(a->N, SB_N);
  if (a->grouped_dim == 0) {
    grid.y = (unsigned)ceil_div(a->max_rows > 0 ? a->max_rows : 1, SB_M);
    grid.z = 1;
  } else {
    grid.y = (unsigned)ceil_div(a->M, SB_M);
    grid.z = (unsigned)a->G;
  }
  using bf = __nv_bfloat16;
  const int ka = a->dtype_in == B200MOE_BF16, kb = a->dtype_b == B200MOE_BF16,
            kc = a->dtype_out == B200MOE_BF16;
#define GS(TA, TB, TC) gemm_simt_kernel<TA, TB, TC><<<grid, 256, 0, st>>>(*a)
  switch (ka * 4 + kb * 2 + kc) {
    case 0: GS(float, float, float); break;
    case 1: GS(float, float, bf); break;
    case 2: GS(float, bf, float); break;
    case 3: GS(float, bf, bf); break;
    case 4: GS(bf, float, float); break;
    case 5: GS(bf, float, bf); break;
    case 6: GS(bf, bf, float); break;
    default: GS(bf, bf, bf); break;
  }
#undef GS
  B200MOE_CHECK_LAUNCH("gemm_simt");
  return B200MOE_OK;
}

// ---------------------------------------------------------------- activations
__device__ __forceinline__ float gelu_f(float x) {
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.f + tanhf(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * x * x);
}
__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

template <typename T>
__global__ void act_fwd_kernel(const T* __restrict__ pre, int act, const int32_t* __restrict__ goff,
                               int G, int64_t F, T* __restrict__ h) {
  const int64_t rows = goff[G];
  const int64_t n = rows * F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, f = i % F;
    float out;
    if (act == B200MOE_ACT_SWIGLU) {
      const int64_t base = r * 2 * F + (f / 32) * 64 + (f % 32);
      const float g = to_f32(pre[base]), u = to_f32(pre[base + 32]);
      out = g * sigm(g) * u;
    } else {
      const float p = to_f32(pre[i]);
      out = act == B200MOE_ACT_RELU ? fmaxf(p, 0.f) : gelu_f(p);
    }
    h[i] = from_f32<T>(out);
  }
}

template <typename T>
__global__ void act_bwd_kernel(const T* __restrict__ dh, const T* __restrict__ pre, int act,
                               const int32_t* __restrict__ goff, int G, int64_t F,
                               T* __restrict__ dpre) {
  const int64_t rows = goff[G];
  const int64_t n = rows * F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, f = i % F;
    const float d = to_f32(dh[i]);
    if (act == B200MOE_ACT_SWIGLU) {
      const int64_t base = r * 2 * F + (f / 32) * 64 + (f % 32);
      const float g = to_f32(pre[base]), u = to_f32(pre[base + 32]);
      const float s = sigm(g);
      dpre[base] = from_f32<T>(d * u * s * (1.f + g * (1.f - s)));
      dpre[base + 32] = from_f32<T>(d * g * s);
    } else {
      const float p = to_f32(pre[i]);
      const float gr = act == B200MOE_ACT_RELU ? (p > 0.f ? 1.f : 0.f) : gelu_grad_f(p);
      dpre[i] = from_f32<T>(d * gr);
    }
  }
}

int act_fwd(const void* pre, int dt, int act, const int32_t* goff, int G, int64_t max_rows,
            int64_t F, void* h, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(max_rows * F, 256), 148 * 16);
  if (grid == 0) return B200MOE_OK;
  if (dt == B200MOE_BF16)
    act_fwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(pre), act, goff, G, F,
                                         static_cast<__nv_bfloat16*>(h));
  else
    act_fwd_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(pre), act, goff, G, F,
                                         static_cast<float*>(h));
  B200MOE_CHECK_LAUNCH("act_fwd");
  return B200MOE_OK;
}

int act_bwd(const void* dh, const void* pre, int dt, int act, const int32_t* goff, int G,
            int64_t max_rows, int64_t F, void* dpre, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(max_rows * F, 256), 148 * 16);
  if (grid == 0) return B200MOE_OK;
  if (dt == B200MOE_BF16)
    act_bwd_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(dh),
                                         static_cast<const __nv_bfloat16*>(pre), act, goff, G, F,
                                         static_cast<__nv_bfloat16*>(dpre));
  else
    act_bwd_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(dh),
                                         static_cast<const float*>(pre), act, goff, G, F,
                                         static_cast<float*>(dpre));
  B200MOE_CHECK_LAUNCH("act_bwd");
  return B200MOE_OK;
}

}  // namespace b200moe
