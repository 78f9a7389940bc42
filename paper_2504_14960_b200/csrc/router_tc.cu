// K1 fused router forward on the 5th-gen tensor cores (sm_100a):
//
//   logits = x @ W_g       (router.py:145)  tcgen05.mma, x streamed once by TMA
//   scores = softmax/sigmoid(logits) in float64    (router.py:146-149)
//   top-k  (score desc, expert id asc), gates raw or renormalised (:150-153)
//
// W_g is fp32; it enters the MMA as three bf16 parts hi + mid + lo == W_g
// exactly (split on the host once, GatingParams.device_w_g_tc), stacked as
// the N dimension: B = [hi | mid | lo] ([NP, H], rows p*EP + e, zero padded
// to NP = round_up(3 EP, 16)).  bf16 x bf16 products are exact in fp32, so
// the accumulator holds the three partial dot products of the fp32 logit,
// which the epilogue folds in fixed order (hi + mid) + lo.
//
// One CTA per 128-token tile (M = 128, N = NP, K = H): warp 0 lane 0 is the
// TMA producer (x tile 128 x 64 + the W parts 64 x NP per stage, 128B
// swizzle), warp 1 lane 0 issues tcgen05.mma into a [128 x NP] fp32 TMEM
// accumulator, warp 2 owns the TMEM allocation, warps 4..7 are the epilogue:
// one thread per token reads its accumulator row (tcgen05.ld), and for
// E <= 32 does softmax/sigmoid and the top-k in registers (logits, scores,
// ids and gates written once); for larger E it writes the logits and the
// warp-per-token top-k kernel follows (router.cu).
//
// Non-finite logits (non-finite tokens or gating weights, router.py:141-144)
// set bit 0 of *status and the token gets the valid placeholder routing
// 0..k-1, so nothing downstream indexes out of range; the host raises
// NumericError when it reads the status (dispatcher.py, no blocking check).
#include "tcgen05.cuh"

namespace b200moe {

int router_topk(const float*, int64_t, int, int, int, int, float*, int32_t*, float*, double*, int32_t*,
                cudaStream_t);

namespace rtc {
using namespace tc;

constexpr int BM = 128, BK = 64;

__host__ __device__ constexpr int np_of(int ep) { return (3 * ep + 15) / 16 * 16; }
__host__ __device__ constexpr int tmem_cols(int np) { return np <= 32 ? 32 : np <= 64 ? 64 : np <= 128 ? 128 : 256; }

// kind::f16 instruction descriptor: bf16 A/B (K-major), fp32 D, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

struct Args {
  int64_t T;
  int E, k, gate_fn, renorm, nkb, stages;
  int bm;    // tokens per CTA tile (multiple of 8, <= 128): the grid covers every SM
  int ksub;  // 64-column K blocks per pipeline stage (stages = smem slots / ksub)
  int krot;  // K-walk stagger between CTAs (blocks per CTA index; 0 = none)
  float* logits;
  float* scores;
  int32_t* idx;
  float* gates;
  double* gates64;
  int32_t* status;
};

template <int EP>
__device__ __forceinline__ void epilogue_row(const Args& a, int64_t t, const float (&lg)[EP]) {
  const int E = a.E, k = a.k;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) bad |= !isfinite(lg[e]);
  float* lrow = a.logits + t * E;
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) lrow[e] = lg[e];
  if (EP > 32) return;  // logits only; router_topk follows
  if (bad) {
    if (a.status) atomicOr(a.status, 1);
    for (int e = 0; e < E; ++e) a.scores[t * E + e] = 0.f;
    for (int s = 0; s < k; ++s) {
      a.idx[t * k + s] = s;
      a.gates[t * k + s] = 0.f;
      if (a.gates64) a.gates64[t * k + s] = 0.0;
    }
    return;
  }
  double s[EP];
  if (a.gate_fn == B200MOE_GATE_SOFTMAX) {
    double m = -1.0e308;
#pragma unroll
    for (int e = 0; e < EP; ++e)
      if (e < E) m = fmax(m, (double)lg[e]);
    double sum = 0.0;
#pragma unroll
    for (int e = 0; e < EP; ++e) {
      s[e] = e < E ? exp((double)lg[e] - m) : 0.0;
      sum += s[e];
    }
#pragma unroll
    for (int e = 0; e < EP; ++e) s[e] = s[e] / sum;
  } else {
#pragma unroll
    for (int e = 0; e < EP; ++e) s[e] = e < E ? 1.0 / (1.0 + exp(-(double)lg[e])) : 0.0;
  }
  float* srow = a.scores + t * E;
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) srow[e] = (float)s[e];
  // k rounds of arg-max over (score desc, id asc): strict > in ascending id
  // order keeps the lower id on ties (the stable argsort of router.py:123)
  uint64_t taken = 0;
  double raw[32];
  double raw_sum = 0.0;
  for (int r = 0; r < k; ++r) {
    double best = -1.0;
    int bid = 0;
#pragma unroll
    for (int e = 0; e < EP; ++e) {
      if (e < E && !((taken >> e) & 1ull) && s[e] > best) {
        best = s[e];
        bid = e;
      }
    }
    taken |= 1ull << bid;
    raw[r] = best;
    raw_sum += best;
    a.idx[t * k + r] = bid;
  }
  for (int r = 0; r < k; ++r) {
    const double g = a.renorm ? raw[r] / raw_sum : raw[r];
    a.gates[t * k + r] = (float)g;
    if (a.gates64) a.gates64[t * k + r] = g;
  }
}

template <int EP>
__global__ void __launch_bounds__(256, 1) router_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                                                           const __grid_constant__ CUtensorMap map_w,
                                                           const Args a) {
  constexpr int NP = np_of(EP);
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = NP * BK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int COLS = tmem_cols(NP);
  const int S = a.stages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base, sB = base + S * A_BYTES;
  const uint32_t bars = base + S * STAGE;
  const uint32_t full_bar = bars, empty_bar = bars + 8 * S, done_bar = bars + 16 * S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + S * STAGE + 16 * S + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * a.bm;
  // the TMA box is bm rows (the rest of the 128-row A tile is never read
  // back: the MMA's extra accumulator rows are ignored by the epilogue)
  const uint32_t a_tx = (uint32_t)a.bm * BK * 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full_bar + 8 * i, 1);
      mbar_init(empty_bar + 8 * i, 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    prefetch_map(&map_x);
    prefetch_map(&map_w);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Every tile walks K from block 0 (krot = 0, the default): a token's fp32
  // logit is then the same whatever tile -- i.e. whatever position in
  // whatever rank's block -- it sits in, so splitting tokens over ranks
  // changes no routing bit (tests/test_gpu_random_layers.py).  krot > 0
  // staggers the CTAs' K walks (B200MOE_ROUTER_KROT, experiments: 31.2 vs
  // 31.7 us at C2, not worth the batch-position dependence).
  const int kb_rot = (int)((blockIdx.x * (unsigned)a.krot) % (unsigned)a.nkb);
  // a pipeline stage holds KS consecutive 64-column K blocks (KS smem slots,
  // one barrier pair): each x row is then read as KS x 128 contiguous bytes
  // per stage instead of 128 B -- DRAM page locality for the 8 KB-strided rows
  const int KS = a.ksub, G = S / KS, nst = (a.nkb + KS - 1) / KS;
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nst; ++i) {
        const int nsub = min(KS, a.nkb - i * KS);
        mbar_wait(empty_bar + 8 * g, phase ^ 1);
        mbar_expect_tx(full_bar + 8 * g, (uint32_t)nsub * (a_tx + B_BYTES));
        for (int sub = 0; sub < nsub; ++sub) {
          const int kk = i * KS + sub;
          const int kb = kk + kb_rot < a.nkb ? kk + kb_rot : kk + kb_rot - a.nkb;
          const int slot = g * KS + sub;
          tma_load_3d(&map_x, sA + slot * A_BYTES, full_bar + 8 * g, kb * BK, (int)m0, 0);
          tma_load_3d(&map_w, sB + slot * B_BYTES, full_bar + 8 * g, kb * BK, 0, 0);
        }
        if (++g == G) {
          g = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_n(NP);
      int g = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nst; ++i) {
        const int nsub = min(KS, a.nkb - i * KS);
        mbar_wait(full_bar + 8 * g, phase);
        tc_fence_after();
        for (int sub = 0; sub < nsub; ++sub) {
          const int slot = g * KS + sub;
          const uint32_t a_s = sA + slot * A_BYTES, b_s = sB + slot * B_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma(tmem, smem_desc(a_s + k * 32, 16, 1024), smem_desc(b_s + k * 32, 16, 1024), idesc,
                   (i | sub | k) != 0);
        }
        tc_commit(empty_bar + 8 * g);
        if (++g == G) {
          g = 0;
          phase ^= 1;
        }
      }
      tc_commit(done_bar);
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    mbar_wait(done_bar, 0);
    tc_fence_after();
    const uint32_t t_row = tmem + ((uint32_t)(32 * q) << 16);
    // columns p * EP + e arrive in increasing order, so lg = (hi + mid) + lo
    constexpr int NCH = (3 * EP + 31) / 32;
    float lg[EP];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      uint32_t v[32];
      tmem_ld32(t_row + c * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = c * 32 + j;
        if (col < EP) lg[col] = __uint_as_float(v[j]);
        else if (col < 3 * EP) lg[col % EP] += __uint_as_float(v[j]);
      }
    }
    const int r = 32 * q + lane;
    const int64_t t = m0 + r;
    if (r < a.bm && t < a.T) epilogue_row<EP>(a, t, lg);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
  }
}

template <int EP>
static int launch(const void* x, int64_t T, int64_t H, const void* w, Args a, cudaStream_t st) {
  constexpr int NP = np_of(EP);
  constexpr int STAGE = BM * BK * 2 + NP * BK * 2;
  // tile height 128.  Experiments: B200MOE_ROUTER_BM=n (multiple of 8), or
  // 0 = the fewest rows that spread T over every SM in one wave (112 at
  // T = 16384: measured no faster)
  static const int bm_env = [] {
    const char* e = getenv("B200MOE_ROUTER_BM");
    return e ? atoi(e) : -1;
  }();
  int bm = BM;
  if (bm_env == 0) bm = (int)std::min<int64_t>(BM, std::max<int64_t>(8, ceil_div(ceil_div(T, num_sms()), 8) * 8));
  if (bm_env >= 8 && bm_env <= BM && bm_env % 8 == 0) bm = bm_env;
  a.bm = bm;
  CUtensorMap mx, mw;
  int rc = make_map(&mx, x, (uint64_t)H, (uint64_t)T, 1, (uint64_t)H, (uint64_t)H * T, (uint32_t)bm);
  if (rc) return rc;
  rc = make_map(&mw, w, (uint64_t)H, (uint64_t)NP, 1, (uint64_t)H, (uint64_t)H * NP, NP);
  if (rc) return rc;
  a.nkb = (int)ceil_div(H, BK);
  a.stages = std::max(2, std::min(8, (196 * 1024) / STAGE));  // smem slots of one K block
  static const int ks_env = [] {
    const char* e = getenv("B200MOE_ROUTER_KSUB");
    return e ? atoi(e) : 0;
  }();
  // measured neutral (C2: 30.1-31.2 us for ksub 1 / 2 / 4, 128- or 112-row
  // tiles alike): the kernel's ~30 us is not DRAM-locality or SM-count bound
  a.ksub = ks_env >= 1 ? std::min(ks_env, a.stages / 2) : 1;
  a.stages = a.stages / a.ksub * a.ksub;
  static const int krot_env = [] {
    const char* e = getenv("B200MOE_ROUTER_KROT");
    return e ? atoi(e) : 0;
  }();
  a.krot = krot_env;
  const int smem = 1024 + a.stages * STAGE + 16 * a.stages + 64;
  if (int e = ensure_max_smem(router_tc_kernel<EP>, 232448, "router_fwd_tc")) return e;
  router_tc_kernel<EP><<<(unsigned)ceil_div(T, bm), 256, smem, st>>>(mx, mw, a);
  B200MOE_CHECK_LAUNCH("router_fwd_tc");
  if (EP > 32)
    return router_topk(a.logits, T, a.E, a.k, a.gate_fn, a.renorm, a.scores, a.idx, a.gates, a.gates64,
                       a.status, st);
  return B200MOE_OK;
}

// ---------------------------------------------------------------------------
// dW_g = x^T dz (dispatcher.py:489) on the tensor cores: M = H (128 columns of
// x per tile), N = NB (the three exact bf16 parts of dz, [T, NB] written by
// router_bwd, cols p * EPW + e, zero padded to a multiple of 64), K = tokens.
// Both operands are MN-major in memory (x is [T, H], dz parts [T, NB]): the
// TMA boxes are {64 columns, 64 tokens} with 128B swizzle.  The tokens are
// split over the grid's y dimension; each CTA folds the parts of its
// accumulator rows, (hi + mid) + lo, into an fp32 partial dW_g [split, H, E]
// which router_wgrad_reduce_kernel sums in split order (deterministic).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr uint32_t idesc_mn(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

struct WArgs {
  int64_t T, H;
  int E, epw, kb_per_split, nkb, stages;
  float* part;
};

template <int EPW>
__global__ void __launch_bounds__(256) router_wgrad_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                                                              const __grid_constant__ CUtensorMap map_d,
                                                              const WArgs a) {
  constexpr int NB = (3 * EPW + 63) / 64 * 64;
  constexpr int A_BYTES = BM * BK * 2, B_BYTES = NB * BK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int COLS = tmem_cols(NB);
  const int S = a.stages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base, sB = base + S * A_BYTES;
  const uint32_t bars = base + S * STAGE;
  const uint32_t full_bar = bars, empty_bar = bars + 8 * S, done_bar = bars + 16 * S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + S * STAGE + 16 * S + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int kb0 = blockIdx.y * a.kb_per_split;
  const int kb1 = min(a.nkb, kb0 + a.kb_per_split);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full_bar + 8 * i, 1);
      mbar_init(empty_bar + 8 * i, 1);
    }
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    prefetch_map(&map_x);
    prefetch_map(&map_d);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int nk = kb1 - kb0;
  const int kb_rot = nk > 0 ? (int)((blockIdx.x * 5u) % (unsigned)nk) : 0;  // staggered walk, as above
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nk; ++i) {
        const int kb = kb0 + (i + kb_rot < nk ? i + kb_rot : i + kb_rot - nk);
        mbar_wait(empty_bar + 8 * stage, phase ^ 1);
        mbar_expect_tx(full_bar + 8 * stage, STAGE);
#pragma unroll
        for (int i = 0; i < BM / 64; ++i)  // x: {64 columns, 64 tokens} per box
          tma_load_3d(&map_x, sA + stage * A_BYTES + i * 8192, full_bar + 8 * stage, m0 + 64 * i, kb * BK, 0);
#pragma unroll
        for (int i = 0; i < NB / 64; ++i)
          tma_load_3d(&map_d, sB + stage * B_BYTES + i * 8192, full_bar + 8 * stage, 64 * i, kb * BK, 0);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_mn(NB);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nk; ++i) {
        mbar_wait(full_bar + 8 * stage, phase);
        tc_fence_after();
        const uint32_t a_s = sA + stage * A_BYTES, b_s = sB + stage * B_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)  // MN-major: +16 K-rows = 2 KB per step
          tc_mma(tmem, smem_desc(a_s + k * 2048, 8192, 1024), smem_desc(b_s + k * 2048, 8192, 1024), idesc,
                 (i | k) != 0);
        tc_commit(empty_bar + 8 * stage);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (kb1 > kb0) tc_commit(done_bar);
      else mbar_arrive(done_bar);
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    mbar_wait(done_bar, 0);
    tc_fence_after();
    const uint32_t t_row = tmem + ((uint32_t)(32 * q) << 16);
    float dw[EPW];
#pragma unroll
    for (int e = 0; e < EPW; ++e) dw[e] = 0.f;
    if (kb1 > kb0) {
      // parts arrive in column order p * EPW + e: dw = (hi + mid) + lo
#pragma unroll
      for (int c = 0; c < (3 * EPW + 31) / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(t_row + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = c * 32 + j;
          if (col < 3 * EPW) dw[col % EPW] += __uint_as_float(v[j]);
        }
      }
    }
    const int64_t h = (int64_t)m0 + 32 * q + lane;
    if (h < a.H) {
      float* o = a.part + ((int64_t)blockIdx.y * a.H + h) * a.E;
#pragma unroll
      for (int e = 0; e < EPW; ++e)
        if (e < a.E) o[e] = dw[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
  }
}

__global__ void wgrad_reduce_kernel(const float* __restrict__ part, int64_t nsplit, int64_t HE,
                                    float* __restrict__ dwg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < HE; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t c = 0; c < nsplit; ++c) s += part[c * HE + i];
    dwg[i] = s;
  }
}

template <int EPW>
static int launch_wgrad(const void* x, const void* dz_parts, int64_t T, int64_t H, int E, int epw, float* dwg,
                        void* ws, size_t ws_bytes, cudaStream_t st) {
  constexpr int NB = (3 * EPW + 63) / 64 * 64;
  constexpr int STAGE = BM * BK * 2 + NB * BK * 2;
  CUtensorMap mx, md;
  int rc = make_map(&mx, x, (uint64_t)H, (uint64_t)T, 1, (uint64_t)H, (uint64_t)H * T, 64);
  if (rc) return rc;
  rc = make_map(&md, dz_parts, (uint64_t)NB, (uint64_t)T, 1, (uint64_t)NB, (uint64_t)NB * T, 64);
  if (rc) return rc;
  WArgs a{T, H, E, epw, 0, (int)ceil_div(T, BK), 0, static_cast<float*>(ws)};
  // two CTAs per SM when four stages fit in half of the shared memory
  a.stages = 4;
  const int smem = 1024 + a.stages * STAGE + 16 * a.stages + 64;
  const int per_sm = smem <= 113 * 1024 ? 2 : 1;
  const int mt = (int)ceil_div(H, BM);
  int split = std::max(1, std::min(a.nkb, num_sms() * per_sm / mt));
  a.kb_per_split = (int)ceil_div(a.nkb, split);
  split = (int)ceil_div(a.nkb, a.kb_per_split);
  if ((size_t)split * H * E * sizeof(float) > ws_bytes) {
    set_error("router_wgrad_tc: workspace too small");
    return B200MOE_EINVAL;
  }
  if (int e = ensure_max_smem(router_wgrad_tc_kernel<EPW>, 232448, "router_wgrad_tc")) return e;
  router_wgrad_tc_kernel<EPW><<<dim3((unsigned)mt, (unsigned)split), 256, smem, st>>>(mx, md, a);
  const int64_t HE = H * E;
  wgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(HE, 256), 148 * 8), 256, 0, st>>>(
      a.part, split, HE, dwg);
  B200MOE_CHECK_LAUNCH("router_wgrad_tc");
  return B200MOE_OK;
}

}  // namespace rtc

// dz-part layout of the tensor-core x^T dz: cols p * epw + e, nb columns
int router_parts_layout(int E, int* epw, int* nb) {
  const int ep = E <= 8 ? 8 : E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : 0;
  if (!ep) return 0;
  *epw = ep;
  *nb = (3 * ep + 63) / 64 * 64;
  return 1;
}

size_t router_wgrad_tc_ws_bytes(int64_t T, int64_t H, int E) {
  (void)T;
  return (size_t)std::max(1, num_sms() * 2) * (size_t)H * E * sizeof(float);
}

int router_wgrad_tc(const void* x, const void* dz_parts, int64_t T, int64_t H, int E, float* dwg, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  int epw = 0, nb = 0;
  if (!router_parts_layout(E, &epw, &nb)) {
    set_error("router_wgrad_tc: E=%d > 64 unsupported", E);
    return B200MOE_EUNSUPPORTED;
  }
  if (T == 0) return cudaMemsetAsync(dwg, 0, (size_t)H * E * sizeof(float), st) == cudaSuccess ? B200MOE_OK
                                                                                              : B200MOE_ELAUNCH;
  (void)nb;
  if (epw == 8) return rtc::launch_wgrad<8>(x, dz_parts, T, H, E, epw, dwg, ws, ws_bytes, st);
  if (epw == 16) return rtc::launch_wgrad<16>(x, dz_parts, T, H, E, epw, dwg, ws, ws_bytes, st);
  if (epw == 32) return rtc::launch_wgrad<32>(x, dz_parts, T, H, E, epw, dwg, ws, ws_bytes, st);
  return rtc::launch_wgrad<64>(x, dz_parts, T, H, E, epw, dwg, ws, ws_bytes, st);
}

int router_fwd_tc_np(int E) {
  const int ep = E <= 8 ? 8 : E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : 0;
  return ep ? rtc::np_of(ep) : 0;
}

int router_fwd_tc(const void* x, int64_t T, int64_t H, const void* w_parts, int E, int k, int gate_fn,
                  int renorm, float* logits, float* scores, int32_t* idx, float* gates, double* gates64,
                  int32_t* status, cudaStream_t st) {
  if (T == 0) return B200MOE_OK;
  rtc::Args a{T, E, k, gate_fn, renorm, 0, 0, rtc::BM, 1, 0, logits, scores, idx, gates, gates64, status};
  if (E <= 8) return rtc::launch<8>(x, T, H, w_parts, a, st);
  if (E <= 16) return rtc::launch<16>(x, T, H, w_parts, a, st);
  if (E <= 32) return rtc::launch<32>(x, T, H, w_parts, a, st);
  if (E <= 64) return rtc::launch<64>(x, T, H, w_parts, a, st);
  set_error("router_fwd_tc: E=%d > 64 unsupported", E);
  return B200MOE_EUNSUPPORTED;
}

}  // namespace b200moe
