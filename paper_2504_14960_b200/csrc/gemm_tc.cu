// K3: grouped expert GEMM on 5th-gen tensor cores (sm_100a).
//
//   tcgen05.mma (kind::f16, bf16 x bf16 -> fp32 in TMEM), operands staged in
//   shared memory by TMA (cp.async.bulk.tensor, 128B swizzle) through an
//   mbarrier ring, accumulators double-buffered in TMEM (2 x 256 columns) so
//   the epilogue of tile i overlaps the MMAs of tile i+1.  Persistent CTAs
//   (one per SM) walk a static tile schedule built from the group offsets in
//   device memory, so variable per-expert token counts never reach the host.
//
//   warp 0      TMA producer (one lane)
//   warp 1      MMA issuer   (one lane)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld -> fused activation -> global stores
//
// Reference arithmetic: experts.py:130-172 (forward x@W1, act, @W2; backward
// dW2 = act^T dy, dh = dy W2^T, dpre = dh*act', dW1 = x^T dpre, dx = dpre W1^T).
#include <cuda.h>

#include <atomic>

#include "common.cuh"
#include "tcgen05.cuh"

namespace b200moe {

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int TMEM_COLS = 512;  // 2 accumulator buffers of BN fp32 columns
constexpr int MAX_G = 512;
constexpr int NUM_THREADS = 256;
constexpr int STG_BYTES = 128 * 128;  // one epilogue staging tile: 128 rows x 128 B

enum Epi : int {
  EPI_STORE = 0,       // C = acc (bf16 or fp32, optional accumulate)
  EPI_SWIGLU_FWD = 1,  // acc = [gate|up] interleaved 32-col blocks -> pre (bf16), h = silu(g)*u
  EPI_SWIGLU_BWD = 2,  // acc = dh [.. F]; reads pre -> dpre (interleaved)
  EPI_ACT_FWD = 3,     // acc = pre -> pre (bf16), h = act(pre)
  EPI_ACT_BWD = 4,     // acc = dh; reads pre -> dpre = dh * act'(pre)
  EPI_SCATTER = 5,     // bf16 rows straight to the ranks they came from (peer memory)
};

struct Params {
  int G;
  int grouped_k;   // 0: groups over M, 1: groups over K
  int64_t M, N, K; // fixed extents (M for grouped-K, K for grouped-M)
  const int32_t* goff;
  const int32_t* gexp;
  const int32_t* gend;  // nullable: explicit group ends (gaps between groups)
  int64_t max_rows;
  // epilogue
  int epi;
  int act;         // relu/gelu for EPI_ACT_*
  int out_f32;
  int accumulate;
  void* C;
  int64_t ldc;
  int64_t c_sg;
  void* H;         // second output (h) for *_FWD epilogues
  int64_t ldh;
  const void* PRE; // pre-activation input for *_BWD epilogues
  int64_t ldpre;
  int panel_m;     // raster panel height in m-tiles
  int tile_m;      // rows per tile: 128 (1 CTA) or 256 (CTA pair)
  int debug_ops;      // energy experiments only: 1 = operand loads from one L2-hot block, 2 = none
  int debug_nostore;  // perf experiments only: 1 = no epilogue global traffic, 2 = no bulk
                      // stores, 3 = SwiGLU backward without its pre loads
  int use_tma;        // output tensor maps are valid (TMA-store epilogue)
  // EPI_SCATTER: row r -> peer_base[origin[2r]] + scatter_off + origin[2r+1] * ldc * 2
  const int32_t* origin;
  const uint64_t* peer_base;
  int64_t scatter_off;
  // grouped-K weight gradient of the SwiGLU W1: output rows are packed rows
  // ([32 gate | 32 up] per 64) and are stored de-interleaved ([gate | up])
  int64_t glu_f;
  int store_hint;  // L2 evict_first policy on the epilogue's bulk stores
  int kstagger;    // K walk of a tile starts at (n-tile * kstagger) mod nkb (0: off)
};

// packed SwiGLU row -> [gate | up] row (rows come in 32-row halves)
__device__ __forceinline__ int64_t glu_row(int64_t m, int64_t F) {
  const int64_t b = m >> 6, w = m & 63;
  return w < 32 ? b * 32 + w : F + b * 32 + (w - 32);
}

// Per-CTA-group configuration.  CG = 2: a CTA pair (cluster of 2 on one TPC)
// computes a 256 x 256 tile with tcgen05.mma.cta_group::2; each CTA stages
// its 128 rows of A and its 128 rows (half of N) of B, so a stage is 32 KB
// and six stages fit.
// The epilogue stages 128 B row chunks in NSTG swizzled 16 KB buffers and
// writes them with TMA bulk tensor stores.
template <int CG>
struct Cfg {
  static constexpr int STAGES_ = CG == 1 ? 3 : 5;
  static constexpr int NSTG = 3;
  static constexpr int B_CTA = BN / CG;  // B rows staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_CTA * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = 1024 + STAGES_ * STAGE + NSTG * STG_BYTES + 1024 + (MAX_G + 1) * 4;
};


// ---- epilogue: shared-memory staging + TMA bulk tensor stores
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2,
                                                  uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d_hint(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                                       int c2, uint64_t pol) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group.L2::cache_hint"
      " [%0, {%2, %3, %4}], [%1], %5;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                                  int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void st_global_v4(uint64_t addr, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
// one 128-byte row chunk (8 x 16 B) into a 128B-swizzled staging tile
__device__ __forceinline__ void st_row_chunk(uint32_t buf, int r, const uint4 (&v)[8]) {
  const uint32_t row = buf + (uint32_t)r * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) st_shared_v4(row + ((uint32_t)(j ^ (r & 7)) << 4), v[j]);
}

// Ring of NSTG staging tiles shared by the 128 epilogue threads.
template <int NSTG>
struct Stager {
  uint32_t base;
  int buf;
  bool leader;
  bool skip;  // perf experiments: everything but the bulk store itself
  bool hint;  // L2 evict_first on the stores
  uint64_t pol;
  __device__ __forceinline__ uint32_t acquire() {
    if (leader) bulk_wait_read<NSTG - 1>();  // the store that last used this tile has read it
    epi_bar();
    return base + buf * STG_BYTES;
  }
  __device__ __forceinline__ void issue(const CUtensorMap* map, int c0, int c1, int c2, bool reduce) {
    fence_async_smem();  // generic-proxy smem writes -> visible to the TMA (async proxy)
    epi_bar();
    if (leader && !skip) {
      const uint32_t src = base + buf * STG_BYTES;
      if (hint) {
        if (reduce) tma_reduce_add_3d_hint(map, src, c0, c1, c2, pol);
        else tma_store_3d_hint(map, src, c0, c1, c2, pol);
      } else {
        if (reduce) tma_reduce_add_3d(map, src, c0, c1, c2);
        else tma_store_3d(map, src, c0, c1, c2);
      }
      bulk_commit();
    }
    buf = (buf + 1) % NSTG;
  }
  // the staged 128 rows as four 32-row sub-tiles to rows glu_row(row0 + 32 i)
  // (map box: 32 rows)
  __device__ __forceinline__ void issue_glu(const CUtensorMap* map, int c0, int64_t row0, int c2, bool reduce,
                                            int64_t F) {
    fence_async_smem();
    epi_bar();
    if (leader && !skip) {
      const uint32_t src = base + buf * STG_BYTES;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int dr = (int)glu_row(row0 + 32 * i, F);
        if (reduce) {
          if (hint) tma_reduce_add_3d_hint(map, src + i * 4096, c0, dr, c2, pol);
          else tma_reduce_add_3d(map, src + i * 4096, c0, dr, c2);
        } else {
          if (hint) tma_store_3d_hint(map, src + i * 4096, c0, dr, c2, pol);
          else tma_store_3d(map, src + i * 4096, c0, dr, c2);
        }
      }
      bulk_commit();
    }
    buf = (buf + 1) % NSTG;
  }
};

// ---- CTA-pair (cta_group::2) helpers
// A cluster-shared address with this bit cleared names the leader CTA's copy
// of a shared variable (the pair's TMA completions all land on the leader's
// full barrier).
constexpr uint32_t PEER_BIT_MASK = 0xFEFFFFFFu;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t local_bar, uint32_t target_cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_bar), "r"(target_cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load(const CUtensorMap* map, uint32_t dst, uint32_t bar, int c0,
                                         int c1, int c2) {
  if (CG == 1) {
    tma_load_3d(map, dst, bar, c0, c1, c2);
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  if (CG == 1) {
    tc_mma(d_tmem, adesc, bdesc, idesc, accum);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}
// commit the issued MMAs to the barrier at this offset in every CTA of the pair
template <int CG>
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  if (CG == 1) {
    tc_commit(bar);
  } else {
    const uint16_t mask = 0x3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"(mask)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void arrive_all(uint32_t bar) {
  mbar_arrive(bar);
  if (CG == 2) mbar_arrive_remote(bar, 1);
}
template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t slot, uint32_t cols) {
  if (CG == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  if (CG == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}


// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, M (128 or 256), N=BN.
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int m) {
  return (1u << 4)                     // D format f32
         | (1u << 7) | (1u << 10)      // A, B = bf16
         | ((a_mn ? 1u : 0u) << 15)    // A major
         | ((b_mn ? 1u : 0u) << 16)    // B major
         | ((uint32_t)(BN >> 3) << 17) // N
         | ((uint32_t)(m >> 4) << 24); // M
}

// ------------------------------------------------------------- scheduling
struct Tile {
  int g;
  int64_t m0, m_end;  // rows (grouped-M: absolute rows of the padded layout)
  int64_t n0;
  int64_t kbeg;       // first K coordinate (grouped-K: absolute row)
  int nkb;            // number of BK blocks
  int bidx;           // weight/expert index for B (grouped-M)
  int krot;           // first BK block of the tile's K walk (rotated, wraps)
};

// Panel rasterisation inside a group: panels of `pm` m-tiles x all n-tiles,
// m fastest inside a panel.  pm is chosen on the host per GEMM (see
// choose_panel): pm >= mt keeps the whole A operand of a group L2-resident
// while B streams once; a small pm keeps B resident while A streams once;
// when neither fits L2, pm ~ sqrt(148 * BN / BM) balances the k-slab reuse of
// the ~148 concurrent tiles.
__device__ __forceinline__ void raster(int local, int mt, int nt, int pm, int& mb, int& nb) {
  const int full = mt / pm;
  if (local < full * pm * nt) {
    const int pnl = local / (pm * nt), r = local % (pm * nt);
    mb = pnl * pm + r % pm;
    nb = r / pm;
  } else {
    const int rem = mt - full * pm, r = local - full * pm * nt;
    mb = full * pm + r % rem;
    nb = r / rem;
  }
}

__device__ __forceinline__ Tile decode(const Params& p, const int32_t* prefix, int t) {
  // largest g with prefix[g] <= t
  int lo = 0, hi = p.G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  Tile r;
  r.g = lo;
  const int local = t - prefix[lo];
  const int64_t g0 = p.goff[lo], g1 = p.gend ? p.gend[lo] : p.goff[lo + 1];
  const int nt = (int)((p.N + BN - 1) / BN);
  int mb, nb;
  if (!p.grouped_k) {
    // a 256-row pair tile may run past the group end: those rows are
    // computed with this group's weights and masked at store
    const int mt = (int)((g1 - g0 + p.tile_m - 1) / p.tile_m);
    raster(local, mt, nt, p.panel_m, mb, nb);
    r.m0 = g0 + (int64_t)mb * p.tile_m;
    r.m_end = g1;
    r.n0 = (int64_t)nb * BN;
    r.kbeg = 0;
    r.nkb = (int)((p.K + BK - 1) / BK);
    r.bidx = p.gexp ? p.gexp[lo] : lo;
  } else {
    const int mt = (int)((p.M + p.tile_m - 1) / p.tile_m);
    raster(local, mt, nt, p.panel_m, mb, nb);
    r.m0 = (int64_t)mb * p.tile_m;
    r.m_end = p.M;
    r.n0 = (int64_t)nb * BN;
    r.kbeg = g0;
    // groups are 64-aligned in the padded layout; a ragged last group reads
    // past the buffer end, which TMA zero-fills
    r.nkb = (int)((g1 - g0 + BK - 1) / BK);
    r.bidx = 0;
  }
  // the tiles of one m-panel share A's K slabs; staggering their K walks by
  // output column block keeps them from requesting the same slab at the same
  // instant (a row's result depends only on its column block's order, so
  // outputs stay independent of the row layout)
  r.krot = (p.kstagger && r.nkb > 0) ? (int)(((r.n0 / BN) * p.kstagger) % r.nkb) : 0;
  return r;
}

// ------------------------------------------------------------- epilogues
// fast divide (MUFU.RCP): exact limits at +-inf, ~2 ulp, far below bf16 rounding
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.f + __expf(-g)); }
__device__ __forceinline__ float sigmoid_f(float g) { return __fdividef(1.f, 1.f + __expf(-g)); }
__device__ __forceinline__ float gelu_tc(float x) {
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.f + tanhf(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_tc(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * x * x);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t v) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(h);
}
// 32 floats -> 4 x uint4 of bf16 (64 B)
__device__ __forceinline__ void pack32_bf16(const float* f, uint4* out) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    out[i] = make_uint4(pack_bf16(f[8 * i], f[8 * i + 1]), pack_bf16(f[8 * i + 2], f[8 * i + 3]),
                        pack_bf16(f[8 * i + 4], f[8 * i + 5]), pack_bf16(f[8 * i + 6], f[8 * i + 7]));
}
// 32 floats -> 8 x uint4 of fp32 (128 B)
__device__ __forceinline__ void pack32_f32(const float* f, uint4* out) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    out[i] = make_uint4(__float_as_uint(f[4 * i]), __float_as_uint(f[4 * i + 1]),
                        __float_as_uint(f[4 * i + 2]), __float_as_uint(f[4 * i + 3]));
}

// store 32 consecutive values (fp32 in f[]) of one row at column n (masked by N)
__device__ __forceinline__ void store_row32(void* base, bool f32, int64_t row_off, int64_t n,
                                            int64_t N, const float* f, bool accumulate) {
  if (f32) {
    float* p = static_cast<float*>(base) + row_off + n;
    if (n + 32 <= N && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 v = make_float4(f[i], f[i + 1], f[i + 2], f[i + 3]);
        if (accumulate) {
          const float4 o = *reinterpret_cast<const float4*>(p + i);
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        *reinterpret_cast<float4*>(p + i) = v;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (n + i < N) p[i] = accumulate ? p[i] + f[i] : f[i];
    }
  } else {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + row_off + n;
    // bf16 accumulate: C = bf16(C + bf16(acc)), matching the TMA bf16 reduce-add
    auto term = [&](int i) {
      return accumulate ? __bfloat162float(p[i]) + __bfloat162float(__float2bfloat16_rn(f[i])) : f[i];
    };
    if (n + 32 <= N && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 v;
        v.x = pack_bf16(term(i), term(i + 1));
        v.y = pack_bf16(term(i + 2), term(i + 3));
        v.z = pack_bf16(term(i + 4), term(i + 5));
        v.w = pack_bf16(term(i + 6), term(i + 7));
        *reinterpret_cast<uint4*>(p + i) = v;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (n + i < N) p[i] = __float2bfloat16_rn(term(i));
    }
  }
}

__device__ __forceinline__ void load_row32_bf16(const void* base, int64_t off, float* f) {
  const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = p[i];
    float2 a = unpack_bf16(v.x), b = unpack_bf16(v.y), c = unpack_bf16(v.z), d = unpack_bf16(v.w);
    f[8 * i + 0] = a.x; f[8 * i + 1] = a.y; f[8 * i + 2] = b.x; f[8 * i + 3] = b.y;
    f[8 * i + 4] = c.x; f[8 * i + 5] = c.y; f[8 * i + 6] = d.x; f[8 * i + 7] = d.y;
  }
}

// ------------------------------------------------------------------ kernel
#ifdef B200MOE_WAIT_PROF
// perf diagnosis build only: summed clock64 cycles per role
// [0] MMA waiting for operands (full), [1] MMA waiting for a free accumulator
// (tempty), [2] MMA warp lifetime, [3] producer waiting for a free stage,
// [4] epilogue waiting for an accumulator (tfull), [5] epilogue lifetime,
// [6] SwiGLU-bwd epilogue waiting for its pre chunk, [7] MMA CTAs
__device__ unsigned long long g_wait_prof[8];
#define WP_T0() const long long wp_t0 = clock64()
#define WP_ADD(var) var += clock64() - wp_t0
#else
#define WP_T0()
#define WP_ADD(var)
#endif

template <bool A_MN, bool B_MN, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_h,
                   const Params p) {
  using C = Cfg<CG>;
  constexpr int S = C::STAGES_;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base;
  const uint32_t sB = base + S * C::A_BYTES;
  const uint32_t stg = base + S * C::STAGE;  // epilogue staging ring (1024-aligned)
  const int bars_off = S * C::STAGE + C::NSTG * STG_BYTES;
  const uint32_t bars = base + bars_off;
  // barrier layout: full[S], empty[S], tfull[2], tempty[2], ldb[NSTG], tmem slot
  const uint32_t full_bar = bars, empty_bar = bars + 8 * S;
  const uint32_t tfull_bar = bars + 16 * S, tempty_bar = tfull_bar + 16;
  const uint32_t ld_bar = tfull_bar + 32;  // epilogue TMA loads into the staging ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + bars_off + 16 * S + 32 + 8 * C::NSTG + 8);
  const uint32_t ld_empty = ld_bar + 8 * C::NSTG + 16;  // staging slot handed back by the epilogue
  int32_t* prefix = reinterpret_cast<int32_t*>(gbase + bars_off + 1024);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;  // 0 = leader CTA of the pair
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;

  // per-group tile counts -> prefix (smem)
  for (int g = threadIdx.x; g < p.G; g += NUM_THREADS) {
    int tiles;
    if (!p.grouped_k) {
      const int64_t rows = (p.gend ? p.gend[g] : p.goff[g + 1]) - p.goff[g];
      tiles = (int)(((rows + p.tile_m - 1) / p.tile_m) * ((p.N + BN - 1) / BN));
    } else {
      tiles = (int)(((p.M + p.tile_m - 1) / p.tile_m) * ((p.N + BN - 1) / BN));
    }
    prefix[g + 1] = tiles;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full_bar + 8 * i, 1);
      mbar_init(empty_bar + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull_bar + 8 * i, 1);
      mbar_init(tempty_bar + 8 * i, 4 * CG);  // epilogue warps of both CTAs
    }
    for (int i = 0; i < C::NSTG; ++i) {
      mbar_init(ld_bar + 8 * i, 1);
      mbar_init(ld_empty + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    prefetch_map(&map_a);
    prefetch_map(&map_b);
  }
  if (warp == 2) tmem_alloc<CG>(smem_u32(tmem_slot), TMEM_COLS);
  __syncthreads();
  if (threadIdx.x == 0) {
    prefix[0] = 0;
    for (int g = 0; g < p.G; ++g) prefix[g + 1] += prefix[g];
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = prefix[p.G];

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Both CTAs of a pair load their halves; TMA completions of both land on
    // the leader's full barrier, which the leader arms for both halves.
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      long long w_empty = 0;
      (void)w_empty;
      for (int t = cid; t < total; t += ncl) {
        const Tile tl = decode(p, prefix, t);
        const int m0 = (p.debug_ops == 1 ? 0 : (int)tl.m0) + BM * (int)crank;
        const int n0 = (p.debug_ops == 1 ? 0 : (int)tl.n0) + C::B_CTA * (int)crank;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          {
            WP_T0();
            mbar_wait(empty_bar + 8 * stage, phase ^ 1);
            WP_ADD(w_empty);
          }
          const uint32_t fb = full_bar + 8 * stage;
          if (p.debug_ops == 2) {  // energy experiment: no operand loads at all
            if (crank == 0) mbar_arrive(fb);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          // energy experiment 3: the pair's second CTA skips its A load (half
          // of A's L2 reads, as a 2-pair multicast of A would give)
          const bool skip_a = p.debug_ops == 3 && crank == 1;
          if (crank == 0) mbar_expect_tx(fb, C::STAGE * CG - (p.debug_ops == 3 && CG == 2 ? C::A_BYTES : 0));
          const uint32_t fb_tma = CG == 2 ? (fb & PEER_BIT_MASK) : fb;
          const int kbr = kb + tl.krot < tl.nkb ? kb + tl.krot : kb + tl.krot - tl.nkb;
          // energy experiment 1: every load reads the first K block of the
          // CTA's first tile rows (L2-resident, no DRAM traffic)
          const int kc = p.debug_ops == 1 ? 0 : (int)(tl.kbeg + (int64_t)kbr * BK);
          const uint32_t a_dst = sA + stage * C::A_BYTES;
          const uint32_t b_dst = sB + stage * C::B_BYTES;
          if (skip_a) {
          } else if (!A_MN) {
            // A [rows, K] K-major: box {64 K, 128 rows}
            tma_load<CG>(&map_a, a_dst, fb_tma, kc, m0, 0);
          } else {
            // A stored [K, M] (M contiguous): 2 boxes {64 M, 64 K}
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load<CG>(&map_a, a_dst + i * 8192, fb_tma, m0 + 64 * i, kc, 0);
          }
          if (!B_MN) {
            // B stored [L, N, K]: box {64 K, B_CTA N, 1}
            tma_load<CG>(&map_b, b_dst, fb_tma, kc, n0, tl.bidx);
          } else {
            // B stored [L, K, N] (N contiguous): B_CTA/64 boxes {64 N, 64 K, 1}
#pragma unroll
            for (int i = 0; i < C::B_CTA / 64; ++i)
              tma_load<CG>(&map_b, b_dst + i * 8192, fb_tma, n0 + 64 * i, kc, tl.bidx);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
#ifdef B200MOE_WAIT_PROF
      atomicAdd(&g_wait_prof[3], (unsigned long long)w_empty);
#endif
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (leader CTA only for a pair: one tcgen05.mma.cta_group::2 covers 256 x 256)
    if (lane == 0 && crank == 0) {
      constexpr uint32_t idesc = make_idesc(A_MN, B_MN, BM * CG);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      long long w_full = 0, w_tempty = 0;
      (void)w_full;
      (void)w_tempty;
#ifdef B200MOE_WAIT_PROF
      const long long life0 = clock64();
#endif
      for (int t = cid; t < total; t += ncl) {
        const Tile tl = decode(p, prefix, t);
        {
          WP_T0();
          mbar_wait(tempty_bar + 8 * acc, acc_phase ^ 1);
          WP_ADD(w_tempty);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          {
            WP_T0();
            mbar_wait(full_bar + 8 * stage, phase);
            WP_ADD(w_full);
          }
          tc_fence_after();
          const uint32_t a_s = sA + stage * C::A_BYTES;
          const uint32_t b_s = sB + stage * C::B_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 32 B inside the 128B swizzle atom; MN-major:
            // advance 16 K-rows (2 x 1024 B core-matrix groups).
            const uint64_t ad = A_MN ? smem_desc(a_s + k * 2048, 8192, 1024)
                                     : smem_desc(a_s + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(b_s + k * 2048, 8192, 1024)
                                     : smem_desc(b_s + k * 32, 16, 1024);
            tc_mma<CG>(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit<CG>(empty_bar + 8 * stage);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (tl.nkb > 0) tc_commit<CG>(tfull_bar + 8 * acc);
        else arrive_all<CG>(tfull_bar + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef B200MOE_WAIT_PROF
      atomicAdd(&g_wait_prof[0], (unsigned long long)w_full);
      atomicAdd(&g_wait_prof[1], (unsigned long long)w_tempty);
      atomicAdd(&g_wait_prof[2], (unsigned long long)(clock64() - life0));
      atomicAdd(&g_wait_prof[7], 1ull);
#endif
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ epilogue input
    // SwiGLU backward reads the saved pre-activations: this lane streams the
    // 64-column pre chunks of each tile into the staging ring ahead of the
    // epilogue (same tile/chunk sequence), so their DRAM latency overlaps the
    // mainloop instead of stalling the epilogue.
    if (lane == 0 && p.epi == EPI_SWIGLU_BWD && p.use_tma && p.debug_nostore != 1 && p.debug_nostore != 3) {
      prefetch_map(&map_h);
      uint32_t ctr = 0;
      for (int t = cid; t < total; t += ncl) {
        const Tile tl = decode(p, prefix, t);
        const int64_t row0 = tl.m0 + BM * (int64_t)crank;
        if (!(row0 + BM <= tl.m_end)) continue;  // not the epilogue's TMA path
        for (int c = 0; c < BN / 32 && tl.n0 + c * 32 < p.N; ++c, ++ctr) {
          const uint32_t sl = ctr % C::NSTG, ph = (ctr / C::NSTG) & 1u;
          mbar_wait(ld_empty + 8 * sl, ph ^ 1u);
          mbar_expect_tx(ld_bar + 8 * sl, STG_BYTES);
          tma_load_3d(&map_h, stg + sl * STG_BYTES, ld_bar + 8 * sl, (int)(((tl.n0 + c * 32) / 32) * 64),
                      (int)row0, 0);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp - 4;  // TMEM lanes [32q, 32q+32)
    const int row_in_tile = BM * (int)crank + 32 * q + lane;
    Stager<C::NSTG> stgr{stg, 0, threadIdx.x == 128, p.debug_nostore == 2, p.store_hint != 0,
                         policy_evict_first()};
    uint32_t bwd_ctr = 0;  // SwiGLU-backward staging chunks consumed (matches warp 3)
    int acc = 0;
    uint32_t acc_phase = 0;
    long long w_tfull = 0, w_pre = 0;
    (void)w_tfull;
    (void)w_pre;
#ifdef B200MOE_WAIT_PROF
    const long long elife0 = clock64();
#endif
    for (int t = cid; t < total; t += ncl) {
      const Tile tl = decode(p, prefix, t);
      {
        WP_T0();
        mbar_wait(tfull_bar + 8 * acc, acc_phase);
        WP_ADD(w_tfull);
      }
      tc_fence_after();
      const int64_t row = tl.m0 + row_in_tile;
      const bool live = row < tl.m_end && p.debug_nostore != 1;
      const bool zero = tl.nkb == 0;
      const int64_t c_off = p.grouped_k ? (int64_t)tl.g * p.c_sg : 0;
      const uint32_t t_row = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      // This CTA's 128-row block is either entirely inside the group (TMA
      // store path), entirely past it (nothing to do) or -- only for
      // unaligned groups -- ragged (direct masked stores).
      const int64_t row0 = tl.m0 + BM * (int64_t)crank;
      const bool cta_live = row0 < tl.m_end && p.debug_nostore != 1;
      const bool tma_path = p.use_tma && row0 + BM <= tl.m_end && p.epi <= EPI_SWIGLU_BWD;
      const int r = 32 * q + lane;
      if (!cta_live) {
        // this CTA half holds no rows of the group
      } else if (p.epi == EPI_SCATTER) {
        // Fused return exchange: each bf16 row goes straight to the rank that
        // sent it, at that rank's own row, so the transfer overlaps the MMAs
        // of the next tile.  A warp stages its 32 rows (swizzled) in its own
        // 4 KB of the staging tile and writes them back 4 rows x 128 B per
        // instruction (full-line NVLink writes); only __syncwarp is needed.
        uint64_t dst = 0;
        if (live) {
          const int32_t d = p.origin[2 * row];
          if (d >= 0)
            dst = p.peer_base[d] + (uint64_t)p.scatter_off + (uint64_t)p.origin[2 * row + 1] * p.ldc * 2;
        }
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          const int64_t n = tl.n0 + c * 64;
          if (n >= p.N) break;
          uint32_t v0[32], v1[32];
          tmem_ld32(t_row + c * 64, v0);
          tmem_ld32(t_row + c * 64 + 32, v1);
          float f0[32], f1[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            f0[i] = __uint_as_float(v0[i]);
            f1[i] = __uint_as_float(v1[i]);
          }
          uint4 o[8];
          pack32_bf16(f0, o);
          pack32_bf16(f1, o + 4);
          st_row_chunk(stg, r, o);
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int src = 4 * it + (lane >> 3), j = lane & 7;
            const uint64_t d = __shfl_sync(0xffffffffu, dst, src);
            const int rr = 32 * q + src;
            const uint4 v = ld_shared_v4(stg + rr * 128 + ((j ^ (rr & 7)) << 4));
            const int64_t col = n + 8 * j;
            if (d && col < p.N) st_global_v4(d + col * 2, v);
          }
          __syncwarp();
        }
      } else if (tma_path) {
        const int crow = (int)row0;
        if (p.epi == EPI_STORE && p.out_f32) {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            const int64_t n = tl.n0 + c * 32;
            if (n >= p.N) break;
            uint32_t v[32];
            tmem_ld32(t_row + c * 32, v);
            float f[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = zero ? 0.f : __uint_as_float(v[i]);
            uint4 o[8];
            pack32_f32(f, o);
            st_row_chunk(stgr.acquire(), r, o);
            if (p.glu_f)
              stgr.issue_glu(&map_h, (int)n, row0, tl.g, p.accumulate, p.glu_f);
            else
              stgr.issue(&map_c, (int)n, crow, p.grouped_k ? tl.g : 0, p.accumulate);
          }
        } else if (p.epi == EPI_STORE) {
#pragma unroll 1
          for (int c = 0; c < BN / 64; ++c) {
            const int64_t n = tl.n0 + c * 64;
            if (n >= p.N) break;
            uint32_t v0[32], v1[32];
            tmem_ld32(t_row + c * 64, v0);
            tmem_ld32(t_row + c * 64 + 32, v1);
            float f0[32], f1[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              f0[i] = zero ? 0.f : __uint_as_float(v0[i]);
              f1[i] = zero ? 0.f : __uint_as_float(v1[i]);
            }
            uint4 o[8];
            pack32_bf16(f0, o);
            pack32_bf16(f1, o + 4);
            st_row_chunk(stgr.acquire(), r, o);
            stgr.issue(&map_c, (int)n, crow, p.grouped_k ? tl.g : 0, p.accumulate);  // bf16 reduce-add
          }
        } else if (p.epi == EPI_SWIGLU_FWD) {
          uint4 hb[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) hb[i] = make_uint4(0, 0, 0, 0);
          int b = 0;
#pragma unroll 1
          for (; b < BN / 64; ++b) {
            const int64_t n = tl.n0 + b * 64;
            if (n >= p.N) break;
            uint32_t vg[32], vu[32];
            tmem_ld32(t_row + b * 64, vg);
            tmem_ld32(t_row + b * 64 + 32, vu);
            float g[32], u[32], h[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              // round the pre-activations to bf16 first so the saved `pre`
              // and `h` agree exactly with what the backward recomputes
              g[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(vg[i])));
              u[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(vu[i])));
              h[i] = silu_f(g[i]) * u[i];
            }
            uint4 o[8];
            pack32_bf16(g, o);
            pack32_bf16(u, o + 4);
            st_row_chunk(stgr.acquire(), r, o);
            stgr.issue(&map_c, (int)n, crow, 0, false);
            uint4 hq[4];
            pack32_bf16(h, hq);
            if (b & 1) {
#pragma unroll
              for (int i = 0; i < 4; ++i) hb[4 + i] = hq[i];
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) hb[i] = hq[i];
            }
            if (b & 1) {  // two blocks of h = one 64-column (128 B) chunk
              st_row_chunk(stgr.acquire(), r, hb);
              stgr.issue(&map_h, (int)((tl.n0 + (b - 1) * 64) / 2), crow, 0, false);
            }
          }
          if (b & 1) {  // odd number of blocks: flush the half chunk (TMA clips at F)
            st_row_chunk(stgr.acquire(), r, hb);
            stgr.issue(&map_h, (int)((tl.n0 + (b - 1) * 64) / 2), crow, 0, false);
          }
        } else {  // EPI_SWIGLU_BWD: acc = dh over F columns; pre/dpre [.., 2F] interleaved
          // The matching 64-column pre chunk (32 gate | 32 up, 128 B per row)
          // arrives in the staging ring from warp 3, is transformed in place
          // into d[gate|up] and TMA-stored: pre and dpre share the layout.
          // The slot goes back to warp 3 once its store has read it (checked
          // one chunk later, so the epilogue never waits on its own store).
          int nch = 0;
          while (nch < BN / 32 && tl.n0 + nch * 32 < p.N) ++nch;
#pragma unroll 1
          for (int c = 0; c < nch; ++c) {
            const uint32_t ctr = bwd_ctr++;
            const uint32_t sl = ctr % C::NSTG;
            uint32_t v[32];
            tmem_ld32(t_row + c * 32, v);
            if (p.debug_nostore != 3) {
              WP_T0();
              mbar_wait(ld_bar + 8 * sl, (ctr / C::NSTG) & 1u);
              WP_ADD(w_pre);
            }
            const uint32_t rowp = stg + sl * STG_BYTES + (uint32_t)r * 128;
            uint4 o[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = ld_shared_v4(rowp + ((uint32_t)(j ^ (r & 7)) << 4));
            float g[32], u[32], dg[32], du[32];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t* gw = reinterpret_cast<const uint32_t*>(&o[j]);
              const uint32_t* uw = reinterpret_cast<const uint32_t*>(&o[4 + j]);
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                const float2 a = unpack_bf16(gw[w]), b = unpack_bf16(uw[w]);
                g[8 * j + 2 * w] = a.x; g[8 * j + 2 * w + 1] = a.y;
                u[8 * j + 2 * w] = b.x; u[8 * j + 2 * w + 1] = b.y;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float d = __uint_as_float(v[i]);
              const float s = sigmoid_f(g[i]);
              dg[i] = d * u[i] * s * (1.f + g[i] * (1.f - s));
              du[i] = d * g[i] * s;
            }
            pack32_bf16(dg, o);
            pack32_bf16(du, o + 4);
            st_row_chunk(stg + sl * STG_BYTES, r, o);
            fence_async_smem();
            epi_bar();
            if (threadIdx.x == 128) {
              if (p.debug_nostore != 2) {
                if (stgr.hint)
                  tma_store_3d_hint(&map_c, stg + sl * STG_BYTES, (int)(((tl.n0 + c * 32) / 32) * 64), crow, 0,
                                    stgr.pol);
                else
                  tma_store_3d(&map_c, stg + sl * STG_BYTES, (int)(((tl.n0 + c * 32) / 32) * 64), crow, 0);
                bulk_commit();
              }
              bulk_wait_read<1>();  // the previous chunk's store has read its slot
              if (ctr > 0) mbar_arrive(ld_empty + 8 * ((ctr - 1) % C::NSTG));
            }
          }
        }
      } else if (p.epi == EPI_STORE) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_row + c * 32, v);
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = zero ? 0.f : __uint_as_float(v[i]);
          const int64_t n = tl.n0 + c * 32;
          const int64_t drow = p.glu_f ? glu_row(row, p.glu_f) : row;
          if (live && n < p.N) store_row32(p.C, p.out_f32, c_off + drow * p.ldc, n, p.N, f, p.accumulate);
        }
      } else if (p.epi == EPI_SWIGLU_FWD) {
        // columns: 4 blocks of [32 gate | 32 up]; h column = (n0 + 64 b)/2 + i
#pragma unroll 1
        for (int b = 0; b < BN / 64; ++b) {
          uint32_t vg[32], vu[32];
          tmem_ld32(t_row + b * 64, vg);
          tmem_ld32(t_row + b * 64 + 32, vu);
          const int64_t n = tl.n0 + b * 64;
          if (!live || n >= p.N) continue;
          float g[32], u[32], h[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            // round the pre-activations to bf16 first so the saved `pre`
            // and `h` agree exactly with what the backward recomputes
            g[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(vg[i])));
            u[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(vu[i])));
            h[i] = silu_f(g[i]) * u[i];
          }
          store_row32(p.C, false, row * p.ldc, n, p.N, g, false);
          store_row32(p.C, false, row * p.ldc, n + 32, p.N, u, false);
          store_row32(p.H, false, row * p.ldh, n / 2, p.N / 2, h, false);
        }
      } else if (p.epi == EPI_SWIGLU_BWD) {
        // acc = dh over F columns; pre/dpre are [.., 2F] interleaved
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_row + c * 32, v);
          const int64_t n = tl.n0 + c * 32;  // F column, multiple of 32
          if (!live || n >= p.N) continue;
          const int64_t pc = (n / 32) * 64;  // gate block column in pre
          float g[32], u[32], dg[32], du[32];
          load_row32_bf16(p.PRE, row * p.ldpre + pc, g);
          load_row32_bf16(p.PRE, row * p.ldpre + pc + 32, u);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float d = __uint_as_float(v[i]);
            const float s = sigmoid_f(g[i]);
            dg[i] = d * u[i] * s * (1.f + g[i] * (1.f - s));
            du[i] = d * g[i] * s;
          }
          store_row32(p.C, false, row * p.ldc, pc, 2 * p.N, dg, false);
          store_row32(p.C, false, row * p.ldc, pc + 32, 2 * p.N, du, false);
        }
      } else if (p.epi == EPI_ACT_FWD) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_row + c * 32, v);
          const int64_t n = tl.n0 + c * 32;
          if (!live || n >= p.N) continue;
          float pre[32], h[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            pre[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[i])));
            h[i] = p.act == B200MOE_ACT_RELU ? fmaxf(pre[i], 0.f) : gelu_tc(pre[i]);
          }
          store_row32(p.C, false, row * p.ldc, n, p.N, pre, false);
          store_row32(p.H, false, row * p.ldh, n, p.N, h, false);
        }
      } else {  // EPI_ACT_BWD
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(t_row + c * 32, v);
          const int64_t n = tl.n0 + c * 32;
          if (!live || n >= p.N) continue;
          float pre[32], d[32];
          load_row32_bf16(p.PRE, row * p.ldpre + n, pre);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float gr = p.act == B200MOE_ACT_RELU ? (pre[i] > 0.f ? 1.f : 0.f) : gelu_grad_tc(pre[i]);
            d[i] = __uint_as_float(v[i]) * gr;
          }
          store_row32(p.C, false, row * p.ldc, n, p.N, d, false);
        }
      }
      tc_fence_before();
      __syncwarp();
      // the leader's MMA warp waits on its own tempty barrier for both CTAs
      if (lane == 0) {
        if (CG == 2 && crank != 0) mbar_arrive_remote(tempty_bar + 8 * acc, 0);
        else mbar_arrive(tempty_bar + 8 * acc);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (threadIdx.x == 128) bulk_wait_all();  // staged stores done before smem is released
#ifdef B200MOE_WAIT_PROF
    if (lane == 0 && warp == 4) {
      atomicAdd(&g_wait_prof[4], (unsigned long long)w_tfull);
      atomicAdd(&g_wait_prof[5], (unsigned long long)(clock64() - elife0));
      atomicAdd(&g_wait_prof[6], (unsigned long long)w_pre);
    }
#endif
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();  // the peer may still arrive on our barriers
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<CG>(tmem_base, TMEM_COLS);
}

}  // namespace tc


// Raster policy from the typical per-group operand footprints (bf16 bytes).
static int choose_panel(const b200moe_tc_gemm_args* a, int tile_m) {
  const double G = a->G > 0 ? a->G : 1;
  const double Mg = a->grouped_dim == 0 ? (double)a->a_rows / G : (double)a->M;
  const double Kg = a->grouped_dim == 0 ? (double)a->K : (double)a->a_rows / G;
  const double a_bytes = Mg * Kg * 2, b_bytes = (double)a->N * Kg * 2;
  const double resident = 40.0 * 1024 * 1024;  // comfortably inside the 126 MB L2
  const int mt = (int)((Mg + tile_m - 1) / tile_m);
  const int small = tile_m == 256 ? 4 : 8;
  if (a_bytes <= resident) return mt > 0 ? mt : 1;  // A resident, B streamed once
  if (b_bytes <= resident) return small;             // B resident, A streamed once
  return 2 * small;                                  // balanced k-slab reuse
}

int gemm_tc(const b200moe_tc_gemm_args* a, cudaStream_t st) {
  using namespace tc;
  if (a->G < 1 || a->G > MAX_G) {
    set_error("gemm_tc: G=%d out of range [1, %d]", a->G, MAX_G);
    return B200MOE_EUNSUPPORTED;
  }
  const bool a_mn = a->a_major == B200MOE_MAJOR_MN;
  const bool b_mn = a->b_major == B200MOE_MAJOR_MN;
  if (a->grouped_dim == 0 && a_mn) {
    set_error("gemm_tc: grouped-M needs a K-major A operand");
    return B200MOE_EUNSUPPORTED;
  }
  if (a->grouped_dim == 1 && !(a_mn && b_mn)) {
    set_error("gemm_tc: grouped-K needs MN-major A and B operands");
    return B200MOE_EUNSUPPORTED;
  }
  if ((a->lda % 8) || (a->ldb % 8)) {
    set_error("gemm_tc: leading dimensions must be multiples of 8 elements (16 B)");
    return B200MOE_EUNSUPPORTED;
  }
  if (a->glu_f && (a->grouped_dim != 1 || a->epilogue != EPI_STORE || a->out_dtype != B200MOE_F32 ||
                   a->M != 2 * a->glu_f || (a->glu_f % 32))) {
    set_error("gemm_tc: glu_f needs a grouped-K fp32 store with M == 2 * glu_f, glu_f %% 32 == 0");
    return B200MOE_EUNSUPPORTED;
  }
  if (a->epilogue == EPI_SCATTER &&
      (a->grouped_dim != 0 || a->out_dtype != B200MOE_BF16 || !a->row_origin || !a->peer_base ||
       (a->ldc % 8) || (a->N % 8))) {
    set_error("gemm_tc: the scatter epilogue needs grouped M, bf16 output, row_origin, peer_base "
              "and N, ldc multiples of 8");
    return B200MOE_EUNSUPPORTED;
  }
  // CTA pairs (cta_group::2, 256 x 256 tiles) by default; B200MOE_CTA_GROUP=1
  // selects single-CTA 128 x 256 tiles.  num_ctas must be even for pairs.
  const char* cg_str = getenv("B200MOE_CTA_GROUP");
  const int cg_env = (cg_str && cg_str[0] == '1') ? 1 : 2;
  int grid = a->num_ctas > 0 ? a->num_ctas : num_sms();
  const int cg = (cg_env == 2 && grid >= 2) ? 2 : 1;
  if (cg == 2) grid &= ~1;
  const uint32_t b_box = BN / cg;
  CUtensorMap ma, mb;
  int rc;
  const uint64_t R = (uint64_t)a->a_rows;
  if (!a_mn)  // A [R, K]: box {64 K, 128 rows}
    rc = make_map(&ma, a->A, (uint64_t)a->K, R, 1, (uint64_t)a->lda, (uint64_t)a->lda * R, BM);
  else        // A [R(K), M]: box {64 M, 64 K}
    rc = make_map(&ma, a->A, (uint64_t)a->M, R, 1, (uint64_t)a->lda, (uint64_t)a->lda * R, 64);
  if (rc) return rc;
  if (!b_mn)  // B [batch, N, K]: box {64 K, BN/cg N, 1}
    rc = make_map(&mb, a->B, (uint64_t)a->K, (uint64_t)a->N, (uint64_t)a->b_batch,
                  (uint64_t)a->ldb, (uint64_t)a->b_batch_stride, b_box);
  else {      // B [batch, Kdim, N]: box {64 N, 64 K, 1}
    const uint64_t kdim = a->grouped_dim == 1 ? R : (uint64_t)a->K;
    const uint64_t bstride = a->b_batch > 1 ? (uint64_t)a->b_batch_stride : (uint64_t)a->ldb * kdim;
    rc = make_map(&mb, a->B, (uint64_t)a->N, kdim, (uint64_t)a->b_batch, (uint64_t)a->ldb, bstride, 64);
  }
  if (rc) return rc;

  // Output maps for the TMA-store epilogue (row dim = a_rows for grouped M,
  // M for grouped K; 3rd dim = per-group output for grouped K).
  CUtensorMap mc, mh;
  int use_tma = 0;
  if (a->epilogue <= 2) {
    const bool of32 = a->out_dtype == B200MOE_F32;
    const uint64_t crows = a->grouped_dim == 0 ? R : (uint64_t)a->M;
    const uint64_t cg_n = a->grouped_dim == 0 ? 1 : (uint64_t)a->G;
    const uint64_t ccols = a->epilogue == 2 ? 2 * (uint64_t)a->N : (uint64_t)a->N;
    const uint64_t csg = a->grouped_dim == 0 ? (uint64_t)a->ldc * crows : (uint64_t)a->c_sg;
    rc = make_map(&mc, a->C, ccols, crows, cg_n, (uint64_t)a->ldc, csg, BM, of32);
    if (rc == B200MOE_OK && a->epilogue == 1)  // h [R, F]
      rc = make_map(&mh, a->H, (uint64_t)a->N / 2, R, 1, (uint64_t)a->ldh, (uint64_t)a->ldh * R, BM);
    else if (rc == B200MOE_OK && a->epilogue == 2)  // pre [R, 2F], read by the epilogue
      rc = make_map(&mh, a->PRE, 2 * (uint64_t)a->N, R, 1, (uint64_t)a->ldpre, (uint64_t)a->ldpre * R, BM);
    else if (rc == B200MOE_OK && a->glu_f)  // C again, 32-row boxes for the de-interleaving store
      rc = make_map(&mh, a->C, ccols, crows, cg_n, (uint64_t)a->ldc, csg, 32, of32);
    else
      mh = mc;
    use_tma = rc == B200MOE_OK && (a->ldc % 8 == 0) && (a->epilogue != 1 || a->ldh % 8 == 0) &&
              (a->epilogue != 2 || a->ldpre % 8 == 0);
    if (rc != B200MOE_OK) mc = mh = ma;  // fall back to direct stores
  } else {
    mc = mh = ma;
  }

  Params p{};
  p.use_tma = use_tma;
  p.G = a->G;
  p.grouped_k = a->grouped_dim;
  p.M = a->M;
  p.N = a->N;
  p.K = a->K;
  p.goff = a->group_off;
  p.gexp = a->group_expert;
  p.gend = a->group_end;
  p.max_rows = a->a_rows;
  p.epi = a->epilogue;
  p.act = a->act;
  p.out_f32 = a->out_dtype == B200MOE_F32;
  p.accumulate = a->accumulate;
  p.C = a->C;
  p.ldc = a->ldc;
  p.c_sg = a->c_sg;
  p.H = a->H;
  p.ldh = a->ldh;
  p.PRE = a->PRE;
  p.ldpre = a->ldpre;
  p.origin = a->row_origin;
  p.peer_base = a->peer_base;
  p.scatter_off = a->scatter_off;
  p.glu_f = a->glu_f;
  // epilogue outputs stream through L2 once: evict them first so the operand
  // panels stay (ncu: 10-20 % fewer DRAM reads in the weight-gradient GEMMs,
  // same cycles); B200MOE_STORE_HINT=0 turns it off
  const char* sh = getenv("B200MOE_STORE_HINT");
  p.store_hint = (sh && sh[0] == '0') ? 0 : 1;
  p.tile_m = BM * cg;
  const char* dops = getenv("B200MOE_DEBUG_OPS");
  p.debug_ops = (dops && dops[0] >= '1' && dops[0] <= '3') ? dops[0] - '0' : 0;
  const char* ns = getenv("B200MOE_DEBUG_NOSTORE");
  p.debug_nostore = (ns && ns[0] >= '1' && ns[0] <= '3') ? ns[0] - '0' : 0;
  p.panel_m = choose_panel(a, p.tile_m);
  const char* ks = getenv("B200MOE_KSTAGGER");
  p.kstagger = ks ? atoi(ks) : 0;
  // experiments: B200MOE_PANEL_M=n forces the raster panel height (m-tiles)
  const char* pm = getenv("B200MOE_PANEL_M");
  if (pm && atoi(pm) > 0) p.panel_m = atoi(pm);

  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const Params);
  KernT kern;
  int smem;
  if (cg == 1) {
    kern = a_mn ? (b_mn ? gemm_tc_kernel<true, true, 1> : gemm_tc_kernel<true, false, 1>)
                : (b_mn ? gemm_tc_kernel<false, true, 1> : gemm_tc_kernel<false, false, 1>);
    smem = Cfg<1>::SMEM;
  } else {
    kern = a_mn ? (b_mn ? gemm_tc_kernel<true, true, 2> : gemm_tc_kernel<true, false, 2>)
                : (b_mn ? gemm_tc_kernel<false, true, 2> : gemm_tc_kernel<false, false, 2>);
    smem = Cfg<2>::SMEM;
  }
  // the shared-memory opt-in is per device and per kernel (thread-safe: a
  // repeated set is harmless)
  constexpr int MAX_DEV = 64;
  static std::atomic<bool> attr_set[MAX_DEV][8];
  int dev = 0;
  cudaGetDevice(&dev);
  const int ki = (cg == 2 ? 4 : 0) + (a_mn ? 2 : 0) + (b_mn ? 1 : 0);
  if (dev >= MAX_DEV || !attr_set[dev][ki].load()) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      set_error("gemm_tc: cannot set %d B dynamic shared memory", smem);
      return B200MOE_ELAUNCH;
    }
    if (dev < MAX_DEV) attr_set[dev][ki].store(true);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mh, p) != cudaSuccess) {
    set_error("gemm_tc: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return B200MOE_ELAUNCH;
  }
  B200MOE_CHECK_LAUNCH("gemm_tc");
  return B200MOE_OK;
}

}  // namespace b200moe

#ifdef B200MOE_WAIT_PROF
// perf diagnosis build only (not declared in include/b200moe.h)
extern "C" B200MOE_API int b200moe_debug_wait_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, b200moe::tc::g_wait_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(b200moe::tc::g_wait_prof, z, sizeof(z));
  }
  return 0;
}
#endif
