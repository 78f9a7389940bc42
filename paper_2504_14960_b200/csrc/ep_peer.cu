// EP all-to-all over NVLink peer memory (symmetric buffers), fused with the
// permute / combine work -- the device-side replacement of the reference's
// all_to_all_v + exchange_meta + regroup of dispatcher.py:309-362, 425-468.
//
// Every rank of an EP group maps the same symmetric buffer layout; peer
// addresses are  peer_base[d] + region offset.  Per forward step:
//   counts_push   each rank writes its per-expert kept counts into row `me` of
//                 every peer's count matrix                      (+ barrier)
//   layout        every rank derives, from the full count matrix, the
//                 receive layout of each destination: expert-major, senders
//                 contiguous in rank order inside an expert (the reference's
//                 stable `grp_order` regroup), each expert padded to `align`
//                 rows; it keeps its own push offsets and its GEMM groups
//   dispatch      one warp per token reads x[t] once and stores it straight
//                 into the destination ranks' receive buffers    (+ barrier)
//   ... grouped GEMM on the local receive buffer; its epilogue stores every
//   expert row straight back to the sender's return buffer     (+ barrier)
//   combine       local: each sender gate-combines its returned rows
// Split sizes never leave the device.  The barrier is a flag exchange in the
// symmetric buffer with system-scope release/acquire and a bounded spin
// (a missing peer traps instead of hanging the GPU).
#include "common.cuh"

namespace b200moe {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ barrier
// flags[p] on rank r = last epoch rank p announced to r.
__global__ void ep_barrier_kernel(const uint64_t* __restrict__ peer_base, int64_t flag_off, int me,
                                  int ep, uint32_t epoch, uint64_t timeout_ns) {
  const int p = threadIdx.x;
  __threadfence_system();  // this rank's prior writes (local and remote) before the flags
  __syncthreads();
  if (p < ep) {
    uint32_t* remote = reinterpret_cast<uint32_t*>(peer_base[p] + flag_off) + me;
    st_release_sys(remote, epoch);
  }
  if (p < ep) {
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(peer_base[me] + flag_off) + p;
    // bounded by wall time (a peer that died traps this rank after
    // $B200MOE_BARRIER_TIMEOUT_S, default 60 s, instead of hanging its GPU);
    // the legitimate wait is one GEMM's skew between ranks
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > timeout_ns) {
        printf("b200moe ep_barrier: rank %d timed out waiting for rank %d (epoch %u)\n", me, p, epoch);
        __trap();
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

// ------------------------------------------------------------------ counts
// A rank whose step already failed (status != 0: non-finite router input,
// oversized block) pushes an abort marker (-1 in every entry) instead of its
// counts; every member then lays out the step without it and skips its
// pushes, so all ranks finish the step's barriers and raise on the host.
__global__ void ep_counts_push_kernel(const int32_t* __restrict__ counts, int me, int ep, int E,
                                      const uint64_t* __restrict__ peer_base, int64_t cnt_off,
                                      const int32_t* __restrict__ status) {
  const bool abort = status && *status != 0;
  for (int i = threadIdx.x; i < ep * E; i += blockDim.x) {
    const int p = i / E, e = i % E;
    int32_t* dst = reinterpret_cast<int32_t*>(peer_base[p] + cnt_off) + me * E + e;
    *dst = abort ? -1 : counts[e];
  }
}

// ------------------------------------------------------------------ layout
// The exchange group is the EP x ETP block of ranks (member m = ep_idx * etp +
// etp_idx).  cnt: this rank's copy of the [ep*etp, E] matrix (row s = member
// s's kept counts).  The ETP members of one EP index receive the same rows
// in the same layout (the reference's ETP all-gather, dispatcher.py:325-334,
// folded into the dispatch).  Receive buffers are expert-major: local expert
// le's rows from all senders are contiguous (member order), and only the
// expert's group is padded to `align` rows -- one GEMM group per local
// expert, no per-sender padding.
// seg_off[d*L + le] = first row of (me, le) in EP index d's receive buffers;
// goff[le] / gcount[le] = group start / real rows in this rank's buffer,
// goff[L] = end.  A layout beyond cap_rows (the buffer size) fails the step
// (status bit 4) or, without a status word, traps.
__global__ void ep_layout_kernel(const int32_t* __restrict__ cnt, int me, int ep, int etp, int L,
                                 int align, int64_t cap_rows, int32_t* __restrict__ seg_off,
                                 int32_t* __restrict__ goff, int32_t* __restrict__ gcount,
                                 int32_t* __restrict__ status) {
  const int E = ep * L, nmem = ep * etp;
  const int d = threadIdx.x;  // one thread per destination EP index
  if (d >= ep) return;
  const bool mine = d == me / etp;
  if (d == 0 && status) {  // an aborted member (marker row, see counts_push) fails the step
    for (int s = 0; s < nmem; ++s)
      if (cnt[s * E] < 0) {
        atomicOr(status, 2);
        break;
      }
  }
  int64_t run = 0;
  for (int le = 0; le < L; ++le) {
    int64_t tot = 0;
    for (int s = 0; s < nmem; ++s) {
      if (s == me) seg_off[d * L + le] = (int32_t)(run + tot);
      tot += max(cnt[s * E + d * L + le], 0);
    }
    if (mine) {
      goff[le] = (int32_t)run;
      gcount[le] = (int32_t)tot;
    }
    run += (tot + align - 1) / align * align;
  }
  if (run > cap_rows) {
    // this step's routing does not fit EP index d's receive buffers: every
    // member sees the same counts, so all of them fail the step (status bit
    // 4; no pushes) and this rank's groups shrink to nothing (no GEMM reads
    // past the buffer); without a status word there is no safe way on
    if (!status) {
      printf("b200moe ep_layout: EP index %d receive layout needs %lld rows > capacity %lld\n", d,
             (long long)run, (long long)cap_rows);
      __trap();
    }
    atomicOr(status, 16);
    if (mine) {
      for (int le = 0; le <= L; ++le) goff[le] = 0;
      for (int le = 0; le < L; ++le) gcount[le] = 0;
    }
    return;
  }
  if (mine) goff[L] = (int32_t)run;
}

// zero the alignment pad rows of this rank's receive buffer (and, forward,
// mark them "no origin" so the scatter epilogue skips them)
__global__ void ep_zero_pads_kernel(__nv_bfloat16* __restrict__ buf, int64_t H,
                                    const int32_t* __restrict__ goff, const int32_t* __restrict__ gcount,
                                    int32_t* __restrict__ origin) {
  const int g = blockIdx.y;
  const int64_t row = (int64_t)goff[g] + gcount[g] + blockIdx.x;
  if (row >= goff[g + 1]) return;
  __nv_bfloat16* p = buf + row * H;
  for (int64_t c = threadIdx.x; c < H; c += blockDim.x) p[c] = __float2bfloat16_rn(0.f);
  if (origin && threadIdx.x == 0) origin[2 * row] = -1;
}

// ------------------------------------------------------------------ dispatch
// Forward: x[t] -> row rr of the owner's receive buffer, and origin[rr] =
// (this rank, the pair's row in this rank's padded layout) so the owner's
// GEMM epilogue can return the expert output straight to that row.
// Backward (BWD): g*u[t] -> the same rows of the owner's dyr, and
// dgate = <u[t], y> with y read locally from the returned expert outputs.
//
// Deduplication (dup_off >= 0): the pairs of a token that go to experts of
// the same remote EP index d carry the same row, so it crosses the link once:
// the lowest such slot (the leader) is pushed and every other one (a
// duplicate) only records its leader's row in the receiver's dup table
// [rows] int2 (rows for this rank's own EP index are stored per pair, (-1, 0)):
//   forward:  leader (-1, 0); duplicate (leader row, 0)         -> the
//             receiver copies the leader row (ep_expand phase 0);
//   backward: a leader without duplicates is pushed scaled, (-1, 0); one
//             with duplicates is pushed raw, (-2, gate); a duplicate gets
//             (leader row, gate) -> phase 1 writes bf16(gate * raw) into the
//             duplicates, phase 2 scales the raw leaders in place.
// Each row ends up with exactly the value the undeduplicated push stores.
//
// Split push (part != 0), for overlapping the exchange with the first GEMM:
// part 1 performs only the stores into this rank's own buffers (the rows its
// own experts take from itself: origin, dup entries, data), part 2 only the
// stores into the other members' buffers.  Each pair's dgate (backward) is
// written by exactly one part: part 1 for pairs routed to this rank's EP
// index, part 2 for the rest.  part 0 = everything (one launch).
template <int KMAX, bool BWD>
__device__ __forceinline__ void dispatch_token(
    int64_t t, int lane, int64_t H, int k, int L, const __nv_bfloat16* __restrict__ x,
    const int32_t* __restrict__ topk, const int32_t* __restrict__ gemm_row,
    const int32_t* __restrict__ poff, const int32_t* __restrict__ seg_off,
    const uint64_t* __restrict__ peer_base, int me, int etp, int part, int64_t dst_off,
    int64_t origin_off, int64_t dup_off, const __nv_bfloat16* __restrict__ y_rows,
    const float* __restrict__ gates, float* __restrict__ dgates) {
  const int self_mem = (me / etp) * etp;  // first member of this rank's EP index
  // which members of a pair's destination EP index this part stores to
  auto keep = [&](int mm) { return part == 0 || ((part == 1) == (mm == me)); };
  int mem[KMAX];
  int32_t rrs[KMAX], grs[KMAX];
  int64_t roff[KMAX];
  float g[KMAX], dot[KMAX];
  bool push[KMAX], scale[KMAX], wdg[KMAX];
  bool work = false;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    mem[s] = -1;
    rrs[s] = -1;
    grs[s] = 0;
    roff[s] = 0;
    g[s] = 1.f;
    dot[s] = 0.f;
    push[s] = false;
    scale[s] = BWD;
    wdg[s] = false;
    if (s >= k) continue;
    const int32_t gr = gemm_row[t * k + s];
    if (gr < 0) continue;
    const int e = topk[t * k + s];
    const int d = e / L, le = e % L;
    const int32_t rr = seg_off[d * L + le] + (gr - poff[e]);
    mem[s] = d * etp;  // the ETP members of EP index d all get the row
    rrs[s] = rr;
    grs[s] = gr;
    roff[s] = dst_off + (int64_t)rr * H * 2;
    push[s] = true;
    bool any = false;
    for (int m = 0; m < etp; ++m) any |= keep(mem[s] + m);
    if (BWD) {
      g[s] = gates[t * k + s];
      wdg[s] = part == 0 || ((part == 1) == (mem[s] == self_mem));
      any |= wdg[s];
    } else if (lane < etp && keep(mem[s] + lane)) {
      int2* o = reinterpret_cast<int2*>(peer_base[mem[s] + lane] + origin_off) + rr;
      *o = make_int2(me, gr);
    }
    work |= any;
  }
  if (!work) {  // warp-uniform: nothing of this token belongs to this part
    if (BWD && part != 2 && lane == 0)
      for (int s = 0; s < k && s < KMAX; ++s)
        if (mem[s] < 0) dgates[t * k + s] = 0.f;  // dropped pairs
    return;
  }
  if (dup_off >= 0) {
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      if (mem[s] < 0) continue;
      if (mem[s] == self_mem) {  // rows for this rank's own EP index stay per pair (the
                                 // local store; ETP siblings get their own copy)
        if (lane < etp && keep(mem[s] + lane))
          reinterpret_cast<int2*>(peer_base[mem[s] + lane] + dup_off)[rrs[s]] = make_int2(-1, 0);
        continue;
      }
      int lead = s, ndup = 0;
#pragma unroll
      for (int q = 0; q < KMAX; ++q) {
        if (q < s && lead == s && mem[q] == mem[s]) lead = q;
        if (q > s && mem[q] == mem[s]) ++ndup;
      }
      int2 entry;
      if (lead != s) {  // duplicate: no data, the receiver copies the leader row
        push[s] = false;
        entry = make_int2(rrs[lead], BWD ? __float_as_int(g[s]) : 0);
      } else if (BWD && ndup > 0) {  // leader pushed raw, scaled by the receiver
        scale[s] = false;
        entry = make_int2(-2, __float_as_int(g[s]));
      } else {
        entry = make_int2(-1, 0);
      }
      if (lane < etp && keep(mem[s] + lane))
        reinterpret_cast<int2*>(peer_base[mem[s] + lane] + dup_off)[rrs[s]] = entry;
    }
  }
  // U column chunks per iteration keep several 16 B loads in flight per lane
  constexpr int U = (BWD && KMAX >= 8) ? 1 : (KMAX >= 4 ? 2 : 4);
  const __nv_bfloat16* src = x + t * H;
  for (int64_t c0 = (int64_t)lane * 8; c0 < H; c0 += 256 * U) {
    Vec16<__nv_bfloat16> v[U];
    Vec16<__nv_bfloat16> y[BWD ? U : 1][BWD ? KMAX : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + u * 256;
      if (c < H) v[u].raw = ld_nc_v4(src + c);
      if (BWD) {
#pragma unroll
        for (int s = 0; s < KMAX; ++s)
          if (wdg[s] && c < H) y[u][s].raw = ld_nc_v4(y_rows + (int64_t)grs[s] * H + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + u * 256;
      if (c >= H) break;
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (mem[s] < 0) continue;
        uint4 val;
        if (BWD) {
          Vec16<__nv_bfloat16> o;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float uv = __bfloat162float(v[u].v[i]);
            if (wdg[s]) dot[s] = fmaf(uv, __bfloat162float(y[BWD ? u : 0][BWD ? s : 0].v[i]), dot[s]);
            o.v[i] = __float2bfloat16_rn(scale[s] ? uv * g[s] : uv);
          }
          val = o.raw;
        } else {
          val = v[u].raw;
        }
        if (!push[s]) continue;
        for (int m = 0; m < etp; ++m)  // NVLink push (or the local store)
          if (keep(mem[s] + m))
            st_v4(reinterpret_cast<__nv_bfloat16*>(peer_base[mem[s] + m] + roff[s]) + c, val);
      }
    }
  }
  if (BWD) {
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      if (s >= k) break;
      const float d = warp_sum(dot[s]);
      if (lane == 0 && (mem[s] < 0 ? part != 2 : wdg[s])) dgates[t * k + s] = mem[s] >= 0 ? d : 0.f;
    }
  }
}

// One warp per token, grid-stride.  NT = 256: the one-launch push (the whole
// GPU).  NT = 128 (forward) / 64 (backward): the overlapped remote push, one
// block per SM with a register budget (<= 80 / 144 per thread) that fits
// next to a resident gemm_tc CTA (256 threads x 216 registers of 64 K), so
// the push runs beside the GEMM instead of waiting for its SMs.
template <int KMAX, bool BWD, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? (BWD && KMAX >= 4 ? 2 : 1) : (NT == 128 ? 6 : 7)) ep_dispatch_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t Tn, int64_t H, int k, int L,
    const int32_t* __restrict__ topk, const int32_t* __restrict__ gemm_row,
    const int32_t* __restrict__ poff, const int32_t* __restrict__ seg_off,
    const uint64_t* __restrict__ peer_base, int me, int etp, int part, int64_t dst_off,
    int64_t origin_off, int64_t dup_off, const __nv_bfloat16* __restrict__ y_rows,
    const float* __restrict__ gates, float* __restrict__ dgates, const int32_t* __restrict__ status) {
  if (status && *status != 0) return;  // failed step: nothing is pushed (see counts_push)
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (NT / 32);
  for (int64_t t = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); t < Tn; t += nw)
    dispatch_token<KMAX, BWD>(t, lane, H, k, L, x, topk, gemm_row, poff, seg_off, peer_base, me, etp,
                              part, dst_off, origin_off, dup_off, y_rows, gates, dgates);
}

// Receiver side of the deduplicated push, over the real rows of each group
// (goff/gcount) of this rank's receive buffer:
//   phase 0 (forward):  rows with dup.x >= 0 copy row dup.x;
//   phase 1 (backward): rows with dup.x >= 0 get bf16(gate * row dup.x);
//   phase 2 (backward): rows with dup.x == -2 get bf16(gate * row) in place.
// One warp per row, 16-byte vectors; the arithmetic is the push kernel's.
__global__ void __launch_bounds__(256) ep_expand_kernel(__nv_bfloat16* __restrict__ buf, int64_t H,
                                                        const int32_t* __restrict__ goff,
                                                        const int32_t* __restrict__ gcount,
                                                        const int2* __restrict__ dup, int phase) {
  const int g = blockIdx.y, lane = threadIdx.x & 31;
  const int64_t r0 = goff[g], n = gcount[g];
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t row = r0 + i;
    const int2 e = dup[row];
    int64_t from;
    if (phase == 2) {
      if (e.x != -2) continue;
      from = row;
    } else {
      if (e.x < 0) continue;
      from = e.x;
    }
    const float gate = __int_as_float(e.y);
    const __nv_bfloat16* s = buf + from * H;
    __nv_bfloat16* d = buf + row * H;
    for (int64_t c = (int64_t)lane * 8; c < H; c += 256) {
      Vec16<__nv_bfloat16> v;
      v.raw = ld_nc_v4(s + c);
      if (phase != 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v.v[j] = __float2bfloat16_rn(__bfloat162float(v.v[j]) * gate);
      }
      st_v4(d + c, v.raw);
    }
  }
}

// ------------------------------------------------------------------ ETP reduce
// out = sum over the ETP members' partial rows, fp32, ascending member order
// (the reduce-scatter fold of collectives.py:386-388), rounded to bf16 once.
__global__ void ep_reduce_parts_kernel(const __nv_bfloat16* __restrict__ parts, int nparts,
                                       int64_t stride, int64_t n8, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int p = 0; p < nparts; ++p) {
      Vec16<__nv_bfloat16> v;
      v.raw = ld_nc_v4(parts + p * stride + i * 8);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v.v[j]);
    }
    Vec16<__nv_bfloat16> o;
#pragma unroll
    for (int j = 0; j < 8; ++j) o.v[j] = __float2bfloat16_rn(acc[j]);
    st_v4(out + i * 8, o.raw);
  }
}

// ------------------------------------------------------------------ host
int ep_reduce_parts(const void* parts, int nparts, int64_t stride, int64_t n, void* out, cudaStream_t st) {
  const int64_t n8 = n / 8;
  if (n8 == 0) return B200MOE_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n8, 256), 148 * 16);
  ep_reduce_parts_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(parts), nparts, stride, n8,
                                               static_cast<__nv_bfloat16*>(out));
  B200MOE_CHECK_LAUNCH("ep_reduce_parts");
  return B200MOE_OK;
}

#define KSW(k, M)                       \
  if (k <= 1) { M(1); }                 \
  else if (k <= 2) { M(2); }            \
  else if (k <= 4) { M(4); }            \
  else if (k <= 8) { M(8); }            \
  else { set_error("ep: k=%d > 8 unsupported", k); return B200MOE_EUNSUPPORTED; }

int ep_barrier(const uint64_t* peer_base, int64_t flag_off, int me, int ep, uint32_t epoch,
               cudaStream_t st) {
  static const uint64_t timeout_ns = [] {
    const char* e = getenv("B200MOE_BARRIER_TIMEOUT_S");
    const double s = e ? atof(e) : 60.0;
    return (uint64_t)((s > 0 ? s : 60.0) * 1e9);
  }();
  if (ep < 1 || ep > 32 || me < 0 || me >= ep) {  // one lane per member
    set_error("ep_barrier: %d members (me=%d) outside [1, 32]", ep, me);
    return B200MOE_EUNSUPPORTED;
  }
  ep_barrier_kernel<<<1, 32, 0, st>>>(peer_base, flag_off, me, ep, epoch, timeout_ns);
  B200MOE_CHECK_LAUNCH("ep_barrier");
  return B200MOE_OK;
}

int ep_counts_push(const int32_t* counts, int me, int ep, int E, const uint64_t* peer_base,
                   int64_t cnt_off, const int32_t* status, cudaStream_t st) {
  ep_counts_push_kernel<<<1, 256, 0, st>>>(counts, me, ep, E, peer_base, cnt_off, status);
  B200MOE_CHECK_LAUNCH("ep_counts_push");
  return B200MOE_OK;
}

int ep_layout(const int32_t* cnt_local, int me, int ep, int etp, int L, int align, int64_t cap_rows,
              int32_t* seg_off, int32_t* goff, int32_t* gcount, int32_t* status, cudaStream_t st) {
  if (ep < 1 || ep > 32 || etp < 1) {  // one thread per destination EP index
    set_error("ep_layout: ep=%d outside [1, 32] (etp=%d)", ep, etp);
    return B200MOE_EUNSUPPORTED;
  }
  ep_layout_kernel<<<1, 32, 0, st>>>(cnt_local, me, ep, etp, L, align, cap_rows, seg_off, goff, gcount, status);
  B200MOE_CHECK_LAUNCH("ep_layout");
  return B200MOE_OK;
}

int ep_zero_pads(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount, int G, int align,
                 int32_t* origin, cudaStream_t st) {
  if (align <= 1 || G <= 0) return B200MOE_OK;
  dim3 grid((unsigned)(align - 1), (unsigned)G);
  ep_zero_pads_kernel<<<grid, 128, 0, st>>>(static_cast<__nv_bfloat16*>(buf), H, goff, gcount, origin);
  B200MOE_CHECK_LAUNCH("ep_zero_pads");
  return B200MOE_OK;
}

int ep_dispatch(const void* x, int64_t Tn, int64_t H, int k, int L, const int32_t* topk,
                const int32_t* gemm_row, const int32_t* poff, const int32_t* seg_off,
                const uint64_t* peer_base, int me, int etp, int64_t dst_off, int64_t origin_off,
                int64_t dup_off, const void* y_rows, const float* gates, float* dgates, int bwd,
                int part, const int32_t* status, cudaStream_t st) {
  if (part < 0 || part > 2) {
    set_error("ep_dispatch: part=%d outside [0, 2]", part);
    return B200MOE_EINVAL;
  }
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
  const __nv_bfloat16* yb = static_cast<const __nv_bfloat16*>(y_rows);
  // part 2 runs beside the first GEMM: one small block per SM (see the kernel)
  static const int n_sm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const bool beside = part == 2;
  // the side push must not hold an SM in a small-shared-memory carveout:
  // the smem/L1 split only changes on an idle SM, so a push block resident
  // first would keep the GEMM CTA (~214 KB of shared memory) off that SM
  // until it drains.  Experiments: B200MOE_PUSH_CARVEOUT=0 skips this.
  static const bool carve = [] {
    const char* e = getenv("B200MOE_PUSH_CARVEOUT");
    if (e && atoi(e) == 0) return false;
    cudaFuncSetAttribute(ep_dispatch_kernel<1, false, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<2, false, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<4, false, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<8, false, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<1, true, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<2, true, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<4, true, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ep_dispatch_kernel<8, true, 64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)carve;
  const int nt = beside ? (bwd ? 64 : 128) : 256;
  // experiments: B200MOE_PUSH_BLOCKS_PER_SM = blocks of the side push per SM
  static const int beside_blocks = [] {
    const char* e = getenv("B200MOE_PUSH_BLOCKS_PER_SM");
    const int v = e ? atoi(e) : 1;
    return v >= 1 ? v : 1;
  }();
  const unsigned grid =
      (unsigned)std::min<int64_t>(ceil_div(Tn, nt / 32), beside ? (int64_t)n_sm * beside_blocks : INT32_MAX);
#define DARGS xb, Tn, H, k, L, topk, gemm_row, poff, seg_off, peer_base, me, etp, part, dst_off, origin_off, dup_off, yb, gates, dgates, status
#define DF(KM)                                                                  \
  if (beside) ep_dispatch_kernel<KM, false, 128><<<grid, 128, 0, st>>>(DARGS); \
  else ep_dispatch_kernel<KM, false, 256><<<grid, 256, 0, st>>>(DARGS)
#define DB(KM)                                                               \
  if (beside) ep_dispatch_kernel<KM, true, 64><<<grid, 64, 0, st>>>(DARGS); \
  else ep_dispatch_kernel<KM, true, 256><<<grid, 256, 0, st>>>(DARGS)
  if (Tn > 0) {
    if (bwd) { KSW(k, DB) }
    else { KSW(k, DF) }
  }
#undef DF
#undef DB
#undef DARGS
  B200MOE_CHECK_LAUNCH("ep_dispatch");
  return B200MOE_OK;
}

// GEMM groups of the split first GEMM (push overlapped with the GEMM): per
// local expert le, its group [goff[le], goff[le+1]) of the receive buffer
// splits into the rows this rank sent itself -- [s, s + c), s = seg_off[d*L
// + le] for d = this rank's EP index, c its own count -- and the rest
// (before and after them, pads included).  split (int32, 8L + 2):
//   [0, L]            loc_off  (loc_off[L] = goff[L], the bound)
//   [L+1, 2L+1)       loc_end
//   [2L+1, 4L+2)      rem_off  (2 groups per expert; rem_off[2L] = goff[L])
//   [4L+2, 6L+2)      rem_end
//   [6L+2, 8L+2)      rem_exp  (= le)
// An empty group (the layout failed, or no rows) is [goff[le], goff[le]).
__global__ void ep_split_groups_kernel(const int32_t* __restrict__ cnt, int me, int ep, int etp, int L,
                                       const int32_t* __restrict__ seg_off, const int32_t* __restrict__ goff,
                                       const int32_t* __restrict__ gcount, int32_t* __restrict__ split) {
  const int E = ep * L, d = me / etp;
  int32_t* loc_off = split;
  int32_t* loc_end = split + L + 1;
  int32_t* rem_off = split + 2 * L + 1;
  int32_t* rem_end = split + 4 * L + 2;
  int32_t* rem_exp = split + 6 * L + 2;
  for (int le = threadIdx.x; le <= L; le += blockDim.x) {
    if (le == L) {
      loc_off[L] = goff[L];
      rem_off[2 * L] = goff[L];
      continue;
    }
    const int32_t g0 = goff[le], g1 = goff[le + 1];
    const bool live = gcount[le] > 0;
    const int32_t s = live ? seg_off[d * L + le] : g0;
    const int32_t c = live ? max(cnt[me * E + d * L + le], 0) : 0;
    loc_off[le] = s;
    loc_end[le] = s + c;
    rem_off[2 * le] = g0;
    rem_end[2 * le] = s;
    rem_off[2 * le + 1] = s + c;
    rem_end[2 * le + 1] = live ? g1 : s + c;
    rem_exp[2 * le] = rem_exp[2 * le + 1] = le;
  }
}

int ep_split_groups(const int32_t* cnt_local, int me, int ep, int etp, int L, const int32_t* seg_off,
                    const int32_t* goff, const int32_t* gcount, int32_t* split, cudaStream_t st) {
  ep_split_groups_kernel<<<1, 128, 0, st>>>(cnt_local, me, ep, etp, L, seg_off, goff, gcount, split);
  B200MOE_CHECK_LAUNCH("ep_split_groups");
  return B200MOE_OK;
}

int ep_expand(void* buf, int64_t H, const int32_t* goff, const int32_t* gcount, int G, const void* dup,
              int phase, cudaStream_t st) {
  if (G <= 0) return B200MOE_OK;
  dim3 grid(256u, (unsigned)G);
  ep_expand_kernel<<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(buf), H, goff, gcount,
                                         static_cast<const int2*>(dup), phase);
  B200MOE_CHECK_LAUNCH("ep_expand");
  return B200MOE_OK;
}

}  // namespace b200moe
