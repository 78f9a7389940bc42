// tcgen05.mma.cta_group::2 with M = 128 (sm_100a): where do the 128 rows of
// D land in the pair's TMEM, and are they bit-identical to the same rows of
// an M = 256 pair MMA?  Needed before the grouped GEMM can run a group's
// half-empty last tile as an M = 128 pair tile.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/m128 tools/m128_probe.cu && /tmp/m128
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

constexpr int KDIM = 64, NDIM = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t sw128(int row, int k) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 3) ^ (row & 7))) << 4) + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((16 >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out, int m) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;              // 16 KB
  uint8_t* sB = smem + 16384;      // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int rows_cta = m / 2;  // 128 (M = 256) or 64 (M = 128)
  for (int i = threadIdx.x; i < rows_cta * KDIM; i += blockDim.x) {
    const int r = i / KDIM, k = i % KDIM;
    *reinterpret_cast<__nv_bfloat16*>(sA + sw128(r, k)) = A[(crank * rows_cta + r) * KDIM + k];
  }
  for (int i = threadIdx.x; i < 128 * KDIM; i += blockDim.x) {
    const int r = i / KDIM, k = i % KDIM;
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128(r, k)) = B[(crank * 128 + r) * KDIM + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  if (crank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NDIM >> 3) << 17) |
                           ((uint32_t)(m >> 4) << 24);
    for (int k = 0; k < KDIM / 16; ++k) {
      const uint64_t ad = desc(su32(sA) + k * 32), bd = desc(su32(sB) + k * 32);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(k));
    }
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            su32(bar)),
        "h"(mask)
        : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
          : "=r"(done) : "r"(su32(bar)), "r"(0) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < NDIM; c += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(32 * w) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) out[((crank * 128) + 32 * w + lane) * NDIM + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  const int MA = 256;
  __nv_bfloat16 *hA = (__nv_bfloat16*)malloc(MA * KDIM * 2), *hB = (__nv_bfloat16*)malloc(NDIM * KDIM * 2);
  float *fA = (float*)malloc(MA * KDIM * 4), *fB = (float*)malloc(NDIM * KDIM * 4);
  srand(1);
  for (int i = 0; i < MA * KDIM; ++i) { hA[i] = __float2bfloat16((rand() % 2001 - 1000) / 500.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < NDIM * KDIM; ++i) { hB[i] = __float2bfloat16((rand() % 2001 - 1000) / 500.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float* dO;
  cudaMalloc(&dA, MA * KDIM * 2); cudaMalloc(&dB, NDIM * KDIM * 2); cudaMalloc(&dO, 256 * NDIM * 4);
  cudaMemcpy(dA, hA, MA * KDIM * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, NDIM * KDIM * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  float* o256 = (float*)malloc(256 * NDIM * 4);
  float* o128 = (float*)malloc(256 * NDIM * 4);
  for (int pass = 0; pass < 2; ++pass) {
    const int m = pass == 0 ? 256 : 128;
    cudaMemset(dO, 0xff, 256 * NDIM * 4);
    probe<<<2, 128, 40000>>>(dA, dB, dO, m);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("m=%d: %s\n", m, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(pass == 0 ? o256 : o128, dO, 256 * NDIM * 4, cudaMemcpyDeviceToHost);
  }
  // reference rows
  auto ref = [&](int r, int c) { double s = 0; for (int k = 0; k < KDIM; ++k) s += (double)fA[r * KDIM + k] * fB[c * KDIM + k]; return s; };
  int bad256 = 0;
  for (int r = 0; r < 256; ++r)
    for (int c = 0; c < NDIM; ++c) if (fabs(o256[r * NDIM + c] - ref(r, c)) > 1e-2) ++bad256;
  printf("M=256: %d mismatches vs reference (row r of CTA r/128, lane r%%128)\n", bad256);
  // M = 128: for every (cta, lane) output row, which A row (0..127) does it hold?
  int identical = 0, found = 0;
  for (int cta = 0; cta < 2; ++cta) {
    for (int lane = 0; lane < 128; ++lane) {
      const float* o = o128 + (cta * 128 + lane) * NDIM;
      int who = -1;
      for (int r = 0; r < 128 && who < 0; ++r) {
        bool ok = true;
        for (int c = 0; c < NDIM && ok; ++c) ok = fabs(o[c] - ref(r, c)) < 1e-2;
        if (ok) who = r;
      }
      if (who >= 0) {
        ++found;
        bool same = true;
        for (int c = 0; c < NDIM; ++c) same &= o[c] == o256[who * NDIM + c];
        identical += same;
      }
      if (lane % 16 == 0) printf("cta %d lanes %3d..%3d -> A rows %d..", cta, lane, lane + 15, who);
      if (lane % 16 == 15) printf("%d\n", who);
    }
  }
  printf("M=128: %d of 256 (cta, lane) rows hold an A row; %d of them bit-identical to the M=256 result\n", found, identical);
  // element-level map: which (row, col) of D = A[0:128] B^T does each output element hold?
  for (int cta = 0; cta < 2; ++cta)
    for (int lane = 0; lane < 128; lane += 8)
      for (int c = 0; c < NDIM; c += 64) {
        const float v = o128[(cta * 128 + lane) * NDIM + c];
        int wr = -1, wc = -1;
        for (int r = 0; r < 256 && wr < 0; ++r)
          for (int cc = 0; cc < NDIM; ++cc)
            if (fabs(v - o256[r * NDIM + cc]) < 1e-6 && v != 0.f) { wr = r; wc = cc; break; }
        printf("  cta %d lane %3d col %3d = %10.4f -> D256[%d][%d]\n", cta, lane, c, v, wr, wc);
      }
  return 0;
}
