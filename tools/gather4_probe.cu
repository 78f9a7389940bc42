// TMA tile::gather4 probe (sm_100a): which smem layout does a 4-row gather
// with a 128B-swizzled 2-D tensor map produce?  Needed before the grouped
// GEMM's producer can load A rows by index (a permute- and expansion-free
// dispatch).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 tools/gather4_probe.cu -lcuda && /tmp/g4
// Prints, for each 16-byte chunk of the 512-byte destination, the (row, col)
// of its first element, and checks it against the row-major 128B-swizzle
// pattern the MMA descriptors expect (chunk c of row i at c ^ (i & 7)).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void probe(const __grid_constant__ CUtensorMap map, uint16_t* out, int r0, int r1, int r2, int r3) {
  __shared__ __align__(1024) uint16_t tile[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(tile);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s),
        "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
        : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(b), "r"(0)
          : "memory");
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int R = 64, K = 64;  // 64 bf16 = 128 B per row: one swizzle atom wide
  uint16_t h[R * K];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < K; ++c) h[r * K + c] = (uint16_t)(r << 8 | c);  // raw bits: (row, col)
  uint16_t *d, *o;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 512);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const int rows[4] = {5, 17, 3, 40};
  for (int box1 = 1; box1 <= 4; box1 *= 4) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    CUresult e = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {64, %d}: encode %d\n", box1, (int)e);
    if (e != CUDA_SUCCESS) continue;
    cudaMemset(o, 0xff, 512);
    probe<<<1, 128>>>(map, o, rows[0], rows[1], rows[2], rows[3]);
    cudaError_t ce = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(ce));
    if (ce != cudaSuccess) return 1;
    uint16_t t[256];
    cudaMemcpy(t, o, 512, cudaMemcpyDeviceToHost);
    int ok = 1;
    for (int i = 0; i < 4; ++i) {
      printf("  smem row %d:", i);
      for (int c = 0; c < 8; ++c) {
        const uint16_t v = t[i * 64 + c * 8];
        printf(" (%d,%d)", v >> 8, v & 255);
        // expected: row rows[i], 16-byte chunk (c ^ (i & 7)) of it
        const int want_col = (c ^ (i & 7)) * 8;
        if ((v >> 8) != rows[i] || (v & 255) != want_col) ok = 0;
      }
      printf("\n");
    }
    printf("  matches row-major 128B swizzle: %s\n", ok ? "yes" : "no");
  }
  return 0;
}
