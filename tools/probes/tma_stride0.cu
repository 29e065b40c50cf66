// Probe: does cuTensorMapEncodeTiled accept a zero global stride (pixel duplication by TMA)?
// Build+run on the GPU box: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/p tma_stride0.cu -lcuda && /tmp/p
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, uint4* out, int n) {
  __shared__ __align__(128) uint4 buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    unsigned d = (unsigned)__cvta_generic_to_shared(buf);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n * 16));
    // coords: (ch0=0, dup=0, x=-1 (one left of the row: zero fill), y=1)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(d), "l"(&map), "r"(0), "r"(0), "r"(-1), "r"(1), "r"(b) : "memory");
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W2 = 8, H2 = 4;
  std::vector<__half> h(W2 * H2 * 8);
  for (int y = 0; y < H2; ++y)
    for (int x = 0; x < W2; ++x)
      for (int c = 0; c < 8; ++c) h[(y * W2 + x) * 8 + c] = __float2half(y * 100 + x * 10 + c);
  __half* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  uint4* out;
  cudaMalloc(&out, 256 * 16);
  cudaMemset(out, 0xff, 256 * 16);
  CUtensorMap map;
  cuuint64_t dims[4] = {8, 2, (cuuint64_t)W2, (cuuint64_t)H2};
  cuuint64_t strides[3] = {0, 16, (cuuint64_t)W2 * 16};
  cuuint32_t box[4] = {8, 2, 5, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode stride0: %d\n", (int)r);
  if (r != CUDA_SUCCESS) {
    // try stride 16 for dup, to make sure the rest works
    strides[0] = 16;
    r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode stride16: %d\n", (int)r);
  }
  const int n = 8 * 2 * 5 / 8;  // 10 uint4 (pixels)
  k<<<1, 32>>>(map, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<__half> o(n * 8);
  cudaMemcpy(o.data(), out, n * 16, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("slot %d: ch0=%g ch7=%g\n", i, __half2float(o[i * 8]), __half2float(o[i * 8 + 7]));
  return 0;
}
