// Development probe: which TMA/mbarrier forms run on this B200 (each variant
// in its own process, since a fault poisons the context).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1907_02731_b200/csrc/device_common.cuh"

struct Args { CUtensorMap tm; float* out; int variant; };

__global__ void k(const __grid_constant__ Args a) {
  __shared__ __align__(128) float buf[256 * 16];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    sfk::mbar_init(&bar, 1);
    if (a.variant & 1) sfk::fence_barrier_init();
    if (a.variant & 2) sfk::prefetch_tensormap(&a.tm);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sfk::mbar_arrive_expect_tx(&bar, a.variant >> 3);
    sfk::tma_load_3d(buf, &a.tm, &bar, (a.variant & 4) ? -3 : (a.variant & 2) ? -4 : (a.variant & 1) ? 3 : 0, (a.variant & 4) ? -2 : 0, 0);
  }
  sfk::mbar_wait(&bar, 0);
  a.out[threadIdx.x] = buf[threadIdx.x];
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int W = argc > 2 ? atoi(argv[2]) : 64, H = 16, T = 2, P = (W + 31) / 32 * 32;
  int bw = argc > 3 ? atoi(argv[3]) : 32;
  float* d; cudaMalloc(&d, sizeof(float) * P * H * T);
  float* h = (float*)malloc(sizeof(float) * P * H * T);
  for (int i = 0; i < P * H * T; ++i) h[i] = (float)i;
  cudaMemcpy(d, h, sizeof(float) * P * H * T, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Args a; a.variant = variant | (bw * 16 * 4) << 3;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T};
  cuuint64_t str[2] = {(cuuint64_t)P * 4, (cuuint64_t)P * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, 16, 1}, es[3] = {1, 1, 1};
  CUresult r = ((EncodeTiledFn)fn)(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMalloc(&a.out, 4096);
  k<<<1, 128>>>(a);
  cudaError_t e = cudaDeviceSynchronize();
  float o[8]; cudaMemcpy(o, a.out, sizeof o, cudaMemcpyDeviceToHost);
  printf("variant %d W=%d bw=%d encode=%d -> %s  out[0..3]=%g %g %g %g\n", variant, W, bw, (int)r, cudaGetErrorString(e), o[0], o[1], o[2], o[3]);
  return e != cudaSuccess;
}
