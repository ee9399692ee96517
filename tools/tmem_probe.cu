// Development probe: TMEM load/store throughput per SM (tcgen05.ld/st
// 32x32b.x16 from every warp against its lane quadrant), and the latency of a
// dependent ld -> wait chain. Decides whether a register ring can live in TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>  // 0: loads, 1: stores, 2: load+store (read-modify-write ring update)
__global__ void __launch_bounds__(512, 1) probe(unsigned long long* cyc, float* sink, int iters) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(1.0f + lane + i);
    float acc = 0.0f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t addr = base + (uint32_t)((it & 7) * 16);
        if (MODE == 0 || MODE == 2) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                  "=r"(r[14]), "=r"(r[15])
                : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
        }
        if (MODE == 1 || MODE == 2) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
                    addr),
                "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] += 1;
        }
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc + __uint_as_float(r[0]);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <int MODE>
void run(const char* name, int warps_per_cta) {
    const int grid = 148, iters = 4096;
    unsigned long long* cyc;
    float* sink;
    cudaMalloc(&cyc, grid * 16 * sizeof(unsigned long long));
    cudaMalloc(&sink, grid * 512 * sizeof(float));
    cudaMemset(cyc, 0, grid * 16 * sizeof(unsigned long long));
    probe<MODE><<<grid, 32 * warps_per_cta>>>(cyc, sink, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148 * 16];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid * 16; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes = double(warps_per_cta) * iters * 32 * 16 * 4 * (MODE == 2 ? 2 : 1);
    printf("%-28s warps/CTA %2d: %8.0f cycles (slowest warp)  %7.1f B/clk/SM  %6.1f cyc per op/warp  [%s]\n",
           name, warps_per_cta, mx, bytes / mx, mx / iters, cudaGetErrorString(e));
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    for (int w : {1, 4, 8, 16}) run<0>("tcgen05.ld 32x32b.x16", w);
    for (int w : {1, 4, 8, 16}) run<1>("tcgen05.st 32x32b.x16", w);
    for (int w : {4, 16}) run<2>("ld+st (ring update)", w);
    return 0;
}
