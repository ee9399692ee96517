// Issue-rate microbenchmark for the FP32 forms the stencil kernels use on
// sm_100a: FFMA (3 registers), FFMA with a uniform-register tap, FFMA2 (packed
// f32x2) with a broadcast tap, the exact mul-then-add pair written as two
// FFMA2 (product + runtime zero, then sum * runtime one), and LDS widths.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_fp32.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_taps[32];
__constant__ float c_one_zero[2];

constexpr int kIters = 4096;

__device__ __forceinline__ unsigned long long as_u64(float2 a) {
    return *reinterpret_cast<unsigned long long*>(&a);
}
__device__ __forceinline__ float2 as_f2(unsigned long long r) {
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(as_u64(a)), "l"(as_u64(b)), "l"(as_u64(c)));
    return as_f2(r);
}

// 8 independent chains, reg-reg-reg FFMA
__global__ void k_ffma_rrr(float* out, float seed) {
    float a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = seed + threadIdx.x + j; b[j] = seed * (j + 1); }
    const float m = seed * 0.999f + threadIdx.x * 1e-9f;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, b[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = fmaf(b[j], m, a[j]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += a[j] + b[j];
    if (s == 12345.f) out[threadIdx.x] = s;
}

// FFMA with the multiplier from the constant bank (uniform register)
__global__ void k_ffma_const(float* out, float seed) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x + j;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], c_taps[(j + k) & 31], a[(j + 1) & 7]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.f) out[threadIdx.x] = s;
}

// FFMA2, tap broadcast from the constant bank; counts 2 lane-ops per instr
__global__ void k_ffma2_const(float* out, float seed) {
    float2 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = make_float2(seed + threadIdx.x + j, seed - j);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float w = c_taps[(j + k) & 31];
            a[j] = fma2(a[j], make_float2(w, w), a[(j + 1) & 7]);
        }
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
    if (s == 12345.f) out[threadIdx.x] = s;
}

// FFMA2 with all three operands full 64-bit registers
__global__ void k_ffma2_rrr(float* out, float seed) {
    float2 a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = make_float2(seed + threadIdx.x + j, seed - j); b[j] = make_float2(seed * j, seed + 2 * j); }
    const float2 m = make_float2(seed * 0.999f, seed * 0.998f + threadIdx.x * 1e-9f);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma2(a[j], m, b[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = fma2(b[j], m, a[j]);
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y + b[j].x + b[j].y;
    if (s == 12345.f) out[threadIdx.x] = s;
}

// exact pair: p = x*w + zero ; acc = p*one + acc  (2 FFMA2 per 2 voxel-taps)
__global__ void k_exact2(float* out, float seed) {
    float2 acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] = make_float2(seed + j, seed - j + threadIdx.x); }
    const float2 one = make_float2(c_one_zero[0], c_one_zero[0]);
    const float2 zero = make_float2(c_one_zero[1], c_one_zero[1]);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float w = c_taps[j];
            float2 p = fma2(acc[(j + 1) & 7], make_float2(w, w), zero);
            acc[j] = fma2(p, one, acc[j]);
        }
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += acc[j].x + acc[j].y;
    if (s == 12345.f) out[threadIdx.x] = s;
}

// scalar exact pair: FMUL (const tap) + FADD
__global__ void k_exact1(float* out, float seed) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] = seed + j + threadIdx.x; }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(acc[(j + 1) & 7], c_taps[j]));
    }
    float s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int W>
__global__ void k_lds(float* out, float seed) {
    __shared__ __align__(16) float sm[4096 * 2];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = seed + i;
    __syncthreads();
    float acc = 0;
    for (int i = 0; i < kIters; ++i) {
        int base = ((threadIdx.x * W) + (i & 7) * 32 * W) & (8192 - 1);
        if (W == 1) acc += sm[base];
        if (W == 2) { float2 v = *reinterpret_cast<float2*>(&sm[base]); acc += v.x + v.y; }
        if (W == 4) { float4 v = *reinterpret_cast<float4*>(&sm[base]); acc += v.x + v.y + v.z + v.w; }
    }
    if (acc == 12345.f) out[threadIdx.x] = acc;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <typename K>
float time_kernel(K kern, int blocks, int threads, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, 1.0001f);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1.0001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    float taps[32]; for (int i = 0; i < 32; ++i) taps[i] = 0.9f + i * 1e-3f;
    cudaMemcpyToSymbol(c_taps, taps, sizeof taps);
    float oz[2] = {1.0f, 0.0f};
    cudaMemcpyToSymbol(c_one_zero, oz, sizeof oz);
    float* out; cudaMalloc(&out, 1 << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d, max clock %d MHz\n", sms, clk / 1000);
    const int blocks = sms * 8, threads = 256;
    const double lanes = double(blocks) * threads;
    struct { const char* name; void (*k)(float*, float); double lane_ops_per_iter; } tests[] = {
        {"ffma_rrr (1 op/instr)", k_ffma_rrr, 16},
        {"ffma_const (1 op/instr)", k_ffma_const, 16},
        {"ffma2_const (2 op/instr)", k_ffma2_const, 32},
        {"ffma2_rrr (2 op/instr)", k_ffma2_rrr, 32},
        {"exact2 (voxel-taps)", k_exact2, 16},
        {"exact1 fmul+fadd (voxel-taps)", k_exact1, 8},
    };
    for (auto& t : tests) {
        float ms = time_kernel(t.k, blocks, threads, out);
        double ops = lanes * kIters * t.lane_ops_per_iter;
        printf("%-32s %8.3f ms  %8.2f Tlane-op/s  %6.1f lane-op/clk/SM @max\n", t.name, ms,
               ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    struct { const char* name; void (*k)(float*, float); double bytes; } lt[] = {
        {"lds32", k_lds<1>, 4}, {"lds64", k_lds<2>, 8}, {"lds128", k_lds<4>, 16}};
    for (auto& t : lt) {
        float ms = time_kernel(t.k, blocks, threads, out);
        double by = lanes * kIters * t.bytes;
        printf("%-32s %8.3f ms  %8.2f B/clk/SM @max\n", t.name, ms, by / (ms * 1e-3) / sms / (clk * 1e3));
    }
    size_t n = (size_t(1) << 30) / 16;
    float4 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_copy<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k_copy<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1 GiB: %.1f GB/s (read+write)\n", 2.0 * n * 16 * 10 / (ms * 1e-3) / 1e9);
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
