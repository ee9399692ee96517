// affinity.cuh — the reference's explicit-matrix oracle (oracle.cpp:67-258)
// on the GPU, matrix-free and in fp64, without the 1e6-node cap of
// kOracleMaxNodes (oracle.hpp:25).
//
// The reference materialises the affinity in CSR and multiplies row by row:
//   M_ij = sp_i sp_j pair(i, j) G(dt, dy, dx),  pair = exp(-alpha u) (exact)
//          or base - alpha u (Taylor; base = 1, or C for the channel sum),
//   u = sum_c (f_ci - f_cj)^2,  sp = S^p in fp64 (oracle.cpp:92-97),
//   y_i = sum_j M_ij x_j in ascending column order (oracle.cpp:191-207).
// Here one thread owns a row and regenerates its entries on the fly in the
// same order and with the same separately rounded fp64 operations
// (__dmul_rn / __dadd_rn: no FMA contraction), so the Taylor matvecs are
// bit-identical to the reference's; the exact one differs only through the
// device exp (<= 1 ulp per entry). Entries are never stored: a row costs
// (2rt+1)(2ry+1)(2rx+1)(3C + 6) fp64 operations and reads the neighbours'
// features through L1/L2, so the oracle scales to full BASELINE volumes.
#pragma once

#include <stdint.h>

namespace sfk {

constexpr int kAffMaxTaps = 63;  // 2 * 31 + 1

struct AffArgs {
    const float* f[8];  // feature channels (dense T x H x W), at most 8
    const double* sp;   // S^p per voxel, fp64
    const double* x;
    double* y;
    int T, H, W, C;
    int rt, ry, rx;
    int exact;
    double alpha, base;
    double tt[kAffMaxTaps], ty[kAffMaxTaps], tx[kAffMaxTaps];
};

__global__ void k_affinity_matvec(const __grid_constant__ AffArgs a) {
    const long long n = static_cast<long long>(a.T) * a.H * a.W;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % a.W);
        const int y = static_cast<int>((i / a.W) % a.H);
        const int t = static_cast<int>(i / (static_cast<long long>(a.W) * a.H));
        float fi[8];
        for (int c = 0; c < a.C; ++c) fi[c] = a.f[c][i];
        const double spi = a.sp[i];
        double acc = 0.0;  // fixed ascending-column order per row (oracle.cpp:200-202)
        const int dt0 = max(-a.rt, -t), dt1 = min(a.rt, a.T - 1 - t);
        const int dy0 = max(-a.ry, -y), dy1 = min(a.ry, a.H - 1 - y);
        const int dx0 = max(-a.rx, -x), dx1 = min(a.rx, a.W - 1 - x);
        for (int dt = dt0; dt <= dt1; ++dt)
            for (int dy = dy0; dy <= dy1; ++dy) {
                const double wty = __dmul_rn(a.tt[dt + a.rt], a.ty[dy + a.ry]);
                const long long row = i + (static_cast<long long>(dt) * a.H + dy) * a.W;
                for (int dx = dx0; dx <= dx1; ++dx) {
                    const long long j = row + dx;
                    double u = 0.0;  // oracle.cpp:153-158
                    for (int c = 0; c < a.C; ++c) {
                        const double d = __dsub_rn(static_cast<double>(fi[c]), static_cast<double>(a.f[c][j]));
                        u = __dadd_rn(u, __dmul_rn(d, d));
                    }
                    // oracle.cpp:159-162: sp[i] * sp[j] * pair_factor * kernel.weight(dt, dy, dx)
                    const double pf = a.exact ? exp(__dmul_rn(-a.alpha, u)) : __dsub_rn(a.base, __dmul_rn(a.alpha, u));
                    const double kw = __dmul_rn(wty, a.tx[dx + a.rx]);  // conv3d.hpp:46-50
                    const double w = __dmul_rn(__dmul_rn(__dmul_rn(spi, a.sp[j]), pf), kw);
                    acc = __dadd_rn(acc, __dmul_rn(w, a.x[j]));
                }
            }
        a.y[i] = acc;
    }
}

// S^p in fp64 as the oracle computes it (oracle.cpp:92-97)
__global__ void k_sp64(const float* s, double* sp, long long n, double p) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        sp[i] = p == 0.0 ? 1.0 : pow(static_cast<double>(s[i]), p);
}

// fixed-order fp64 sums: block b sums a strided slice with a fixed tree; the
// host (or k_sum_final) adds the block sums in block order
constexpr int kRedThreads = 256;

template <int OP>  // 0: sum a^2; 1: sum a*b; 2: sum (a/s - b)^2 with s = *scale
__global__ void k_dot_blocks(const double* a, const double* b, const double* scale, long long n,
                             double* out) {
    __shared__ double sh[kRedThreads];
    double acc = 0.0;
    const double s = OP == 2 ? *scale : 1.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double v;
        if (OP == 0) {
            v = __dmul_rn(a[i], a[i]);
        } else if (OP == 1) {
            v = __dmul_rn(a[i], b[i]);
        } else {
            const double d = __dsub_rn(__ddiv_rn(a[i], s), b[i]);
            v = __dmul_rn(d, d);
        }
        acc = __dadd_rn(acc, v);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + k]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

__global__ void k_sum_final(const double* parts, int nb, double* out, int sqrt_it) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s = __dadd_rn(s, parts[b]);
    *out = sqrt_it ? sqrt(s) : s;
}

// x = y / s (power_iteration's y[i] /= ny, and x0 /= n0: a division, as
// oracle.cpp:225 and 236 do)
__global__ void k_div_scale(const double* y, const double* s, double* x, long long n) {
    const double d = *s;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        x[i] = __ddiv_rn(y[i], d);
}

}  // namespace sfk
