// aux_kernels.cuh — the non-stencil device work of the SFSeg path:
// validation, guard rescale, S^p, canonical reductions and their finalize,
// the projection/materialise transform, hard mask, metrics, and the generic
// (any-radius) multi-pass stencil used where no fused instantiation exists.
#pragma once

#include <math.h>

#include "device_common.cuh"
#include "sfseg_types.cuh"
#include "step_common.cuh"  // Arith

namespace sfk {

constexpr int kAuxThreads = 256;

struct Vol {  // pitched device volume view
    float* p;
    int T, H, W, pitch;
    __host__ __device__ size_t at(int t, int y, int x) const {
        return (static_cast<size_t>(t) * H + y) * pitch + x;
    }
};

// (t, y, x) of a pitched volume: blocks stride over rows (one division per
// row, not per voxel), threads over x. The 64-bit div/mod per voxel of a flat
// index kept these streaming kernels at ~0.9 TB/s (ncu, r01h launch list).
#define SFK_FOR_VOXELS(v, t, y, x)                                                      \
    for (long long _r = blockIdx.x, _nr = (long long)(v).T * (v).H; _r < _nr;            \
         _r += gridDim.x)                                                                \
        for (int t = (int)(_r / (v).H), y = (int)(_r % (v).H), _once = 1; _once;         \
             _once = 0)                                                                  \
            _Pragma("unroll 4") for (int x = threadIdx.x; x < (v).W; x += blockDim.x)

// FeatureVolume::validate (volume.cpp:72-84): finite, and >= 0 if required.
__global__ void k_validate(Vol v, int need_nonneg, int* flags) {
    int bad = 0;
    SFK_FOR_VOXELS(v, t, y, x) {
        const float a = v.p[v.at(t, y, x)];
        if (!isfinite(a)) bad |= 1;
        if (need_nonneg && a < 0.0f) bad |= 2;
    }
    if (bad) atomicOr(flags, bad);
}

// per-block min/max for the unit-range guard (engine.cpp:229-233)
__global__ void k_minmax_blocks(Vol v, float* bmin, float* bmax) {
    __shared__ float smin[kAuxThreads], smax[kAuxThreads];
    float lo = INFINITY, hi = -INFINITY;
    SFK_FOR_VOXELS(v, t, y, x) {
        const float a = v.p[v.at(t, y, x)];
        lo = fminf(lo, a);
        hi = fmaxf(hi, a);
    }
    smin[threadIdx.x] = lo;
    smax[threadIdx.x] = hi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            smin[threadIdx.x] = fminf(smin[threadIdx.x], smin[threadIdx.x + s]);
            smax[threadIdx.x] = fmaxf(smax[threadIdx.x], smax[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bmin[blockIdx.x] = smin[0];
        bmax[blockIdx.x] = smax[0];
    }
}

__global__ void k_minmax_final(const float* bmin, const float* bmax, int n, float* out2) {
    __shared__ float smin[kAuxThreads], smax[kAuxThreads];
    float lo = INFINITY, hi = -INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        lo = fminf(lo, bmin[i]);
        hi = fmaxf(hi, bmax[i]);
    }
    smin[threadIdx.x] = lo;
    smax[threadIdx.x] = hi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            smin[threadIdx.x] = fminf(smin[threadIdx.x], smin[threadIdx.x + s]);
            smax[threadIdx.x] = fmaxf(smax[threadIdx.x], smax[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out2[0] = smin[0];
        out2[1] = smax[0];
    }
}

// scale_channel_into_unit_range (engine.cpp:234-242): IEEE ops, no FMA.
__global__ void k_unit_range(Vol v, const float* lohi) {
    const float lo = lohi[0], hi = lohi[1];
    if (lo >= 0.0f && hi <= 1.0f) return;  // leave the bits alone
    SFK_FOR_VOXELS(v, t, y, x) {
        float& a = v.p[v.at(t, y, x)];
        if (hi > lo)
            a = __fdiv_rn(__fsub_rn(a, lo), __fsub_rn(hi, lo));
        else
            a = fminf(fmaxf(lo, 0.0f), 1.0f);
    }
}

// Q = sum_c f_c^2 in channel order (fused_mc.cuh, FAST): one launch per
// channel, q = f*f for the first, then q = fma(f, f, q)
__global__ void k_sq_acc(Vol q, Vol f, int first) {
    SFK_FOR_VOXELS(q, t, y, x) {
        const size_t i = q.at(t, y, x);
        const float v = f.p[i];
        q.p[i] = first ? v * v : fmaf(v, v, q.p[i]);
    }
}

// u = S^p T(x) for the multi-channel FAST step (fused_mc.cuh reads U boxes):
// T = identity at iteration 1 (x = S or x0) and in normalise mode (FAST
// applies 1/||y|| at the output), the FAST sigmoid in binarised iterations
// (engine.cpp:92-100, 185-205). The same product the kernel's old in-box
// form computed, bit for bit. Also k_make_u's output of a step's last
// launch (write_u) is the same S^p * y.
__global__ void k_make_u(Vol xv, Vol sp, Vol u, const IterState* __restrict__ st) {
    griddep_wait();  // PDL: the previous finalize wrote st
    if (st->stop) return;  // sfseg_solve_until already stopped
    const bool sig = st->mode == 2;
    const IterState s = *st;
    SFK_FOR_VOXELS(u, t, y, x) {
        const size_t i = u.at(t, y, x);
        const float v = xv.p[i];
        u.p[i] = sp.p[i] * (sig ? Arith<true>::load_sigmoid(v, s) : v);
    }
}

// FP32 FMA-pipe peak probe (sfseg_probe_fp32_peak): 8 independent FFMA2
// chains per thread with a broadcast multiplier, the stencils' instruction
// form; 2 lanes x 2 flops per FFMA2 lane-pair
__global__ void k_fma_probe(float* out, float seed, int iters) {
    float2 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = make_float2(seed + threadIdx.x + j, seed - j);
    const float2 m = make_float2(seed * 0.999f, seed * 0.999f);
    const float2 c = make_float2(seed * 1e-3f, seed * 2e-3f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = ffma2(a[j], m, c);
    }
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
    if (s == 1234.5f) out[threadIdx.x] = s;  // keeps the chains live
}

// Halo push of the time-sharded solve: the rank's edge frames of the new
// iterate into a neighbour's halo frames (dst is peer memory: NVLink stores)
__global__ void k_halo_push(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

// float(pow(double(a), p)) without the cost of pow's extended-precision path:
// exp2(p * log2(a)) in double is within ~1e-14 relative of the true power, so
// its float rounding is the same as pow's unless it lies that close to a
// float rounding midpoint; only those (rare) values take pow().
__device__ __forceinline__ float pow_to_float(float a, double p) {
    if (a == 0.0f) return 0.0f;  // p > 0 here
    const double r = exp2(p * log2(static_cast<double>(a)));
    const float f = __double2float_rn(r);
    if (r > 0.0 && r < 3.0e38) {
        const double fd = static_cast<double>(f);
        const double lo = 0.5 * (fd + static_cast<double>(nextafterf(f, 0.0f)));
        const double hi = 0.5 * (fd + static_cast<double>(nextafterf(f, INFINITY)));
        const double eps = 1e-13 * r;
        if (fabs(r - lo) > eps && fabs(r - hi) > eps) return f;
    }
    return static_cast<float>(pow(static_cast<double>(a), p));
}

// pow_volume (engine.cpp:52-71): float(pow(double s, p)); p==0 -> 1, p==1 -> copy
__global__ void k_pow(Vol s, Vol out, double p) {
    SFK_FOR_VOXELS(s, t, y, x) {
        const float a = s.p[s.at(t, y, x)];
        float r;
        if (p == 0.0)
            r = 1.0f;
        else if (p == 1.0)
            r = a;
        else
            r = pow_to_float(a, p);
        out.p[out.at(t, y, x)] = r;
    }
}

// Canonical sum(x^2) partials + per-frame max over an existing volume.
// One warp per (frame, 4-row band, 32-column half); lanes = columns.
__global__ void k_partials(Vol v, double* part, float* frame_max, int nbands, int nhalves,
                           int t_off) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nwarps = (long long)v.T * nbands * nhalves;
    if (warp >= nwarps) return;
    const int half = warp % nhalves;
    const int band = (warp / nhalves) % nbands;
    const int t = warp / (nhalves * nbands);
    const int x = half * 32 + lane;
    double colsum = 0.0;
    float m = 0.0f;
    for (int r = 0; r < 4; ++r) {
        const int y = band * 4 + r;
        float a = 0.0f;
        if (x < v.W && y < v.H) a = v.p[v.at(t, y, x)];
        colsum += static_cast<double>(a) * static_cast<double>(a);
        m = fmaxf(m, a);
    }
    const double s = butterfly_sum32(colsum);
    m = butterfly_max32(m);
    if (lane == 0) {
        part[(static_cast<size_t>(t + t_off) * nbands + band) * nhalves + half] = s;
        atomic_max_nonneg(frame_max + t + t_off, m);
    }
}

// frame_sum[t] = fixed-order reduction of the frame's partials: thread i sums
// entries i, i+256, ... sequentially; then a fixed shared-memory tree.
__global__ void k_finalize_frames(const double* part, int per_frame, double* frame_sum,
                                  int t0) {
    __shared__ double s[kAuxThreads];
    griddep_wait();  // PDL: the step's partials are complete
    const int t = blockIdx.x + t0;
    const double* p = part + static_cast<size_t>(t) * per_frame;
    double acc = 0.0;
    for (int i = threadIdx.x; i < per_frame; i += blockDim.x) acc += p[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) frame_sum[t] = s[0];
}

// Total over frames (fixed order: same tree as above over frame index) and
// the scalars the next iteration applies on load (engine.cpp:168-205).
// mode_next: 1 = normalise, 2 = normalise + sigmoid; lambda from the host.
// Shared by k_finalize_total and the last block of k_finalize (one block of
// kAuxThreads threads); frame_sum is read through L2 (written by other blocks).
__device__ __forceinline__ void finalize_total_block(const double* frame_sum, float* frame_max, int T,
                                                     IterState* st, double* norms, int iter_index,
                                                     int mode_next, double lambda,
                                                     double threshold_frac) {
    __shared__ double s[kAuxThreads];
    __shared__ float sm[kAuxThreads];
    double acc = 0.0;
    float m = 0.0f;
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
        acc += __ldcg(frame_sum + i);
        m = fmaxf(m, __ldcg(frame_max + i));
        frame_max[i] = 0.0f;  // reset for the next iteration
    }
    s[threadIdx.x] = acc;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) {
            s[threadIdx.x] += s[threadIdx.x + k];
            sm[threadIdx.x] = fmaxf(sm[threadIdx.x], sm[threadIdx.x + k]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double norm = sqrt(s[0]);
        if (norms) norms[iter_index] = norm;
        IterState n = *st;
        n.norm = norm;
        if (norm == 0.0) {
            n.degenerate = 1;
        } else if (!n.degenerate) {
            n.inv = 1.0 / norm;
            n.max_raw = sm[0];
            // max of the unit vector: the map y -> float(double(y)*inv) is monotone
            n.max_unit = static_cast<float>(static_cast<double>(sm[0]) * n.inv);
            n.mode = mode_next;
            n.lambda = lambda;
            n.theta = threshold_frac * static_cast<double>(n.max_unit);
            n.inv_f = static_cast<float>(n.inv);
            n.theta_f = static_cast<float>(n.theta);
            n.lambda_f = static_cast<float>(n.lambda);
        }
        *st = n;
    }
}

__global__ void k_finalize_total(const double* frame_sum, float* frame_max, int T,
                                 IterState* st, double* norms, int iter_index, int mode_next,
                                 double lambda, double threshold_frac) {
    griddep_wait();  // PDL: the frame sums (or their gather) are complete
    finalize_total_block(frame_sum, frame_max, T, st, norms, iter_index, mode_next, lambda,
                         threshold_frac);
}

// k_finalize_frames + k_finalize_total in one launch (one per iteration
// instead of two): block t sums frame t exactly as k_finalize_frames, and the
// last block to finish runs finalize_total_block (threadfence-reduction
// pattern; *ticket is 0 on entry and is reset by that block). Same operands in
// the same order as the two-launch path, so the same bits.
__global__ void k_finalize(const double* part, int per_frame, double* frame_sum, float* frame_max,
                           unsigned int* ticket, IterState* st, double* norms, int iter_index,
                           int mode_next, double lambda, double threshold_frac) {
    __shared__ double s[kAuxThreads];
    __shared__ bool is_last;
    griddep_wait();  // PDL: the step's partials are complete
    if (st->stop) return;  // sfseg_solve_until already stopped: the state stays as it is
    const int t = blockIdx.x;
    const double* p = part + static_cast<size_t>(t) * per_frame;
    double acc = 0.0;
    for (int i = threadIdx.x; i < per_frame; i += blockDim.x) acc += p[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        frame_sum[t] = s[0];
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    finalize_total_block(frame_sum, frame_max, gridDim.x, st, norms, iter_index, mode_next, lambda,
                         threshold_frac);
    if (threadIdx.x == 0) *ticket = 0u;
}

// x = T(y): the projection of the state, materialised into a volume.
__global__ void k_transform(Vol y, Vol out, const IterState* stp) {
    const IterState st = *stp;
    SFK_FOR_VOXELS(y, t, yy, x) {
        const float a = y.p[y.at(t, yy, x)];
        float r = a;
        if (st.mode >= 1) r = static_cast<float>(static_cast<double>(a) * st.inv);
        if (st.mode == 2) {
            const double z = st.lambda * (static_cast<double>(r) - st.theta);
            r = static_cast<float>(1.0 / (1.0 + exp(-z)));
        }
        out.p[out.at(t, yy, x)] = r;
    }
}

// max of the projected iterate x = T(y) from the state (T is monotone, so
// max x = T(max y)); used for the hard mask of a time shard
__global__ void k_state_max(const IterState* stp, float* out) {
    const IterState st = *stp;
    float m = st.max_unit;
    if (st.mode == 2) {
        const double z = st.lambda * (static_cast<double>(m) - st.theta);
        m = static_cast<float>(1.0 / (1.0 + exp(-z)));
    }
    *out = m;
}

// max(0, max v) (engine.cpp:189-190, 208-210)
__global__ void k_max(Vol v, float* out) {
    float m = 0.0f;
    SFK_FOR_VOXELS(v, t, y, x) m = fmaxf(m, v.p[v.at(t, y, x)]);
    m = butterfly_max32(m);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

// mask_from_volume with cut = float(frac * max) (engine.cpp:212, volume.cpp:107-114)
// dense <-> pitched copy of `rows` rows of w floats (host transfers stage
// through a dense buffer so the DMA runs as one contiguous copy)
__global__ void k_repitch(const float* __restrict__ src, int src_pitch, float* __restrict__ dst,
                          int dst_pitch, size_t rows, int w) {
    for (size_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float* s = src + r * src_pitch;
        float* d = dst + r * dst_pitch;
        for (int x = threadIdx.x; x < w; x += blockDim.x) d[x] = s[x];
    }
}

__global__ void k_mask(Vol v, const float* maxp, double frac, uint8_t* mask) {
    const float cut = static_cast<float>(frac * static_cast<double>(*maxp));
    SFK_FOR_VOXELS(v, t, y, x) {
        mask[(static_cast<size_t>(t) * v.H + y) * v.W + x] = v.p[v.at(t, y, x)] > cut ? 1 : 0;
    }
}

// angle_degrees / jaccard accumulators (metrics.cpp:22-38, 58-69)
__global__ void k_metrics(Vol xv, Vol ref, const uint8_t* gt, const float* maxp, double frac,
                          double* acc3, unsigned long long* cnt2) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    unsigned long long inter = 0, uni = 0;
    const float cut = maxp ? static_cast<float>(frac * static_cast<double>(*maxp)) : 0.0f;
    SFK_FOR_VOXELS(xv, t, y, x) {
        const double a = xv.p[xv.at(t, y, x)];
        if (ref.p) {
            const double b = ref.p[ref.at(t, y, x)];
            dot += a * b;
            na += a * a;
            nb += b * b;
        }
        if (gt) {
            const bool va = xv.p[xv.at(t, y, x)] > cut;
            const bool vb = gt[(static_cast<size_t>(t) * xv.H + y) * xv.W + x] != 0;
            inter += (va && vb);
            uni += (va || vb);
        }
    }
    if (ref.p) {
        atomicAdd(acc3 + 0, dot);
        atomicAdd(acc3 + 1, na);
        atomicAdd(acc3 + 2, nb);
    }
    if (gt) {
        atomicAdd(cnt2 + 0, inter);
        atomicAdd(cnt2 + 1, uni);
    }
}

// Convergence statistics between two consecutive projected iterates
// x_k = T_k(y_k) and x_{k-1} = T_{k-1}(y_{k-1}) (materialised as k_transform
// does; prev_raw: x_{k-1} is the start vector S / x0 as stored):
// per-block fp64 sums of x_k x_{k-1}, x_k^2, x_{k-1}^2 and (x_k - x_{k-1})^2,
// written to part[block][4]; k_conv_final sums the blocks in block order,
// so the result does not depend on timing.
__device__ __forceinline__ float project_state(float a, const IterState& st) {
    float r = a;
    if (st.mode >= 1) r = static_cast<float>(static_cast<double>(a) * st.inv);
    if (st.mode == 2) {
        const double z = st.lambda * (static_cast<double>(r) - st.theta);
        r = static_cast<float>(1.0 / (1.0 + exp(-z)));
    }
    return r;
}

__global__ void k_conv_stats(Vol cur, const IterState* st_cur, Vol prev, const IterState* st_prev,
                             int prev_raw, double* part) {
    __shared__ double s[4][kAuxThreads];
    if (st_cur->stop) return;  // already stopped: nothing new to compare
    const IterState sc = *st_cur;
    const IterState sp = *st_prev;
    double d = 0.0, na = 0.0, nb = 0.0, df = 0.0;
    SFK_FOR_VOXELS(cur, t, y, x) {
        const double a = project_state(cur.p[cur.at(t, y, x)], sc);
        const float pb = prev.p[prev.at(t, y, x)];
        const double b = prev_raw ? pb : project_state(pb, sp);
        d += a * b;
        na += a * a;
        nb += b * b;
        df += (a - b) * (a - b);
    }
    s[0][threadIdx.x] = d;
    s[1][threadIdx.x] = na;
    s[2][threadIdx.x] = nb;
    s[3][threadIdx.x] = df;
    __syncthreads();
    for (int k = blockDim.x / 2; k > 0; k >>= 1) {
        if (threadIdx.x < k)
            for (int j = 0; j < 4; ++j) s[j][threadIdx.x] += s[j][threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = s[threadIdx.x][0];
}

// The stopping rule itself, on the device: criterion 0 is ||x_k - x_{k-1}||_2 <
// tol (oracle.cpp:234-242), 1 is angle(x_k, x_{k-1}) < tol degrees
// (bench.cpp:75-80, metrics.cpp:22-38). When it holds, st->stop = iter and the
// kernels of the later iterations already in the stream do nothing; the host
// reads the state back once per chunk of iterations, not once per iteration.
__global__ void k_conv_final(const double* part, int nblocks, double* out4, IterState* st, int iter,
                             int criterion, double tol) {
    __shared__ double h[4];
    if (st->stop) return;
    if (threadIdx.x < 4) {
        double acc = 0.0;
        for (int b = 0; b < nblocks; ++b) acc += part[b * 4 + threadIdx.x];
        out4[threadIdx.x] = acc;
        h[threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x != 0 || st->degenerate) return;
    bool stop;
    if (criterion == 0) {
        stop = sqrt(h[3]) < tol;
    } else if (h[1] == 0.0 || h[2] == 0.0) {
        st->stop = -iter;  // angle of a zero vector
        return;
    } else {
        const double cs = fmin(1.0, fmax(-1.0, h[0] / (sqrt(h[1]) * sqrt(h[2]))));
        stop = acos(cs) * 57.295779513082320876798154814105 < tol;
    }
    if (stop) st->stop = iter;
}

__global__ void k_clear_stop(IterState* st) { st->stop = 0; }

// ---- generic (any-radius) stencil: conv3d.cpp:80-167 on pitched volumes --

struct Taps {
    float t[64], y[64], x[64];
    int rt, ry, rx;
};

// convolve_direct (conv3d.cpp:187-243): w = (taps_t * taps_y) * taps_x in
// fp64, acc += w * src over dt, dy, dx ascending, skipping out-of-range
// offsets; separately rounded (the reference build has no FMA)
struct TapsD {
    double t[32], y[32], x[32];
    int rt, ry, rx;
};

__global__ void k_conv_direct(Vol in, Vol out, const __grid_constant__ TapsD k) {
    SFK_FOR_VOXELS(in, t, y, x) {
        double acc = 0.0;
        for (int dt = -k.rt; dt <= k.rt; ++dt) {
            const int tt = t + dt;
            if (tt < 0 || tt >= in.T) continue;
            for (int dy = -k.ry; dy <= k.ry; ++dy) {
                const int yy = y + dy;
                if (yy < 0 || yy >= in.H) continue;
                for (int dx = -k.rx; dx <= k.rx; ++dx) {
                    const int xx = x + dx;
                    if (xx < 0 || xx >= in.W) continue;
                    const double w = __dmul_rn(__dmul_rn(k.t[dt + k.rt], k.y[dy + k.ry]), k.x[dx + k.rx]);
                    acc = __dadd_rn(acc, __dmul_rn(w, static_cast<double>(in.p[in.at(tt, yy, xx)])));
                }
            }
        }
        out.p[out.at(t, y, x)] = static_cast<float>(acc);
    }
}

// products u, fu, f2u (engine.cpp:92-100) with the load transform
__global__ void k_products(Vol xsrc, Vol sp, Vol f, Vol u, Vol fu, Vol f2u,
                           const IterState* stp) {
    const IterState st = *stp;
    SFK_FOR_VOXELS(xsrc, t, y, x) {
        const float yv = xsrc.p[xsrc.at(t, y, x)];
        float xv = yv;
        if (st.mode >= 1) xv = static_cast<float>(static_cast<double>(yv) * st.inv);
        if (st.mode == 2) {
            const double z = st.lambda * (static_cast<double>(xv) - st.theta);
            xv = static_cast<float>(1.0 / (1.0 + exp(-z)));
        }
        const float uu = xmul(sp.p[sp.at(t, y, x)], xv);
        const float fv = f.p[f.at(t, y, x)];
        u.p[u.at(t, y, x)] = uu;
        fu.p[fu.at(t, y, x)] = xmul(fv, uu);
        f2u.p[f2u.at(t, y, x)] = xmul(xmul(fv, fv), uu);
    }
}

__global__ void k_pass_x(Vol in, Vol out, const __grid_constant__ Taps k) {
    SFK_FOR_VOXELS(in, t, y, x) {
        float acc = 0.0f;
        const int dlo = -min(k.rx, x), dhi = min(k.rx, in.W - 1 - x);
        for (int d = dlo; d <= dhi; ++d) acc = xadd(acc, xmul(k.x[d + k.rx], in.p[in.at(t, y, x + d)]));
        out.p[out.at(t, y, x)] = acc;
    }
}

__global__ void k_pass_y(Vol in, Vol out, const __grid_constant__ Taps k) {
    SFK_FOR_VOXELS(in, t, y, x) {
        const int dlo = -min(k.ry, y), dhi = min(k.ry, in.H - 1 - y);
        float acc = 0.0f;
        for (int d = dlo; d <= dhi; ++d) {
            const float p = xmul(k.y[d + k.ry], in.p[in.at(t, y + d, x)]);
            acc = (d == dlo) ? p : xadd(acc, p);
        }
        out.p[out.at(t, y, x)] = acc;
    }
}

__global__ void k_pass_t(Vol in, Vol out, const __grid_constant__ Taps k) {
    SFK_FOR_VOXELS(in, t, y, x) {
        const int dlo = -min(k.rt, t), dhi = min(k.rt, in.T - 1 - t);
        float acc = 0.0f;
        for (int d = dlo; d <= dhi; ++d) {
            const float p = xmul(k.t[d + k.rt], in.p[in.at(t + d, y, x)]);
            acc = (d == dlo) ? p : xadd(acc, p);
        }
        out.p[out.at(t, y, x)] = acc;
    }
}

// recombination + channel accumulation (engine.cpp:113-119, 157-162)
__global__ void k_recombine(Vol a, Vol b, Vol c, Vol sp, Vol f, Vol out, float inv_alpha,
                            int first) {
    SFK_FOR_VOXELS(a, t, y, x) {
        const float fv = f.p[f.at(t, y, x)];
        const float t1 = xmul(xsub(inv_alpha, xmul(fv, fv)), a.p[a.at(t, y, x)]);
        const float t2 = xsub(t1, b.p[b.at(t, y, x)]);
        const float t3 = xadd(t2, xmul(xmul(2.0f, fv), c.p[c.at(t, y, x)]));
        const float term = xmul(sp.p[sp.at(t, y, x)], t3);
        float& o = out.p[out.at(t, y, x)];
        o = first ? term : xadd(o, term);
    }
}

}  // namespace sfk
