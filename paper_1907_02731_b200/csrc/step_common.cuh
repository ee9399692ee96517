// step_common.cuh — device helpers shared by the fused step kernels
// (fused_ws.cuh, fused_rs.cuh, fused_mc.cuh): the persistent schedule's plane
// stream, the register-ring switch, packed FFMA2, the EXACT/FAST arithmetic
// policy and the canonical 32-column reduction tree.
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "sfseg_types.cuh"

namespace sfk {

// The planes a CTA walks: its schedule segments (tile, [ta, tb)) in order;
// for each, input planes ta-RT .. tb+RT-1 (relative to out_t0).
struct PlaneStream {
    const int4* seg;
    int n, i;
    int tile_x, tile_y, ta, tb, p;
    bool done;
    int RT, tiles_x;

    __device__ void load_seg() {
        const int4 s = seg[i];
        tile_y = s.x / tiles_x;
        tile_x = s.x - tile_y * tiles_x;
        ta = s.y;
        tb = s.z;
        p = ta - RT;
    }
    __device__ void init(const int4* segs, int nseg, int rt, int tx) {
        seg = segs;
        n = nseg;
        i = 0;
        RT = rt;
        tiles_x = tx;
        done = nseg <= 0;
        if (!done) load_seg();
    }
    __device__ void next() {
        ++p;
        if (p >= tb + RT) {
            ++i;
            if (i >= n)
                done = true;
            else
                load_seg();
        }
    }
};

// switch on the ring slot so every ring index is a compile-time constant
// (the ring stays in registers)
#define SFK_RING_CASE(S_, fn)                                                   \
    case S_:                                                                    \
        if constexpr (S_ < K) fn(std::integral_constant<int, (S_ < K ? S_ : 0)>{}); \
        break;
#define SFK_RING_SWITCH(slot, fn)                                               \
    switch (slot) {                                                             \
        SFK_RING_CASE(0, fn)                                                    \
        SFK_RING_CASE(1, fn)                                                    \
        SFK_RING_CASE(2, fn)                                                    \
        SFK_RING_CASE(3, fn)                                                    \
        SFK_RING_CASE(4, fn)                                                    \
        SFK_RING_CASE(5, fn)                                                    \
        SFK_RING_CASE(6, fn)                                                    \
        SFK_RING_CASE(7, fn)                                                    \
        SFK_RING_CASE(8, fn)                                                    \
        default:                                                                \
            break;                                                              \
    }

// packed fma.rn.f32x2 (sm_100a FFMA2); with a broadcast tap ptxas encodes
// the tap as a .F32 uniform-register operand
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// arithmetic policy: EXACT (separately rounded) or FAST (fused)
template <bool FMA>
struct Arith {
    // acc + w * v
    static __device__ __forceinline__ float mac(float acc, float w, float v) {
        if constexpr (FMA)
            return fmaf(w, v, acc);
        else
            return xadd(acc, xmul(w, v));
    }
    static __device__ __forceinline__ float mul(float a, float b) {
        if constexpr (FMA)
            return a * b;
        else
            return xmul(a, b);
    }
    // packed forms. EXACT uses two FFMA2 per pair and tap: p = v*w + 0 (the
    // rounded product) then acc = p*1 + acc (the rounded sum); one/zero are
    // runtime values so ptxas cannot contract them into one FFMA2.
    static __device__ __forceinline__ float2 mac2(float2 acc, float w, float2 v, float2 one,
                                                  float2 zero) {
        if constexpr (FMA) {
            return ffma2(v, make_float2(w, w), acc);
        } else {
            const float2 p = ffma2(v, make_float2(w, w), zero);
            return ffma2(p, one, acc);
        }
    }
    static __device__ __forceinline__ float2 mul2(float w, float2 v, float2 zero) {
        return ffma2(v, make_float2(w, w), zero);
    }
    // previous-iteration projection (normalize_l2 engine.cpp:176-181,
    // project_binary engine.cpp:196-203). Iteration 1 (mode 0) runs the
    // normalise branch with inv == 1: float(double(y) * 1.0) == y exactly.
    static __device__ __forceinline__ float load_norm(float y, double inv, float inv_f) {
        if constexpr (FMA)
            return y * inv_f;
        else
            return static_cast<float>(static_cast<double>(y) * inv);
    }
    static __device__ __forceinline__ float load_sigmoid(float y, const IterState& st) {
        if constexpr (FMA) {
            const float xu = y * st.inv_f;
            return 1.0f / (1.0f + __expf(-st.lambda_f * (xu - st.theta_f)));
        } else {
            const float xu = static_cast<float>(static_cast<double>(y) * st.inv);
            const double z = st.lambda * (static_cast<double>(xu) - st.theta);
            return static_cast<float>(1.0 / (1.0 + exp(-z)));
        }
    }
    // engine.cpp:116-117: S^p * ((alpha^-1 - f f) * A - B + 2 f * C)
    static __device__ __forceinline__ float recombine(float spv, float fv, float ia, float A,
                                                      float B, float Cc) {
        if constexpr (FMA) {
            return spv * (fmaf(-fv, fv, ia) * A - B + 2.0f * fv * Cc);
        } else {
            const float t1 = xmul(xsub(ia, xmul(fv, fv)), A);
            const float t2 = xsub(t1, B);
            const float t3 = xadd(t2, xmul(xmul(2.0f, fv), Cc));
            return xmul(spv, t3);
        }
    }
};

// canonical 32-column tree (device_common.cuh: butterfly 16, 8, 4, 2, 1) done
// serially by one lane on 32 column sums in shared memory: same operands,
// same order, so the same bits as butterfly_sum32. Evaluated quarter by
// quarter (s4[i] needs columns i, i+4, ..., i+28) to keep few values live.
__device__ __forceinline__ double canonical_s4(const double* v, int i) {
    const double s8a = (v[i] + v[i + 16]) + (v[i + 8] + v[i + 24]);
    const double s8b = (v[i + 4] + v[i + 20]) + (v[i + 12] + v[i + 28]);
    return s8a + s8b;
}
__device__ __forceinline__ double canonical_tree32(const double* v) {
    const double s2a = canonical_s4(v, 0) + canonical_s4(v, 2);
    const double s2b = canonical_s4(v, 1) + canonical_s4(v, 3);
    return s2a + s2b;
}

}  // namespace sfk
