// fused_step.cuh — one SFSeg power-iteration step as ONE sm_100a kernel.
//
// Replaces, per iteration, the reference's products pass (engine.cpp:92-100),
// three convolve_separable calls of three axis passes each (conv3d.cpp:80-185),
// the recombination and channel sum (engine.cpp:107-120, 157-162) and the
// sum-of-squares / max scans of normalize_l2 and project_binary
// (engine.cpp:168-205). The normalisation and sigmoid of the PREVIOUS
// iteration are applied on load, so the iterate makes one HBM round trip per
// iteration: read y_k (+ S^p and the feature channels), write y_{k+1}.
//
// Data layout in HBM: row-pitched fp32 volumes, frame-major. A CTA owns a
// TY x TX tile and streams along t through the segments the host scheduler
// gave it (persistent grid, one CTA per SM; neighbouring tiles advance through
// the same frames together, so the halo rows they share come from L2).
//
// Fields. u = S^p x is convolved as a scalar field; for every channel c the
// two fields F_c u and F_c^2 u are kept interleaved as one float2 field, so
// their x, y and t passes run as packed FFMA2 (sm_100a f32x2) with a
// broadcast tap: the same rounding as two scalar operations, half the issue.
//
// Per input plane:
//   1. TMA brings a (TY+2R) x BW halo tile of y_k, S^p and F_c into shared
//      memory (out-of-volume -> +0, the reference's zero padding);
//   2. products: the previous iteration's normalise/sigmoid, then u, F u,
//      F^2 u (engine.cpp:92-100), float4-vectorised;
//   3. x-pass shared -> shared (register strips); meanwhile the interior
//      S^p/F_c are parked for the epilogue and the previous plane's canonical
//      reduction is finished by warp 0; then the stage goes back to TMA;
//   4. y-pass shared -> a per-thread register ring of the last 2RT+1
//      y-filtered planes (QY rows x 1 column per thread);
//   5. t-pass out of the ring, recombination, channel sum, store.
// EXACT (FMA == false): every product and sum rounded separately with the taps
// and accumulation order of conv3d.cpp, so y_{k+1} is bit-identical to the
// reference's sfseg_step on the same x_k. FAST (FMA == true): the same order
// with fused multiply-adds and a float normalisation.
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "sfseg_types.cuh"

namespace sfk {

template <int RT, int R, int CG, int TY, int TX, int QY, int STAGES>
struct FusedGeom {
    static constexpr int K = 2 * RT + 1;        // t-ring depth
    static constexpr int NIN = 2 + CG;           // raw inputs: x, S^p, F_c
    static constexpr int BH = TY + 2 * R;        // halo tile rows
    // TMA faults on an innermost box coordinate that is not 16-byte aligned,
    // so the x halo is rounded up to whole float4s: the box starts at
    // x0 - RX4 and the x-pass reads from column XOFF = RX4 - R.
    static constexpr int RX4 = (R + 3) / 4 * 4;
    static constexpr int XOFF = RX4 - R;
    static constexpr int BW = TX + 2 * RX4;               // TMA box width
    static constexpr int BW4 = BW / 4;
    static constexpr int FB = (BH * BW + 31) / 32 * 32;   // one raw field (128 B aligned)
    // product buffers: lanes of the x-pass take consecutive rows, so every row
    // stride is an odd number of float4 (conflict-free LDS.128)
    static constexpr int BWU = BW + 4;                    // u rows
    static constexpr int BWP = 2 * BW + 4;                // (F u, F^2 u) rows
    static constexpr int PBU = (BH * BWU + 31) / 32 * 32;
    static constexpr int PBP = (BH * BWP + 31) / 32 * 32;
    static constexpr int TXU = TX + 4;                    // x-pass output rows
    static constexpr int TXQ = 2 * TX + 4;
    static constexpr int XBU = (BH * TXU + 31) / 32 * 32;
    static constexpr int XBP = (BH * TXQ + 31) / 32 * 32;
    static constexpr int NT = (TY / QY) * TX;             // threads
    static constexpr int SPU = 16, SPP = 8;               // x strip lengths (u, pair)
    static constexpr int NSU = TX / SPU, NSP = TX / SPP;
    static constexpr int XU_ITEMS = NSU * BH, XP_ITEMS = CG * NSP * BH;
    static constexpr int XITEMS = XU_ITEMS + XP_ITEMS;
    static constexpr int XIT = (XITEMS + NT - 1) / NT;    // x strips per thread
    static constexpr int NINU = SPU + 2 * R;              // input columns per u strip
    static constexpr int NINP = SPP + 2 * R;              // input columns per pair strip
    static constexpr int SFR = RT + 1;                    // planes of S^p/F kept for the epilogue
    static constexpr int SFB = TY * TX;
    static constexpr int NBANDS = TY / 4, NHALVES = TX / 32;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
    static constexpr size_t PROD_FLOATS = size_t(PBU) + size_t(CG) * PBP;
    static constexpr size_t XB_FLOATS = size_t(XBU) + size_t(CG) * XBP;
    static constexpr size_t SF_FLOATS = size_t(SFR) * (1 + CG) * SFB;
    static constexpr size_t RED_FLOATS = 2 * (2 * NT + 32);  // 2 buffers: doubles + warp max
    static constexpr size_t SMEM_BYTES =
        (RAW_FLOATS + PROD_FLOATS + XB_FLOATS + SF_FLOATS + RED_FLOATS) * sizeof(float) + 64;
    static_assert(TX == 32 || TX == 64, "tiles are one or two 32-column reduction halves");
    static_assert(QY == 4, "one thread = one canonical 4-row reduction band");
    static_assert(TY % QY == 0, "tile height");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert((BWU / 4) % 2 == 1 && (BWP / 4) % 2 == 1, "conflict-free product rows");
    static_assert((TXU / 4) % 2 == 1 && (TXQ / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

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

template <int RT, int R, int CG, int TY, int TX, int QY, int STAGES, bool FMA>
__global__ void __launch_bounds__(FusedGeom<RT, R, CG, TY, TX, QY, STAGES>::NT, 1)
    fused_step(const __grid_constant__ FusedArgs a) {
    using G = FusedGeom<RT, R, CG, TY, TX, QY, STAGES>;
    using A = Arith<FMA>;
    constexpr int K = G::K, NIN = G::NIN, BH = G::BH, BW = G::BW, FB = G::FB, BW4 = G::BW4;
    constexpr int BWU = G::BWU, BWP = G::BWP, PBU = G::PBU, PBP = G::PBP;
    constexpr int TXU = G::TXU, TXQ = G::TXQ, XBU = G::XBU, XBP = G::XBP;
    constexpr int NT = G::NT, SFR = G::SFR, SFB = G::SFB, XIT = G::XIT;
    constexpr int SPU = G::SPU, SPP = G::SPP;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                      // [STAGES][NIN][FB]       TMA boxes
    float* produ = raw + G::RAW_FLOATS;     // [BH][BWU]               u
    float* prodp = produ + PBU;             // [CG][BH][BWP]           (F u, F^2 u)
    float* xbu = prodp + CG * PBP;          // [BH][TXU]               x-pass of u
    float* xbp = xbu + XBU;                 // [CG][BH][TXQ]           x-pass of pairs
    float* spf = xbp + CG * XBP;            // [SFR][1+CG][TY*TX]      S^p, F_c interior
    double* red = reinterpret_cast<double*>(spf + G::SF_FLOATS);  // [2][NT] column sums
    float* redmax = reinterpret_cast<float*>(red + 2 * NT);       // [2][NT/32] warp max
    uint64_t* mbar = reinterpret_cast<uint64_t*>(redmax + 2 * 32);

    // uniform state that is not needed in registers lives in shared memory:
    // the iteration scalars and thread 0's producer cursor
    __shared__ IterState st;
    __shared__ PlaneStream prodq;
    __shared__ int prod_count;

    const int tid = threadIdx.x;
    griddep_wait();  // PDL: the previous step / finalize has completed
    if (a.st->degenerate) return;  // an earlier iteration hit a zero norm

    const int s0 = a.sched_off[blockIdx.x], s1 = a.sched_off[blockIdx.x + 1];
    if (s0 >= s1) return;

    if (tid == 0) {
        st = *a.st;
        for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        prefetch_tensormap(&a.tm_sp);
        for (int c = 0; c < CG; ++c) prefetch_tensormap(&a.tm_f[c]);
    }
    __syncthreads();

    // ---- producer (thread 0): TMA loads of in-volume planes, STAGES ahead ----
    auto issue_next = [&]() {
        while (!prodq.done) {
            const int tg = a.out_t0 + prodq.p;
            if (tg >= 0 && tg < a.T) break;
            prodq.next();
        }
        if (prodq.done) return;
        const int tg = a.out_t0 + prodq.p;
        const int s = prod_count % STAGES;
        float* dst = raw + static_cast<size_t>(s) * NIN * FB;
        uint64_t* bar = &mbar[s];
        mbar_arrive_expect_tx(bar, NIN * BH * BW * sizeof(float));
        const int bx = prodq.tile_x * TX - G::RX4, by = prodq.tile_y * TY - R,
                  bt = tg - a.buf_t0;
        tma_load_3d(dst, &a.tm_x, bar, bx, by, bt);
        tma_load_3d(dst + FB, &a.tm_sp, bar, bx, by, bt);
#pragma unroll
        for (int c = 0; c < CG; ++c) tma_load_3d(dst + (2 + c) * FB, &a.tm_f[c], bar, bx, by, bt);
        ++prod_count;
        prodq.next();
    };
    if (tid == 0) {
        prodq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        prod_count = 0;
        for (int s = 0; s < STAGES; ++s) issue_next();
    }

    // ---- per-thread constant indexing ----
    const int grp = tid / TX;  // rows grp*QY .. grp*QY+QY-1 of the tile (= band grp)
    const int col = tid % TX;
    const int warp = tid >> 5;
    // x-pass strips: lanes take consecutive rows; u strips first, then pairs
    int xsrc[XIT], xdst[XIT];
#pragma unroll
    for (int k = 0; k < XIT; ++k) {
        const int it = tid + k * NT;
        if (it < G::XU_ITEMS) {
            const int r = it % BH, sidx = it / BH;
            xsrc[k] = r * BWU + sidx * SPU;
            xdst[k] = r * TXU + sidx * SPU;
        } else if (it < G::XITEMS) {
            const int jt = it - G::XU_ITEMS;
            const int r = jt % BH, sidx = (jt / BH) % G::NSP, c = jt / (BH * G::NSP);
            xsrc[k] = c * PBP + r * BWP + 2 * sidx * SPP;
            xdst[k] = c * XBP + r * TXQ + 2 * sidx * SPP;
        } else {
            xsrc[k] = -1;
            xdst[k] = 0;
        }
    }
    const float2 one2 = make_float2(a.one, a.one), zero2 = make_float2(a.zero, a.zero);

    float ringu[QY][K];
    float2 ringp[CG][QY][K];
#pragma unroll
    for (int q = 0; q < QY; ++q)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            ringu[q][k] = 0.0f;
#pragma unroll
            for (int c = 0; c < CG; ++c) ringp[c][q][k] = make_float2(0.0f, 0.0f);
        }

    // canonical reduction of the column sums a finished output plane left in
    // red[buf] (warp 0; lane b = band b)
    int pend_to = -1, pend_tile_x = 0, pend_tile_y = 0, pend_buf = 0;
    auto finish_reduction = [&]() {
        if (pend_to < 0 || warp != 0) return;
        const int lane = tid & 31;
        const double* rb = red + pend_buf * NT;
        if (lane < G::NBANDS * G::NHALVES) {
            const int band_l = lane / G::NHALVES, half_l = lane % G::NHALVES;
            const double s = canonical_tree32(rb + band_l * TX + half_l * 32);
            const int band = pend_tile_y * G::NBANDS + band_l;
            const int half = pend_tile_x * G::NHALVES + half_l;
            if (band < a.nbands && half < a.nhalves)
                a.part[(static_cast<size_t>(pend_to - a.part_t0) * a.nbands + band) * a.nhalves + half] = s;
        }
        if (a.last_group) {
            float m = lane < NT / 32 ? redmax[pend_buf * 32 + lane] : 0.0f;
            m = butterfly_max32(m);
            if (lane == 0) atomic_max_nonneg(a.frame_max + (pend_to - a.part_t0), m);
        }
    };

    const float inv_alpha = a.inv_alpha;
    PlaneStream cq;
    cq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
    int cons_count = 0;  // in-volume planes consumed
    int slot = 0;        // ring slot of the current plane
    int pc = 0;          // planes processed (S^p/F ring index)
    int outc = 0;        // output planes emitted (reduction buffer parity)
    while (!cq.done) {
        const int tg = a.out_t0 + cq.p;
        const bool valid = tg >= 0 && tg < a.T;
        if (valid) {
            const int s = cons_count % STAGES;
            mbar_wait(&mbar[s], (cons_count / STAGES) & 1);
            const float* rs = raw + static_cast<size_t>(s) * NIN * FB;
            // (2) products over the halo tile (engine.cpp:92-100), 4 points per item
            const bool sigm = st.mode == 2;
            const double inv = st.mode == 0 ? 1.0 : st.inv;
            const float inv_f = st.mode == 0 ? 1.0f : st.inv_f;
            for (int i = tid; i < BH * BW4; i += NT) {
                const int r = i / BW4, c4 = i - r * BW4;
                const float4 yv = reinterpret_cast<const float4*>(rs)[i];
                const float4 sv = reinterpret_cast<const float4*>(rs + FB)[i];
                float4 xv;
                if (sigm) {
                    xv.x = A::load_sigmoid(yv.x, st);
                    xv.y = A::load_sigmoid(yv.y, st);
                    xv.z = A::load_sigmoid(yv.z, st);
                    xv.w = A::load_sigmoid(yv.w, st);
                } else {
                    xv.x = A::load_norm(yv.x, inv, inv_f);
                    xv.y = A::load_norm(yv.y, inv, inv_f);
                    xv.z = A::load_norm(yv.z, inv, inv_f);
                    xv.w = A::load_norm(yv.w, inv, inv_f);
                }
                float4 u;
                u.x = A::mul(sv.x, xv.x);
                u.y = A::mul(sv.y, xv.y);
                u.z = A::mul(sv.z, xv.z);
                u.w = A::mul(sv.w, xv.w);
                *reinterpret_cast<float4*>(produ + r * BWU + 4 * c4) = u;
#pragma unroll
                for (int cg = 0; cg < CG; ++cg) {
                    const float4 fv = reinterpret_cast<const float4*>(rs + (2 + cg) * FB)[i];
                    // (F S^p X, (F F) S^p X) per point
                    float4 p0, p1;
                    p0.x = A::mul(fv.x, u.x);
                    p0.y = A::mul(A::mul(fv.x, fv.x), u.x);
                    p0.z = A::mul(fv.y, u.y);
                    p0.w = A::mul(A::mul(fv.y, fv.y), u.y);
                    p1.x = A::mul(fv.z, u.z);
                    p1.y = A::mul(A::mul(fv.z, fv.z), u.z);
                    p1.z = A::mul(fv.w, u.w);
                    p1.w = A::mul(A::mul(fv.w, fv.w), u.w);
                    float4* pp = reinterpret_cast<float4*>(prodp + cg * PBP + r * BWP + 8 * c4);
                    pp[0] = p0;
                    pp[1] = p1;
                }
            }
            ++cons_count;
            __syncthreads();  // products ready; every warp left the previous epilogue

            finish_reduction();
            pend_to = -1;

            // park the interior S^p / F_c of this plane for its epilogue
            float* spf_in = spf + (pc % SFR) * (1 + CG) * SFB;
            for (int i = tid; i < TY * (TX / 4); i += NT) {
                const int r = i / (TX / 4), c4 = i - r * (TX / 4);
                const int src = (R + r) * BW + G::RX4 + 4 * c4;
#pragma unroll
                for (int fld = 0; fld <= CG; ++fld)
                    reinterpret_cast<float4*>(spf_in + fld * SFB)[i] =
                        *reinterpret_cast<const float4*>(rs + (1 + fld) * FB + src);
            }

            // (3) x-pass (conv3d.cpp:88-101): out[j] = sum_d w[d] * in[j+d], d
            // ascending. Streaming over input columns m keeps only the strip's
            // accumulators live: output j takes tap m-j when column m arrives,
            // which is exactly d-ascending order for every j.
#pragma unroll
            for (int k = 0; k < XIT; ++k) {
                const int it = tid + k * NT;
                if (it < G::XU_ITEMS) {
                    const float4* src = reinterpret_cast<const float4*>(produ + xsrc[k]);
                    float o[SPU];
                    float4 q4;
#pragma unroll
                    for (int m4 = 0; m4 < (G::XOFF + G::NINU + 3) / 4 * 4; ++m4) {
                        if (m4 % 4 == 0) q4 = src[m4 / 4];
                        const int m = m4 - G::XOFF;  // input column relative to the strip
                        if (m < 0 || m >= G::NINU) continue;
                        const float vin = (m4 % 4 == 0) ? q4.x : (m4 % 4 == 1) ? q4.y
                                        : (m4 % 4 == 2) ? q4.z : q4.w;
#pragma unroll
                        for (int j = 0; j < SPU; ++j) {
                            const int d = m - j;
                            if (d < 0 || d > 2 * R) continue;
                            o[j] = d == 0 ? A::mul(a.taps_x[0], vin) : A::mac(o[j], a.taps_x[d], vin);
                        }
                    }
                    float4* dst = reinterpret_cast<float4*>(xbu + xdst[k]);
#pragma unroll
                    for (int v = 0; v < SPU / 4; ++v)
                        dst[v] = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
                } else if (it < G::XITEMS) {
                    const float4* src = reinterpret_cast<const float4*>(prodp + xsrc[k]);
                    float2 o[SPP];
                    float4 q4;
#pragma unroll
                    for (int m2 = 0; m2 < (G::XOFF + G::NINP + 1) / 2 * 2; ++m2) {
                        if (m2 % 2 == 0) q4 = src[m2 / 2];
                        const int m = m2 - G::XOFF;
                        if (m < 0 || m >= G::NINP) continue;
                        const float2 vin = (m2 % 2 == 0) ? make_float2(q4.x, q4.y)
                                                         : make_float2(q4.z, q4.w);
#pragma unroll
                        for (int j = 0; j < SPP; ++j) {
                            const int d = m - j;
                            if (d < 0 || d > 2 * R) continue;
                            o[j] = d == 0 ? A::mul2(a.taps_x[0], vin, zero2)
                                          : A::mac2(o[j], a.taps_x[d], vin, one2, zero2);
                        }
                    }
                    float4* dst = reinterpret_cast<float4*>(xbp + xdst[k]);
#pragma unroll
                    for (int v = 0; v < SPP / 2; ++v)
                        dst[v] = make_float4(o[2 * v].x, o[2 * v].y, o[2 * v + 1].x, o[2 * v + 1].y);
                }
            }
            __syncthreads();  // x-pass output ready; raw stage s fully read
            if (tid == 0) {
                fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_next();
            }
        }

        // (4) y-pass into the rings (conv3d.cpp:113-135) and t-pass out of
        // them (conv3d.cpp:147-165); planes outside the volume contribute 0.
        float zu[QY];
        float2 zp[CG][QY];
        // y-pass of the u field
        {
            float yv[QY];
            if (valid) {
                // streaming over rows j: output q takes tap j-q (first = w * in)
                const float* src = xbu + (grp * QY) * TXU + col;
#pragma unroll
                for (int j = 0; j < QY + 2 * R; ++j) {
                    const float vin = src[j * TXU];
#pragma unroll
                    for (int q = 0; q < QY; ++q) {
                        const int d = j - q;
                        if (d < 0 || d > 2 * R) continue;
                        yv[q] = d == 0 ? A::mul(a.taps_y[0], vin) : A::mac(yv[q], a.taps_y[d], vin);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < QY; ++q) yv[q] = 0.0f;
            }
            auto t_step = [&](auto slot_c) {
                constexpr int S_ = decltype(slot_c)::value;
#pragma unroll
                for (int q = 0; q < QY; ++q) {
                    ringu[q][S_] = yv[q];
                    float acc = A::mul(a.taps_t[0], ringu[q][(S_ + 1) % K]);
#pragma unroll
                    for (int d = 1; d < K; ++d) acc = A::mac(acc, a.taps_t[d], ringu[q][(S_ + 1 + d) % K]);
                    zu[q] = acc;
                }
            };
            SFK_RING_SWITCH(slot, t_step)
        }
        // y-pass of the (F u, F^2 u) pairs
#pragma unroll
        for (int c = 0; c < CG; ++c) {
            float2 yv[QY];
            if (valid) {
                const float2* src =
                    reinterpret_cast<const float2*>(xbp + c * XBP + (grp * QY) * TXQ) + col;
#pragma unroll
                for (int j = 0; j < QY + 2 * R; ++j) {
                    const float2 vin = src[j * (TXQ / 2)];
#pragma unroll
                    for (int q = 0; q < QY; ++q) {
                        const int d = j - q;
                        if (d < 0 || d > 2 * R) continue;
                        yv[q] = d == 0 ? A::mul2(a.taps_y[0], vin, zero2)
                                       : A::mac2(yv[q], a.taps_y[d], vin, one2, zero2);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < QY; ++q) yv[q] = make_float2(0.0f, 0.0f);
            }
            auto t_step = [&](auto slot_c) {
                constexpr int S_ = decltype(slot_c)::value;
#pragma unroll
                for (int q = 0; q < QY; ++q) {
                    ringp[c][q][S_] = yv[q];
                    float2 acc = A::mul2(a.taps_t[0], ringp[c][q][(S_ + 1) % K], zero2);
#pragma unroll
                    for (int d = 1; d < K; ++d)
                        acc = A::mac2(acc, a.taps_t[d], ringp[c][q][(S_ + 1 + d) % K], one2, zero2);
                    zp[c][q] = acc;
                }
            };
            SFK_RING_SWITCH(slot, t_step)
        }
        slot = (slot + 1 == K) ? 0 : slot + 1;

        // (5) recombination, channel sum, store; column sums for the reduction
        const int out_p = cq.p - RT;  // output frame (relative) completed now
        if (out_p >= cq.ta) {         // the ring holds 2RT+1 planes of this segment
            const int to = a.out_t0 + out_p;  // global output frame
            const int y0 = cq.tile_y * TY + grp * QY;
            const int x = cq.tile_x * TX + col;
            const bool xin = x < a.W;
            const float* spf_out = spf + ((pc - RT) % SFR) * (1 + CG) * SFB + grp * QY * TX + col;
            float* orow = a.out + (static_cast<size_t>(to - a.out_buf_t0) * a.H + y0) * a.pitch + x;
            double colsum = 0.0;
            float cmax = 0.0f;
            const bool first = a.first_group;
            const int rows = xin ? min(QY, a.H - y0) : 0;
#pragma unroll
            for (int q = 0; q < QY; ++q) {
                // earlier channel groups' partial sum (channel order, engine.cpp:157-162)
                const float prev = (!first && q < rows) ? orow[q * a.pitch] : 0.0f;
                float acc = 0.0f;
                const float spv = spf_out[q * TX];
#pragma unroll
                for (int cg = 0; cg < CG; ++cg) {
                    const float fv = spf_out[(1 + cg) * SFB + q * TX];
                    const float term =
                        A::recombine(spv, fv, inv_alpha, zu[q], zp[cg][q].y, zp[cg][q].x);
                    acc = cg > 0 ? xadd(acc, term) : (first ? term : xadd(prev, term));
                }
                if (q < rows)
                    orow[q * a.pitch] = acc;
                else
                    acc = 0.0f;
                colsum += static_cast<double>(acc) * static_cast<double>(acc);
                cmax = fmaxf(cmax, acc);
            }
            if (a.last_group) {
                if (!valid && pend_to >= 0) {  // finish the previous plane first
                    __syncthreads();
                    finish_reduction();
                    pend_to = -1;
                }
                const int buf = outc & 1;
                red[buf * NT + tid] = colsum;
                const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                if ((tid & 31) == 0) redmax[buf * 32 + warp] = __int_as_float(wm);
                pend_to = to;
                pend_tile_x = cq.tile_x;
                pend_tile_y = cq.tile_y;
                pend_buf = buf;
                ++outc;
                if (!valid) {  // no barrier follows before the next epilogue
                    __syncthreads();
                    finish_reduction();
                    pend_to = -1;
                }
            }
        }
        ++pc;
        cq.next();
    }
    __syncthreads();
    finish_reduction();
}

}  // namespace sfk
