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
// Data layout in HBM: row-pitched fp32 volumes, frame-major. Tiles of
// TY x TX output points stream along t: per input plane the CTA
//   1. receives a (TY+2R) x BW halo tile of y_k, S^p and F_c by TMA
//      (out-of-volume -> zero, i.e. the reference's zero padding);
//   2. applies the previous iteration's normalise/sigmoid and forms the
//      1+2C product fields u = S^p x, F u, F^2 u (engine.cpp:92-100);
//   3. x-pass from shared memory into shared memory;
//   4. y-pass from shared memory into a per-thread register ring of the last
//      2RT+1 y-filtered planes;
//   5. t-pass out of the register ring, recombination, store, and the
//      canonical fp64 sum-of-squares + max reductions.
// EXACT arithmetic: every product and sum rounded separately, taps and
// accumulation order of conv3d.cpp, so y_{k+1} is bit-identical to the
// reference's sfseg_step on the same x_k.
#pragma once

#include "device_common.cuh"
#include "sfseg_types.cuh"

namespace sfk {

template <int RT, int R, int CG, int TY, int TX, int QY, int STAGES>
struct FusedGeom {
    static constexpr int K = 2 * RT + 1;        // t-ring depth
    static constexpr int F = 1 + 2 * CG;         // convolved fields
    static constexpr int NIN = 2 + CG;           // raw inputs: x, S^p, F_c
    static constexpr int BH = TY + 2 * R;        // halo tile rows
    // TMA faults on an innermost box coordinate that is not 16-byte aligned,
    // so the x halo is rounded up to whole float4s: the box starts at
    // x0 - RX4 and the x-pass reads from column XOFF = RX4 - R.
    static constexpr int RX4 = (R + 3) / 4 * 4;
    static constexpr int XOFF = RX4 - R;
    static constexpr int BW = TX + 2 * RX4;              // TMA box width (16 B multiple)
    static constexpr int FB = (BH * BW + 31) / 32 * 32;  // one field, 128 B aligned
    static constexpr int TXP = TX + 4;            // x-pass output row stride (bank spread)
    static constexpr int XB = (BH * TXP + 31) / 32 * 32;
    static constexpr int NT = (TY / QY) * TX;     // threads
    static constexpr int SP = 8;                  // x-pass strip length
    static constexpr int NS = TX / SP;            // strips per row
    static constexpr int NV4 = (SP + XOFF + 2 * R + 3) / 4;  // float4 loads per strip
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
    static constexpr size_t PROD_FLOATS = size_t(F) * FB;
    static constexpr size_t XB_FLOATS = size_t(F) * XB;
    static constexpr size_t SMEM_BYTES =
        (RAW_FLOATS + PROD_FLOATS + XB_FLOATS) * sizeof(float) + 64;
    static_assert(TX == 64, "tiles are 64 columns wide (two 32-column reduction halves)");
    static_assert(QY == 4 || QY == 8, "canonical reduction bands are 4 rows");
    static_assert(TY % QY == 0 && TY % 4 == 0, "tile height");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
};

// Which planes a CTA walks: a contiguous range of (tile, output frame) units,
// frame fastest. Each maximal same-tile run is a segment; the CTA processes
// its input planes from 2*RT before the first output to the last output.
struct PlaneStream {
    long long u, u_end;
    int tile, ta, tb, p;
    bool done;
    int RT, Tout;

    __device__ void start_segment() {
        tile = static_cast<int>(u / Tout);
        ta = static_cast<int>(u % Tout);
        const long long left = u_end - u;
        tb = static_cast<int>(left < (long long)(Tout - ta) ? ta + left : Tout);
        p = ta - RT;
    }
    __device__ void init(long long u0, long long u1, int rt, int tout) {
        u = u0;
        u_end = u1;
        RT = rt;
        Tout = tout;
        done = u0 >= u1;
        if (!done) start_segment();
    }
    __device__ void next() {
        ++p;
        if (p >= tb + RT) {
            u += tb - ta;
            if (u >= u_end)
                done = true;
            else
                start_segment();
        }
    }
};

// Previous-iteration projection applied to each loaded voxel
// (normalize_l2 engine.cpp:176-181, project_binary engine.cpp:196-203).
__device__ __forceinline__ float load_transform(float y, const IterState& st) {
    if (st.mode == 0) return y;
    const float xu = static_cast<float>(static_cast<double>(y) * st.inv);
    if (st.mode == 1) return xu;
    const double z = st.lambda * (static_cast<double>(xu) - st.theta);
    return static_cast<float>(1.0 / (1.0 + exp(-z)));
}

template <int RT, int R, int CG, int TY, int QY, int STAGES>
__global__ void __launch_bounds__(FusedGeom<RT, R, CG, TY, 64, QY, STAGES>::NT, 1)
    fused_step_exact(const __grid_constant__ FusedArgs a) {
    using G = FusedGeom<RT, R, CG, TY, 64, QY, STAGES>;
    constexpr int TX = 64;
    constexpr int K = G::K, F = G::F, NIN = G::NIN, BH = G::BH, BW = G::BW, FB = G::FB;
    constexpr int TXP = G::TXP, XB = G::XB, NT = G::NT, SP = G::SP, NS = G::NS;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                        // [STAGES][NIN][FB]
    float* prod = raw + G::RAW_FLOATS;        // [F][FB]  (rows of BW)
    float* xbuf = prod + G::PROD_FLOATS;      // [F][XB]  (rows of TXP)
    uint64_t* mbar = reinterpret_cast<uint64_t*>(xbuf + G::XB_FLOATS);

    const int tid = threadIdx.x;
    const IterState st = *a.st;
    if (st.degenerate) return;  // an earlier iteration hit a zero norm

    const int Tout = a.out_t1 - a.out_t0;
    const long long total = static_cast<long long>(a.tiles_x) * a.tiles_y * Tout;
    const long long u0 = static_cast<long long>(blockIdx.x) * a.units_per_cta;
    const long long u1 = u0 + a.units_per_cta < total ? u0 + a.units_per_cta : total;
    if (u0 >= u1) return;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        prefetch_tensormap(&a.tm_sp);
        for (int c = 0; c < CG; ++c) prefetch_tensormap(&a.tm_f[c]);
    }
    __syncthreads();

    // ---- producer (thread 0): TMA loads of valid planes, STAGES ahead ----
    PlaneStream prodq;
    prodq.init(u0, u1, RT, Tout);
    int prod_count = 0;  // valid planes issued so far
    auto issue_next = [&]() {
        // advance to the next in-volume plane and load it into its stage
        while (!prodq.done) {
            const int tg = a.out_t0 + prodq.p;
            if (tg >= 0 && tg < a.T) break;
            prodq.next();
        }
        if (prodq.done) return;
        const int tg = a.out_t0 + prodq.p;
        const int tile_y = prodq.tile / a.tiles_x, tile_x = prodq.tile % a.tiles_x;
        const int s = prod_count % STAGES;
        float* dst = raw + static_cast<size_t>(s) * NIN * FB;
        uint64_t* bar = &mbar[s];
        mbar_arrive_expect_tx(bar, NIN * BH * BW * sizeof(float));
        const int bx = tile_x * TX - G::RX4, by = tile_y * TY - R, bt = tg - a.buf_t0;
        tma_load_3d(dst, &a.tm_x, bar, bx, by, bt);
        tma_load_3d(dst + FB, &a.tm_sp, bar, bx, by, bt);
        for (int c = 0; c < CG; ++c) tma_load_3d(dst + (2 + c) * FB, &a.tm_f[c], bar, bx, by, bt);
        ++prod_count;
        prodq.next();
    };
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s) issue_next();

    // ---- consumers: all threads ----
    const int grp = tid / TX;          // y-pass row group: rows grp*QY .. +QY
    const int col = tid % TX;
    float ring[F][QY][K];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
        for (int q = 0; q < QY; ++q)
#pragma unroll
            for (int k = 0; k < K; ++k) ring[f][q][k] = 0.0f;

    const float inv_alpha = a.inv_alpha;
    PlaneStream cq;
    cq.init(u0, u1, RT, Tout);
    int cons_count = 0;  // valid planes consumed
    int slot = 0;        // ring slot of the current plane
    while (!cq.done) {
        const int tg = a.out_t0 + cq.p;
        const bool valid = tg >= 0 && tg < a.T;
        const int tile_y = cq.tile / a.tiles_x, tile_x = cq.tile % a.tiles_x;
        if (valid) {
            const int s = cons_count % STAGES;
            mbar_wait(&mbar[s], (cons_count / STAGES) & 1);
            const float* rs = raw + static_cast<size_t>(s) * NIN * FB;
            // (2) products over the halo tile (engine.cpp:92-100)
            for (int i = tid; i < BH * BW; i += NT) {
                const float xv = load_transform(rs[i], st);
                const float u = xmul(rs[FB + i], xv);
                prod[i] = u;
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    const float fv = rs[(2 + c) * FB + i];
                    prod[(1 + 2 * c) * FB + i] = xmul(fv, u);            // F S^p X
                    prod[(2 + 2 * c) * FB + i] = xmul(xmul(fv, fv), u);  // F^2 S^p X
                }
            }
            ++cons_count;
            __syncthreads();  // products ready; raw stage s free
            if (tid == 0) {
                fence_proxy_async();  // generic-proxy reads of stage s before TMA overwrite
                issue_next();
            }

            // (3) x-pass (conv3d.cpp:88-101): acc = 0, += w[d] * in[x+d], d ascending
            for (int it = tid; it < F * NS * BH; it += NT) {
                const int r = it % BH;
                const int sidx = (it / BH) % NS;
                const int f = it / (BH * NS);
                const float* src = prod + f * FB + r * BW + sidx * SP;
                float in[G::NV4 * 4];
#pragma unroll
                for (int v = 0; v < G::NV4; ++v) {
                    const float4 q4 = reinterpret_cast<const float4*>(src)[v];
                    in[4 * v + 0] = q4.x;
                    in[4 * v + 1] = q4.y;
                    in[4 * v + 2] = q4.z;
                    in[4 * v + 3] = q4.w;
                }
                float o[SP];
#pragma unroll
                for (int j = 0; j < SP; ++j) {
                    float acc = 0.0f;
#pragma unroll
                    for (int d = 0; d <= 2 * R; ++d)
                        acc = xadd(acc, xmul(a.taps_x[d], in[G::XOFF + j + d]));
                    o[j] = acc;
                }
                float4* dst = reinterpret_cast<float4*>(xbuf + f * XB + r * TXP + sidx * SP);
#pragma unroll
                for (int v = 0; v < SP / 4; ++v)
                    dst[v] = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
            }
            __syncthreads();  // x-pass output ready
        }

        // (4) y-pass into the ring (conv3d.cpp:113-135): first = w*in, then +=
        // ring slot written this plane; planes outside the volume contribute 0.
        const int out_p = cq.p - RT;            // output frame (relative) completed now
        const bool emit = out_p >= cq.ta;       // the ring holds 2RT+1 planes of this segment
        float z[F][QY];
#pragma unroll
        for (int f = 0; f < F; ++f) {
            float yv[QY];
            if (valid) {
                const float* src = xbuf + f * XB + (grp * QY) * TXP + col;
                float v[QY + 2 * R];
#pragma unroll
                for (int j = 0; j < QY + 2 * R; ++j) v[j] = src[j * TXP];
#pragma unroll
                for (int q = 0; q < QY; ++q) {
                    float acc = xmul(a.taps_y[0], v[q]);
#pragma unroll
                    for (int d = 1; d <= 2 * R; ++d) acc = xadd(acc, xmul(a.taps_y[d], v[q + d]));
                    yv[q] = acc;
                }
            } else {
#pragma unroll
                for (int q = 0; q < QY; ++q) yv[q] = 0.0f;
            }
            // t-pass out of the register ring (conv3d.cpp:147-165): planes
            // oldest..newest take taps_t[0..2RT]; first = w*in, then +=.
            // A switch on the slot keeps every ring index static (registers).
            switch (slot) {
#define SFK_RING_CASE(S_)                                                          \
    case S_:                                                                       \
        if constexpr (S_ < K) {                                                    \
            _Pragma("unroll") for (int q = 0; q < QY; ++q) {                       \
                ring[f][q][S_] = yv[q];                                            \
                float acc = xmul(a.taps_t[0], ring[f][q][(S_ + 1) % K]);           \
                _Pragma("unroll") for (int d = 1; d < K; ++d) acc =                \
                    xadd(acc, xmul(a.taps_t[d], ring[f][q][(S_ + 1 + d) % K]));    \
                z[f][q] = acc;                                                     \
            }                                                                      \
        }                                                                          \
        break;
                SFK_RING_CASE(0)
                SFK_RING_CASE(1)
                SFK_RING_CASE(2)
                SFK_RING_CASE(3)
                SFK_RING_CASE(4)
                SFK_RING_CASE(5)
                SFK_RING_CASE(6)
                SFK_RING_CASE(7)
                SFK_RING_CASE(8)
#undef SFK_RING_CASE
                default:
                    break;
            }
        }
        slot = (slot + 1 == K) ? 0 : slot + 1;

        // (5) recombination, channel sum, store, reductions
        if (emit) {
            const int to = a.out_t0 + out_p;  // global output frame
            const int y0 = tile_y * TY + grp * QY;
            const int x = tile_x * TX + col;
            const bool xin = x < a.W;
            double colsum = 0.0;
            float cmax = 0.0f;
            const size_t in_plane = static_cast<size_t>(to - a.buf_t0) * a.H * a.pitch;
            const size_t out_plane = static_cast<size_t>(to - a.out_buf_t0) * a.H * a.pitch;
#pragma unroll
            for (int q = 0; q < QY; ++q) {
                const int y = y0 + q;
                float v = 0.0f;
                if (xin && y < a.H) {
                    const size_t ii = in_plane + static_cast<size_t>(y) * a.pitch + x;
                    const size_t oi = out_plane + static_cast<size_t>(y) * a.pitch + x;
                    const float spv = __ldg(a.sp + ii);
                    float acc = 0.0f;
#pragma unroll
                    for (int c = 0; c < CG; ++c) {
                        // engine.cpp:116-117:
                        // S^p * ((alpha^-1 - f f) * A - B + 2 f * C)
                        const float fv = __ldg(a.f[c] + ii);
                        const float t1 = xmul(xsub(inv_alpha, xmul(fv, fv)), z[0][q]);
                        const float t2 = xsub(t1, z[2 + 2 * c][q]);
                        const float t3 = xadd(t2, xmul(xmul(2.0f, fv), z[1 + 2 * c][q]));
                        const float term = xmul(spv, t3);
                        if (c == 0)
                            acc = a.first_group ? term : xadd(a.out[oi], term);
                        else
                            acc = xadd(acc, term);  // engine.cpp:157-162 / 317-319
                    }
                    a.out[oi] = acc;
                    v = acc;
                }
                if (a.last_group) {
                    colsum += static_cast<double>(v) * static_cast<double>(v);
                    cmax = fmaxf(cmax, v);
                    if ((q & 3) == 3) {  // close a 4-row canonical band
                        const double bsum = butterfly_sum32(colsum);
                        const int band = (y0 + q - 3) >> 2;
                        const int half = (tile_x * TX + (col & ~31)) >> 5;
                        if ((tid & 31) == 0 && band < a.nbands && half < a.nhalves) {
                            a.part[(static_cast<size_t>(to) * a.nbands + band) * a.nhalves +
                                   half] = bsum;
                        }
                        colsum = 0.0;
                    }
                }
            }
            if (a.last_group) {
                cmax = butterfly_max32(cmax);
                if ((tid & 31) == 0) atomic_max_nonneg(a.frame_max + to, cmax);
            }
        }
        cq.next();
    }
}

}  // namespace sfk
