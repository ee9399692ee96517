// fused_ws.cuh — warp-specialised SFSeg power-iteration step for sm_100a.
//
// One kernel per iteration does what the reference spends three
// convolve_separable calls per channel on (conv3d.cpp:80-185), plus the
// products (engine.cpp:92-100), recombination and channel sum
// (engine.cpp:107-120, 157-162) and the sum-of-squares / max scans of
// normalize_l2 / project_binary (engine.cpp:168-205). The previous
// iteration's normalisation and sigmoid are applied on load.
//
// Roles inside a CTA (NWA + 8 warps, one CTA per SM, persistent over the host
// schedule of (tile, frame-range) segments; a tile is 64 x 32 points):
//   A  = the first NWA warps: thread 0 issues the TMA loads of the
//        (64+2R) x BW halo boxes of y_k, S^p, F_c; all A warps form the
//        product fields (u = S^p x scalar; (F_c u, F_c^2 u) interleaved
//        pairs) and run the x-pass into a double-buffered shared tile.
//   B  = the last 8 warps: each thread owns 4 rows x 2 columns;
//        it runs the y-pass of those 8 points into a register ring holding
//        the last 2RT+1 y-filtered planes, the t-pass out of the ring, the
//        recombination, the store, and the canonical reductions.
// A and B meet only at two mbarrier pairs per x-pass buffer (full/empty),
// so the x-pass of plane p+1 overlaps the y/t/epilogue of plane p; A gives
// registers to B with setmaxnreg (B holds 120 ring registers).
//
// Packed arithmetic: two values that take the same tap (two columns of u, or
// F_c u and F_c^2 u of one column) run as one FFMA2. EXACT keeps the
// reference's rounding (product, then sum: two FFMA2 with runtime one/zero);
// FAST fuses them.
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "step_common.cuh"  // PlaneStream, Arith, ffma2, canonical_tree32
#include "sfseg_types.cuh"

// ablation builds (tools/ablate.sh): bit 0 drops A's arithmetic, bit 1 B's;
// the pipeline (TMA, barriers, stores) still runs. Never set in the product.
#ifndef SFK_EXP
#define SFK_EXP 0
#endif
// SFK_TMR=1: the t-pass ring of y-filtered planes lives in tensor memory
// instead of B's registers
#ifndef SFK_TMR
#define SFK_TMR 0
#endif

// timeline instrumentation (tools/trace_kernel.py; debug builds only):
// clock64 at pipeline events of CTAs 0..3, planes 0..127
#ifdef SFK_TRACE
__device__ unsigned long long sfk_trace[4][128][16];
#define SFK_T(pl, ev)                                                                   \
    do {                                                                               \
        if (blockIdx.x < 4 && (pl) < 128) sfk_trace[blockIdx.x][(pl)][(ev)] = clock64(); \
    } while (0)
#else
#define SFK_T(pl, ev) \
    do {              \
    } while (0)
#endif

namespace sfk {

template <int RT, int R, int CG, int STAGES, int NWA = 8>
struct WsGeom {
    static constexpr int TY = 64, TX = 32;
    static constexpr int NA = 32 * NWA, NB = 256, NT = NA + NB;
    // setmaxnreg budgets. Registers live in the 4 SMSP register files
    // (512 per lane slot each); warp w runs on SMSP w % 4, and the launch
    // grants every warp 512 / (most warps on one SMSP). Budgets must fit the
    // fullest SMSP, or setmaxnreg.inc waits forever.
    static constexpr int NWB = NB / 32;
    static constexpr int WMAX = (NT / 32 + 3) / 4;
    static constexpr int RPOOL = (512 / WMAX) / 8 * 8;
#ifndef SFK_RA
#define SFK_RA 56
#endif
    static constexpr int RA = NWA == 4 ? 80 : SFK_RA;
    static constexpr int RB_SMSP = (512 - (NWA + 3) / 4 * RA) / ((NWB + 3) / 4);
    static constexpr int RB_POOL = (NT * RPOOL - NA * RA) / NB;
    static constexpr int RB_MIN = RB_SMSP < RB_POOL ? RB_SMSP : RB_POOL;
    static constexpr int RB = (RB_MIN < 248 ? RB_MIN : 248) / 8 * 8;
    static constexpr int K = 2 * RT + 1;
    static constexpr int NIN = 2 + CG;
    static constexpr int BH = TY + 2 * R;
    static constexpr int RX4 = (R + 3) / 4 * 4;
    static constexpr int XOFF = RX4 - R;
    static constexpr int BW = TX + 2 * RX4;
    static constexpr int BW4 = BW / 4;
    static constexpr int FB = (BH * BW + 31) / 32 * 32;
    static constexpr int BWU = BW + 4, BWP = 2 * BW + 4;  // odd float4 row strides
    static constexpr int PBU = (BH * BWU + 31) / 32 * 32;
    static constexpr int PBP = (BH * BWP + 31) / 32 * 32;
    static constexpr int TXU = TX + 4, TXQ = 2 * TX + 4;
    static constexpr int XBU = (BH * TXU + 31) / 32 * 32;
    static constexpr int XBP = (BH * TXQ + 31) / 32 * 32;
    static constexpr int XBUF = XBU + CG * XBP;  // one x-pass buffer
    // x-pass work split: the first NWU A warps take u strips of SU outputs
    // (scalar FFMA), the others pair strips of SPP outputs (FFMA2, twice the
    // FMA-pipe cycles per item: NWU : NWA - NWU = 3 : 5 balances them). A
    // warp pass covers 8 consecutive rows x 4 strips; wide strips cut the
    // shared-memory reads per output to (SU + 2R) / SU.
    static constexpr int SU = 8, SPP = 8;
    static constexpr int NSU = TX / SU, NSP = TX / SPP;
    static constexpr int NINU = SU + 2 * R, NINP = SPP + 2 * R;
    static constexpr int RBLK = (BH + 7) / 8;
    static constexpr int UBLK = RBLK * (NSU / 4), PBLK = RBLK * (NSP / 4);
    static constexpr int NWU = NWA == 8 ? 3 : NWA / 2;
    static constexpr int UPASS = (UBLK + NWU - 1) / NWU, PPASSX = (PBLK + (NWA - NWU) - 1) / (NWA - NWU);
    static constexpr int NBANDS = TY / 4;
    // products: thread -> (row lane, float4 column); NPR rows per pass
    static constexpr int NPR = NA / BW4, PPASS = (BH + NPR - 1) / NPR;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
    // (SFK_EXP bit 3, skeleton ablations only: no product / x-pass storage)
    static constexpr size_t PROD_FLOATS = (SFK_EXP & 8) ? 32 : size_t(PBU) + size_t(CG) * PBP;
    static constexpr size_t XB_FLOATS = (SFK_EXP & 8) ? 64 : 2 * size_t(XBUF);
    // per B warp, double-buffered: S^p and F_c of its 8 output rows, TMA-loaded
    // a plane ahead; the S^p slab is overwritten with y_{k+1} and TMA-stored
    static constexpr int SLAB = 8 * TX;
    static constexpr int NSF = 1 + CG;  // slab fields: S^p, F_c...
    static constexpr size_t IN_FLOATS = size_t(NB / 32) * 2 * NSF * SLAB;
    static constexpr size_t SMEM_BYTES =
        (RAW_FLOATS + PROD_FLOATS + XB_FLOATS + IN_FLOATS) * sizeof(float) + 256;
    static_assert(NSU % 4 == 0 && NSP % 4 == 0, "x-pass passes: 4 strips x 8 rows");
    static_assert(NB == 16 * NBANDS, "B threads: 16 column pairs x 16 bands");
    static_assert(CG == 1 || true, "pair strips are split over the second half of A");
    static_assert(NA * RA + NB * RB <= NT * RPOOL, "register pool of the CTA");
    static_assert((NWA + 3) / 4 * RA + (NWB + 3) / 4 * RB <= 512, "register file of one SMSP");
    static_assert(RB <= 248, "setmaxnreg range");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert((BWU / 4) % 2 == 1 && (BWP / 4) % 2 == 1, "conflict-free product rows");
    static_assert((TXU / 4) % 2 == 1 && (TXQ / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// ACC: a later channel group, y_{k+1} += this group's terms (engine.cpp:157-162)
template <int RT, int R, int CG, int STAGES, bool FMA, int NWA = 8, bool ACC = false>
__global__ void __launch_bounds__(32 * NWA + 256, 1) fused_step_ws(const __grid_constant__ FusedArgs a) {
    using G = WsGeom<RT, R, CG, STAGES, NWA>;
    using A = Arith<FMA>;
    constexpr int TY = G::TY, TX = G::TX, NA = G::NA, NB = G::NB, K = G::K;
    constexpr int NIN = G::NIN, BH = G::BH, BW = G::BW, FB = G::FB, BW4 = G::BW4;
    constexpr int BWU = G::BWU, BWP = G::BWP, PBU = G::PBU, PBP = G::PBP;
    constexpr int TXU = G::TXU, TXQ = G::TXQ, XBU = G::XBU, XBP = G::XBP, XBUF = G::XBUF;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                      // [STAGES][NIN][FB]   TMA boxes
    float* produ = raw + G::RAW_FLOATS;     // [BH][BWU]           u
    float* prodp = produ + PBU;             // [CG][BH][BWP]       (F u, F^2 u)
    float* xb = produ + G::PROD_FLOATS;     // [2][XBUF]           x-pass output
    float* bslab = xb + G::XB_FLOATS;       // [NB/32][2][1+CG][8][TX] recombination slabs
    uint64_t* mbar = reinterpret_cast<uint64_t*>(bslab + G::IN_FLOATS);
    uint64_t* raw_full = mbar;             // [STAGES]  TMA -> A
    uint64_t* xb_full = mbar + STAGES;     // [2]       A -> B (count NA)
    uint64_t* xb_empty = mbar + STAGES + 2;  // [2]     B -> A (count NB)
    uint64_t* slab_full = mbar + STAGES + 4;  // [NB/32][2] TMA -> B warp

    __shared__ IterState st;
    __shared__ PlaneStream prodq;
    __shared__ PlaneStream slabq[NB / 32];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int prod_count;

    const int tid = threadIdx.x;
    griddep_wait();  // PDL: the previous step / finalize has completed
    if (a.st->degenerate && SFK_EXP == 0) return;  // an earlier iteration hit a zero norm
    const int s0 = a.sched_off[blockIdx.x], s1 = a.sched_off[blockIdx.x + 1];
    if (s0 >= s1) return;

    if (tid == 0) {
        st = *a.st;
        for (int s = 0; s < STAGES; ++s) mbar_init(&raw_full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xb_full[b], NA);
            mbar_init(&xb_empty[b], NB);
        }
        for (int w = 0; w < 2 * (NB / 32); ++w) mbar_init(&slab_full[w], 1);
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        prefetch_tensormap(&a.tm_sp);
        for (int c = 0; c < CG; ++c) prefetch_tensormap(&a.tm_f[c]);
        prefetch_tensormap(&a.tm_out);
        prefetch_tensormap(&a.tm_spc);
        for (int c = 0; c < CG; ++c) prefetch_tensormap(&a.tm_fc[c]);
    }
    __syncthreads();

    const float2 one2 = make_float2(a.one, a.one), zero2 = make_float2(a.zero, a.zero);

    if (tid < NA) {
        // =====================================================================
        // A: TMA producer + products + x-pass
        // =====================================================================
        setmaxnreg_dec<G::RA>();
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
            uint64_t* bar = &raw_full[s];
            mbar_arrive_expect_tx(bar, NIN * BH * BW * sizeof(float));
            const int bx = prodq.tile_x * TX - G::RX4, by = prodq.tile_y * TY - R,
                      bt = tg - a.buf_t0;
            tma_load_3d(dst, &a.tm_x, bar, bx, by, bt);
            tma_load_3d(dst + FB, &a.tm_sp, bar, bx, by, bt);
#pragma unroll
            for (int c = 0; c < CG; ++c)
                tma_load_3d(dst + (2 + c) * FB, &a.tm_f[c], bar, bx, by, bt);
            ++prod_count;
            prodq.next();
        };
        if (tid == 0) {
            prodq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            prod_count = 0;
            for (int s = 0; s < STAGES; ++s) issue_next();
        }
        const bool sigm = st.mode == 2;
        const double inv = st.mode == 0 ? 1.0 : st.inv;  // float(double(y)*1.0) == y
        const float inv_f = st.mode == 0 ? 1.0f : st.inv_f;

        const int pr0 = tid / BW4, pc4 = tid - (tid / BW4) * BW4;
        const bool pact = tid < G::NPR * BW4;
        const int xw = tid >> 5, xl = tid & 31;  // x-pass: warp, lane (row xl & 7, strip xl >> 3)

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;  // in-volume planes handled
        for (; !q.done; q.next()) {
            const int tg = a.out_t0 + q.p;
            if (tg < 0 || tg >= a.T) continue;  // planes outside the volume: B zero-fills
            const int s = cnt % STAGES;
            if (tid == 32) SFK_T(cnt, 0);
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            if (tid == 32) SFK_T(cnt, 1);
            const float* rs = raw + static_cast<size_t>(s) * NIN * FB;
            // products over the halo box (engine.cpp:92-100): thread -> (row
            // lane pr0, float4 column pc4), rows pr0, pr0 + NPR, ... (constant
            // offsets, no index arithmetic in the loop)
            if (pact && !(SFK_EXP & 1)) {
                const float4* rx = reinterpret_cast<const float4*>(rs) + pr0 * BW4 + pc4;
                float* du = produ + pr0 * BWU + 4 * pc4;
                float* dp = prodp + pr0 * BWP + 8 * pc4;
                // EXACT's double-precision load_norm needs more registers than
                // A's budget allows for an unrolled loop
                constexpr int PU = FMA ? G::PPASS : 1;
#pragma unroll PU
                for (int k = 0; k < G::PPASS; ++k) {
                    if (k == G::PPASS - 1 && pr0 + k * G::NPR >= BH) break;
                    const int i = k * G::NPR * BW4;
                    const float4 yv = rx[i];
                    const float4 sv = rx[FB / 4 + i];
                    // EXACT: the F load goes out with the others (2% faster);
                    // FAST: issuing all of them up front floods the shared-
                    // memory queue the B warps' y-pass shares (measured 40%
                    // slower), so F is loaded where it is used
                    float4 fpre = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    if constexpr (!FMA) fpre = rx[2 * (FB / 4) + i];
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
                    *reinterpret_cast<float4*>(du + k * G::NPR * BWU) = u;
#pragma unroll
                    for (int cg = 0; cg < CG; ++cg) {
                        const float4 fv = (!FMA && cg == 0) ? fpre : rx[(2 + cg) * (FB / 4) + i];
                        float4 p0, p1;  // (F S^p X, (F F) S^p X) per point
                        p0.x = A::mul(fv.x, u.x);
                        p0.z = A::mul(fv.y, u.y);
                        p1.x = A::mul(fv.z, u.z);
                        p1.z = A::mul(fv.w, u.w);
                        if constexpr (FMA) {  // FAST: F (F u), one product less
                            p0.y = fv.x * p0.x;
                            p0.w = fv.y * p0.z;
                            p1.y = fv.z * p1.x;
                            p1.w = fv.w * p1.z;
                        } else {  // engine.cpp:98: fi * fi * sx
                            p0.y = A::mul(A::mul(fv.x, fv.x), u.x);
                            p0.w = A::mul(A::mul(fv.y, fv.y), u.y);
                            p1.y = A::mul(A::mul(fv.z, fv.z), u.z);
                            p1.w = A::mul(A::mul(fv.w, fv.w), u.w);
                        }
                        float4* pp = reinterpret_cast<float4*>(dp + cg * PBP + k * G::NPR * BWP);
                        pp[0] = p0;
                        pp[1] = p1;
                    }
                }
            }
            named_bar_sync(1, NA);  // products ready; raw stage s fully read
            if (tid == 32) SFK_T(cnt, 2);
            if (tid == 0) {
                fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_next();
            }
            // x-pass (conv3d.cpp:88-101) into the free x buffer
            const int b = cnt & 1;
            mbar_wait(&xb_empty[b], ((cnt >> 1) & 1) ^ 1);
            if (tid == 32) SFK_T(cnt, 3);
            float* xbu = xb + b * XBUF;
            float* xbp = xbu + XBU;
            if (SFK_EXP & 1) {
            } else if (xw < G::NWU) {
                // u strips: pass k covers row block / strip group blk
#pragma unroll
                for (int k = 0; k < G::UPASS; ++k) {
                    const int blk = xw + k * G::NWU;
                    if (blk >= G::UBLK) break;
                    const int r = (blk / (G::NSU / 4)) * 8 + (xl & 7);
                    const int st = (blk % (G::NSU / 4)) * 4 + (xl >> 3);
                    if (r >= BH) continue;
                    const float4* src = reinterpret_cast<const float4*>(produ + r * BWU + st * G::SU);
                    float o[G::SU];
                    float4 q4;
#pragma unroll
                    for (int m4 = 0; m4 < (G::XOFF + G::NINU + 3) / 4 * 4; ++m4) {
                        if (m4 % 4 == 0) q4 = src[m4 / 4];
                        const int m = m4 - G::XOFF;
                        if (m < 0 || m >= G::NINU) continue;
                        const float vin = (m4 % 4 == 0) ? q4.x : (m4 % 4 == 1) ? q4.y
                                        : (m4 % 4 == 2) ? q4.z : q4.w;
#pragma unroll
                        for (int j = 0; j < G::SU; ++j) {
                            const int d = m - j;
                            if (d < 0 || d > 2 * R) continue;
                            o[j] = d == 0 ? A::mul(a.taps_x[0], vin) : A::mac(o[j], a.taps_x[d], vin);
                        }
                    }
                    float4* dst = reinterpret_cast<float4*>(xbu + r * TXU + st * G::SU);
#pragma unroll
                    for (int v = 0; v < G::SU / 4; ++v)
                        dst[v] = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
                }
            } else {
                const int wp = xw - G::NWU;
#pragma unroll
                for (int k = 0; k < G::PPASSX; ++k) {
                    const int blk = wp + k * (NA / 32 - G::NWU);
                    if (blk >= G::PBLK) break;
                    const int r = (blk / (G::NSP / 4)) * 8 + (xl & 7);
                    const int st = (blk % (G::NSP / 4)) * 4 + (xl >> 3);
                    if (r >= BH) continue;
#pragma unroll
                    for (int c = 0; c < CG; ++c) {
                        const float4* src =
                            reinterpret_cast<const float4*>(prodp + c * PBP + r * BWP + 2 * st * G::SPP);
                        float2 o[G::SPP];
                        float4 q4;
#pragma unroll
                        for (int m2 = 0; m2 < (G::XOFF + G::NINP + 1) / 2 * 2; ++m2) {
                            if (m2 % 2 == 0) q4 = src[m2 / 2];
                            const int m = m2 - G::XOFF;
                            if (m < 0 || m >= G::NINP) continue;
                            const float2 vin = (m2 % 2 == 0) ? make_float2(q4.x, q4.y)
                                                             : make_float2(q4.z, q4.w);
#pragma unroll
                            for (int j = 0; j < G::SPP; ++j) {
                                const int d = m - j;
                                if (d < 0 || d > 2 * R) continue;
                                o[j] = d == 0 ? A::mul2(a.taps_x[0], vin, zero2)
                                              : A::mac2(o[j], a.taps_x[d], vin, one2, zero2);
                            }
                        }
                        // float2 stores straight from the FFMA2 register pairs
                        float2* dst = reinterpret_cast<float2*>(xbp + c * XBP + r * TXQ + 2 * st * G::SPP);
#pragma unroll
                        for (int j = 0; j < G::SPP; ++j) dst[j] = o[j];
                    }
                }
            }
            if (tid == 32) SFK_T(cnt, 4);
            mbar_arrive(&xb_full[b]);  // release: this thread's x-pass stores
            named_bar_sync(1, NA);     // every A thread is done with the products
            if (tid == 32) SFK_T(cnt, 5);
            ++cnt;
        }
    } else {
        // =====================================================================
        // B: y-pass ring, t-pass, recombination, store, reductions
        // =====================================================================
        // B layout: FAST (B81) gives each thread 8 rows x 1 column (8 + 2R
        // shared-memory rows read per 8 outputs); EXACT keeps 4 rows x 2
        // columns so the u field runs as column-pair FFMA2 (its separately
        // rounded products and sums would double the scalar issue count)
        constexpr bool B81 = FMA;
        if constexpr (B81) {
            setmaxnreg_inc<G::RB>();
            const int bt = tid - NA;
            // B thread = one column (its lane) x 8 rows (8 wb .. 8 wb + 7) of the
            // tile: the y-pass reads 8 + 2R rows for 8 outputs
            const int lane = bt & 31;
            const int wb = bt >> 5;
            const float inv_alpha = a.inv_alpha;
            const bool last = a.last_group;

            constexpr bool TMR = SFK_TMR != 0;
            constexpr int KR = TMR ? 1 : K;  // register ring depth
            float ringu[8][KR];           // u
            float2 ringp[CG][8][KR];      // (F u, F^2 u)
    #pragma unroll
            for (int r = 0; r < 8; ++r)
    #pragma unroll
                for (int k = 0; k < KR; ++k) {
                    ringu[r][k] = 0.0f;
    #pragma unroll
                    for (int c = 0; c < CG; ++c) ringp[c][r][k] = make_float2(0.0f, 0.0f);
                }
            // TMEM ring (TMR): each B thread keeps K slots of RW = 8 + 16 CG words
            // in its TMEM lane; warps w and w+4 share a lane quadrant and split the
            // columns into two halves of 128
            constexpr int RW = 8 + 16 * CG;
            static_assert(!TMR || K * RW <= 128, "TMEM ring of one thread");
            uint32_t tm_ring = 0;
            if constexpr (TMR) {
                if (bt < 32) tmem_alloc<256>(&tmem_base_sh);
                tcgen05_fence_before();
                named_bar_sync(3, NB);
                tcgen05_fence_after();
                const int wq = (NA / 32 + wb) & 3;  // CTA warp id % 4
                tm_ring = tmem_base_sh + (static_cast<uint32_t>(32 * wq) << 16) + static_cast<uint32_t>((wb >> 2) * 128);
            }

            PlaneStream q;
            q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            int cnt = 0;   // in-volume planes consumed
            int ecnt = 0;  // output planes emitted
            // This warp's 8 output rows: S^p / F_c slabs come in by TMA a plane
            // ahead into alternating buffers (cursor eq walks the emitted planes in
            // schedule order); y_{k+1} overwrites the consumed S^p slab and leaves
            // by TMA store. No CTA-wide barrier in B, and no edge masks: the TMA
            // zero-fills S^p outside the volume, so those points come out as
            // exactly 0 and add nothing to the sums, and the store clips them.
            float* myslab = bslab + wb * 2 * G::NSF * G::SLAB;
            PlaneStream& eq = slabq[wb];  // lane 0 only (kept in shared memory: B is register-bound)
            int eissued = 0;              // lane 0: slabs issued so far
            auto issue_slab = [&]() {
                if (eq.done) return;
                const int sb = eissued & 1;
                float* dst = myslab + sb * G::NSF * G::SLAB;
                uint64_t* bar = &slab_full[2 * wb + sb];
                const int x = eq.tile_x * TX, y = eq.tile_y * TY + 8 * wb, t = a.out_t0 + eq.p - a.buf_t0;
                mbar_arrive_expect_tx(bar, G::NSF * G::SLAB * sizeof(float));
                tma_load_3d(dst, &a.tm_spc, bar, x, y, t);
    #pragma unroll
                for (int c = 0; c < CG; ++c) tma_load_3d(dst + (1 + c) * G::SLAB, &a.tm_fc[c], bar, x, y, t);
                eq.next();
                ++eissued;
            };
            if (lane == 0 && !(SFK_EXP & 4)) {
                eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
                issue_slab();
            }

            // one plane with ring slot S_; the caller unrolls K planes so every
            // ring index is a compile-time constant (no rotation moves)
            auto plane = [&](auto slot_c) {
                constexpr int S_ = decltype(slot_c)::value;
                constexpr int SR = TMR ? 0 : S_;  // register slot of this plane
                const int tg = a.out_t0 + q.p;
                const bool valid = tg >= 0 && tg < a.T;
                const bool emit = q.p - RT >= q.ta;
                const int to = tg - RT;

                // y-pass (conv3d.cpp:113-135): first = w * in, then += (d ascending),
                // accumulated straight into this plane's ring slot
                if (valid) {
                    const int b = cnt & 1;
                    if (bt == 0) SFK_T(cnt, 6);
                    mbar_wait(&xb_full[b], (cnt >> 1) & 1);
                    if (bt == 0) SFK_T(cnt, 7);
                    const float* xbu = xb + b * XBUF + (8 * wb) * TXU + lane;
                    const float2* xbp = reinterpret_cast<const float2*>(xb + b * XBUF + XBU + (8 * wb) * TXQ) + lane;
    #pragma unroll
                    for (int j = 0; j < ((SFK_EXP & 2) ? 0 : 8 + 2 * R); ++j) {
                        const float vin = xbu[j * TXU];
    #pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int d = j - r;
                            if (d < 0 || d > 2 * R) continue;
                            ringu[r][SR] = d == 0 ? A::mul(a.taps_y[0], vin) : A::mac(ringu[r][SR], a.taps_y[d], vin);
                        }
    #pragma unroll
                        for (int c = 0; c < CG; ++c) {
                            const float2 pv = xbp[c * (XBP / 2) + j * (TXQ / 2)];
    #pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                const int d = j - r;
                                if (d < 0 || d > 2 * R) continue;
                                ringp[c][r][SR] = d == 0 ? A::mul2(a.taps_y[0], pv, zero2)
                                                         : A::mac2(ringp[c][r][SR], a.taps_y[d], pv, one2, zero2);
                            }
                        }
                    }
                    if (bt == 0) SFK_T(cnt, 8);
                    mbar_arrive(&xb_empty[b]);
                    ++cnt;
                } else {
    #pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        ringu[r][SR] = 0.0f;
    #pragma unroll
                        for (int c = 0; c < CG; ++c) ringp[c][r][SR] = make_float2(0.0f, 0.0f);
                    }
                }
                if constexpr (TMR) {
                    // this plane's slot: u (8 words), then (F u, F^2 u) per channel
                    // (16 words); the slot it replaces held a plane no longer needed
                    float w8[8];
    #pragma unroll
                    for (int r = 0; r < 8; ++r) w8[r] = ringu[r][0];
                    tmem_st8(tm_ring + S_ * RW, w8);
    #pragma unroll
                    for (int c = 0; c < CG; ++c)
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
    #pragma unroll
                            for (int rr = 0; rr < 4; ++rr) {
                                w8[2 * rr] = ringp[c][4 * h + rr][0].x;
                                w8[2 * rr + 1] = ringp[c][4 * h + rr][0].y;
                            }
                            tmem_st8(tm_ring + S_ * RW + 8 + 16 * c + 8 * h, w8);
                        }
                }
                if (emit && !(SFK_EXP & 4)) {
                    if (lane == 0) {
                        // slab buffer of plane ecnt+1 = the one stored from at ecnt-1:
                        // once that store has read it, fetch the next operands
                        bulk_wait_read0();
                        issue_slab();
                    }
                    const int sb = ecnt & 1;
                    float* sl = myslab + sb * G::NSF * G::SLAB + lane;
                    if (bt == 0) SFK_T(ecnt, 9);
                    mbar_wait(&slab_full[2 * wb + sb], (ecnt >> 1) & 1);
                    if (bt == 0) SFK_T(ecnt, 10);
                    // t-pass (conv3d.cpp:147-165): planes oldest..newest take
                    // taps_t[0..2RT]; first = w * in, then +=
                    float tu[8];
                    float2 tp[CG][8];
                    if constexpr (TMR) {
                        tmem_wait_st();
    #pragma unroll
                        for (int d = 0; d < K; ++d) {
                            const int sl2 = (S_ + 1 + d) % K;
                            float lu[8];
                            float2 lp[CG][8];
                            if (sl2 == S_) {
    #pragma unroll
                                for (int r = 0; r < 8; ++r) {
                                    lu[r] = ringu[r][0];
    #pragma unroll
                                    for (int c = 0; c < CG; ++c) lp[c][r] = ringp[c][r][0];
                                }
                            } else {
                                float w8[1 + 2 * CG][8];
                                tmem_ld8(tm_ring + sl2 * RW, w8[0]);
    #pragma unroll
                                for (int c = 0; c < CG; ++c) {
                                    tmem_ld8(tm_ring + sl2 * RW + 8 + 16 * c, w8[1 + 2 * c]);
                                    tmem_ld8(tm_ring + sl2 * RW + 16 + 16 * c, w8[2 + 2 * c]);
                                }
                                tmem_wait_ld();
    #pragma unroll
                                for (int r = 0; r < 8; ++r) {
                                    lu[r] = w8[0][r];
    #pragma unroll
                                    for (int c = 0; c < CG; ++c)
                                        lp[c][r] = make_float2(w8[1 + 2 * c + (r >> 2)][2 * (r & 3)],
                                                               w8[1 + 2 * c + (r >> 2)][2 * (r & 3) + 1]);
                                }
                            }
    #pragma unroll
                            for (int r = 0; r < 8; ++r) {
                                tu[r] = d == 0 ? A::mul(a.taps_t[0], lu[r]) : A::mac(tu[r], a.taps_t[d], lu[r]);
    #pragma unroll
                                for (int c = 0; c < CG; ++c)
                                    tp[c][r] = d == 0 ? A::mul2(a.taps_t[0], lp[c][r], zero2)
                                                      : A::mac2(tp[c][r], a.taps_t[d], lp[c][r], one2, zero2);
                            }
                        }
                    } else {
    #pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            tu[r] = A::mul(a.taps_t[0], ringu[r][(S_ + 1) % KR]);
    #pragma unroll
                            for (int d = 1; d < K; ++d) tu[r] = A::mac(tu[r], a.taps_t[d], ringu[r][(S_ + 1 + d) % KR]);
    #pragma unroll
                            for (int c = 0; c < CG; ++c) {
                                tp[c][r] = A::mul2(a.taps_t[0], ringp[c][r][(S_ + 1) % KR], zero2);
    #pragma unroll
                                for (int d = 1; d < K; ++d)
                                    tp[c][r] = A::mac2(tp[c][r], a.taps_t[d], ringp[c][r][(S_ + 1 + d) % KR], one2, zero2);
                            }
                        }
                    }
                    float v[8];
    #pragma unroll
                    for (int r = 0; r < ((SFK_EXP & 18) ? 0 : 8); ++r) {
                        const float spv = sl[r * TX];
                        float prev = 0.0f;
                        if constexpr (ACC) {  // y so far (earlier groups); 0 outside the volume
                            const int y = q.tile_y * TY + 8 * wb + r, x = q.tile_x * TX + lane;
                            if (y < a.H && x < a.W)
                                prev = a.out[static_cast<long long>(to - a.out_buf_t0) * a.H * a.pitch +
                                             static_cast<long long>(y) * a.pitch + x];
                        }
    #pragma unroll
                        for (int c = 0; c < CG; ++c) {
                            const float fv = sl[(1 + c) * G::SLAB + r * TX];
                            // engine.cpp:113-119, channel sum engine.cpp:157-162
                            const float term = A::recombine(spv, fv, inv_alpha, tu[r], tp[c][r].y, tp[c][r].x);
                            v[r] = c > 0 ? xadd(v[r], term) : (ACC ? xadd(prev, term) : term);
                        }
                        sl[r * TX] = v[r];  // each thread overwrites exactly the S^p value it read
                    }
                    // hand the slab to the TMA unit (generic-proxy writes -> async
                    // proxy; clipped at the volume edge)
                    if (!(SFK_EXP & 32)) fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&a.tm_out, myslab + sb * G::NSF * G::SLAB, q.tile_x * TX,
                                     q.tile_y * TY + 8 * wb, to - a.out_buf_t0);
                        bulk_commit();
                    }
                    if (bt == 0) SFK_T(ecnt, 11);
                    if (bt == 224) SFK_T(ecnt, 12);
                    ++ecnt;
                    if (last && !(SFK_EXP & (18 | 64))) {
                        // canonical reduction (device_common.cuh): the warp holds
                        // two blocks (rows 0-3 and 4-7 of its 8 rows) x 32 columns,
                        // one column per lane: the column sum over the 4 rows runs in
                        // the lane, then the 32-column butterfly (16, 8, 4, 2, 1).
                        // EXACT sums in fp64; FAST in fp32 within a block.
                        double sum[2];
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if constexpr (FMA) {
                                float cs = 0.0f;
    #pragma unroll
                                for (int r = 0; r < 4; ++r) cs = fmaf(v[4 * h + r], v[4 * h + r], cs);
    #pragma unroll
                                for (int o = 16; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
                                sum[h] = static_cast<double>(cs);
                            } else {
                                double cs = 0.0;
    #pragma unroll
                                for (int r = 0; r < 4; ++r)
                                    cs += static_cast<double>(v[4 * h + r]) * static_cast<double>(v[4 * h + r]);
                                sum[h] = butterfly_sum32(cs);
                            }
                        }
                        float cmax = 0.0f;
    #pragma unroll
                        for (int r = 0; r < 8; ++r) cmax = fmaxf(cmax, v[r]);
                        const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                        const int gb = q.tile_y * G::NBANDS + 2 * wb;
                        if (lane < 2 && gb + lane < a.nbands && q.tile_x < a.nhalves)
                            a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb + lane) * a.nhalves +
                                   q.tile_x] = lane ? sum[1] : sum[0];
                        if (lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
                    }
                }
                q.next();
            };
            using std::integral_constant;
            while (!q.done) {
                plane(integral_constant<int, 0>{});
                if constexpr (K > 1) { if (q.done) break; plane(integral_constant<int, (K > 1 ? 1 : 0)>{}); }
                if constexpr (K > 2) { if (q.done) break; plane(integral_constant<int, (K > 2 ? 2 : 0)>{}); }
                if constexpr (K > 3) { if (q.done) break; plane(integral_constant<int, (K > 3 ? 3 : 0)>{}); }
                if constexpr (K > 4) { if (q.done) break; plane(integral_constant<int, (K > 4 ? 4 : 0)>{}); }
                if constexpr (K > 5) { if (q.done) break; plane(integral_constant<int, (K > 5 ? 5 : 0)>{}); }
                if constexpr (K > 6) { if (q.done) break; plane(integral_constant<int, (K > 6 ? 6 : 0)>{}); }
                if constexpr (K > 7) { if (q.done) break; plane(integral_constant<int, (K > 7 ? 7 : 0)>{}); }
                if constexpr (K > 8) { if (q.done) break; plane(integral_constant<int, (K > 8 ? 8 : 0)>{}); }
            }
        } else {
            setmaxnreg_inc<G::RB>();
            const int bt = tid - NA;
            const int band = bt >> 4;  // rows 4*band .. 4*band+3 of the tile
            const int cp = bt & 15;    // columns 2cp, 2cp+1
            const int lane = bt & 31;
            const float inv_alpha = a.inv_alpha;
            const bool last = a.last_group;

            constexpr bool TMR = SFK_TMR != 0;
            constexpr int KR = TMR ? 1 : K;  // register ring depth
            float2 ringu[4][KR];          // (col 2cp, col 2cp+1) of u
            float2 ringp[CG][4][2][KR];   // (F u, F^2 u) per column
    #pragma unroll
            for (int r = 0; r < 4; ++r)
    #pragma unroll
                for (int k = 0; k < KR; ++k) {
                    ringu[r][k] = make_float2(0.0f, 0.0f);
    #pragma unroll
                    for (int c = 0; c < CG; ++c) {
                        ringp[c][r][0][k] = make_float2(0.0f, 0.0f);
                        ringp[c][r][1][k] = make_float2(0.0f, 0.0f);
                    }
                }
            // TMEM ring (TMR): each B thread keeps K slots of RW = 8 + 16 CG words
            // in its TMEM lane; warps w and w+4 share a lane quadrant and split the
            // columns into two halves of 128
            constexpr int RW = 8 + 16 * CG;
            static_assert(!TMR || K * RW <= 128, "TMEM ring of one thread");
            uint32_t tm_ring = 0;
            if constexpr (TMR) {
                if (bt < 32) tmem_alloc<256>(&tmem_base_sh);
                tcgen05_fence_before();
                named_bar_sync(3, NB);
                tcgen05_fence_after();
                const int wq = (NA / 32 + (bt >> 5)) & 3;  // CTA warp id % 4
                tm_ring = tmem_base_sh + (static_cast<uint32_t>(32 * wq) << 16) + static_cast<uint32_t>(((bt >> 5) >> 2) * 128);
            }

            PlaneStream q;
            q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            int cnt = 0;   // in-volume planes consumed
            int ecnt = 0;  // output planes emitted
            // This warp's 8 output rows: S^p / F_c (/ y so far) slabs come in by
            // TMA a plane ahead into alternating buffers (cursor eq walks the
            // emitted planes in schedule order); y_{k+1} overwrites the consumed
            // S^p slab and leaves by TMA store. No CTA-wide barrier in B, and no
            // edge masks: the TMA zero-fills S^p outside the volume, so those
            // points come out as exactly 0 and add nothing to the sums, and the
            // store clips them.
            const int wb = bt >> 5;
            float* myslab = bslab + wb * 2 * G::NSF * G::SLAB;
            PlaneStream& eq = slabq[wb];  // lane 0 only (kept in shared memory: B is register-bound)
            int eissued = 0;              // lane 0: slabs issued so far
            auto issue_slab = [&]() {
                if (eq.done) return;
                const int sb = eissued & 1;
                float* dst = myslab + sb * G::NSF * G::SLAB;
                uint64_t* bar = &slab_full[2 * wb + sb];
                const int x = eq.tile_x * TX, y = eq.tile_y * TY + 8 * wb, t = a.out_t0 + eq.p - a.buf_t0;
                mbar_arrive_expect_tx(bar, G::NSF * G::SLAB * sizeof(float));
                tma_load_3d(dst, &a.tm_spc, bar, x, y, t);
    #pragma unroll
                for (int c = 0; c < CG; ++c) tma_load_3d(dst + (1 + c) * G::SLAB, &a.tm_fc[c], bar, x, y, t);
                eq.next();
                ++eissued;
            };
            if (lane == 0 && !(SFK_EXP & 4)) {
                eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
                issue_slab();
            }
            const int sloff = ((band & 1) * 4) * TX + 2 * cp;  // this thread's rows in a slab

            // one plane with ring slot S_; the caller unrolls K planes so every
            // ring index is a compile-time constant (no rotation moves)
            auto plane = [&](auto slot_c) {
                constexpr int S_ = decltype(slot_c)::value;
                constexpr int SR = TMR ? 0 : S_;  // register slot of this plane
                const int tg = a.out_t0 + q.p;
                const bool valid = tg >= 0 && tg < a.T;
                const bool emit = q.p - RT >= q.ta;
                const int to = tg - RT;

                // y-pass (conv3d.cpp:113-135): first = w * in, then += (d ascending),
                // accumulated straight into this plane's ring slot
                if (valid) {
                    const int b = cnt & 1;
                    if (bt == 0) SFK_T(cnt, 6);
                    mbar_wait(&xb_full[b], (cnt >> 1) & 1);
                    if (bt == 0) SFK_T(cnt, 7);
                    const float* xbu = xb + b * XBUF;
                    const float* xbp = xbu + XBU;
                    const float2* su = reinterpret_cast<const float2*>(xbu + (band * 4) * TXU) + cp;
    #pragma unroll
                    for (int j = 0; j < ((SFK_EXP & 2) ? 0 : 4 + 2 * R); ++j) {
                        const float2 vin = su[j * (TXU / 2)];
    #pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int d = j - r;
                            if (d < 0 || d > 2 * R) continue;
                            ringu[r][SR] = d == 0 ? A::mul2(a.taps_y[0], vin, zero2)
                                                  : A::mac2(ringu[r][SR], a.taps_y[d], vin, one2, zero2);
                        }
                    }
    #pragma unroll
                    for (int c = 0; c < ((SFK_EXP & 2) ? 0 : CG); ++c) {
                        const float4* sq =
                            reinterpret_cast<const float4*>(xbp + c * XBP + (band * 4) * TXQ) + cp;
    #pragma unroll
                        for (int j = 0; j < 4 + 2 * R; ++j) {
                            const float4 v4 = sq[j * (TXQ / 4)];
                            const float2 v0 = make_float2(v4.x, v4.y), v1 = make_float2(v4.z, v4.w);
    #pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const int d = j - r;
                                if (d < 0 || d > 2 * R) continue;
                                if (d == 0) {
                                    ringp[c][r][0][SR] = A::mul2(a.taps_y[0], v0, zero2);
                                    ringp[c][r][1][SR] = A::mul2(a.taps_y[0], v1, zero2);
                                } else {
                                    ringp[c][r][0][SR] =
                                        A::mac2(ringp[c][r][0][SR], a.taps_y[d], v0, one2, zero2);
                                    ringp[c][r][1][SR] =
                                        A::mac2(ringp[c][r][1][SR], a.taps_y[d], v1, one2, zero2);
                                }
                            }
                        }
                    }
                    if (bt == 0) SFK_T(cnt, 8);
                    mbar_arrive(&xb_empty[b]);
                    ++cnt;
                } else {
    #pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        ringu[r][SR] = make_float2(0.0f, 0.0f);
    #pragma unroll
                        for (int c = 0; c < CG; ++c)
                            ringp[c][r][0][SR] = ringp[c][r][1][SR] = make_float2(0.0f, 0.0f);
                    }
                }
                if constexpr (TMR) {
                    // this plane's slot: u (8 words), then (F u, F^2 u) per channel
                    // (16 words); the slot it replaces held a plane no longer needed
                    float w8[8];
    #pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        w8[2 * r] = ringu[r][0].x;
                        w8[2 * r + 1] = ringu[r][0].y;
                    }
                    tmem_st8(tm_ring + S_ * RW, w8);
    #pragma unroll
                    for (int c = 0; c < CG; ++c)
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
    #pragma unroll
                            for (int rr = 0; rr < 2; ++rr) {
                                const int r = 2 * h + rr;
                                w8[4 * rr] = ringp[c][r][0][0].x;
                                w8[4 * rr + 1] = ringp[c][r][0][0].y;
                                w8[4 * rr + 2] = ringp[c][r][1][0].x;
                                w8[4 * rr + 3] = ringp[c][r][1][0].y;
                            }
                            tmem_st8(tm_ring + S_ * RW + 8 + 16 * c + 8 * h, w8);
                        }
                }
                if (emit && !(SFK_EXP & 4)) {
                    if (lane == 0) {
                        // slab buffer of plane ecnt+1 = the one stored from at ecnt-1:
                        // once that store has read it, fetch the next operands
                        bulk_wait_read0();
                        issue_slab();
                    }
                    const int sb = ecnt & 1;
                    float* sl = myslab + sb * G::NSF * G::SLAB + sloff;
                    if (bt == 0) SFK_T(ecnt, 9);
                    mbar_wait(&slab_full[2 * wb + sb], (ecnt >> 1) & 1);
                    if (bt == 0) SFK_T(ecnt, 10);
                    float2 v2[4];
                    // TMR: t-pass (conv3d.cpp:147-165) over the TMEM slots, oldest
                    // first (taps_t[0..2RT], first = w * in, then +=); the newest
                    // plane is still in registers
                    float2 tu[4], tp[CG][4][2];
                    if constexpr (TMR) {
                        tmem_wait_st();
    #pragma unroll
                        for (int d = 0; d < K; ++d) {
                            const int sl = (S_ + 1 + d) % K;
                            float2 lu[4], lp[CG][4][2];
                            if (sl == S_) {
    #pragma unroll
                                for (int r = 0; r < 4; ++r) {
                                    lu[r] = ringu[r][0];
    #pragma unroll
                                    for (int c = 0; c < CG; ++c) {
                                        lp[c][r][0] = ringp[c][r][0][0];
                                        lp[c][r][1] = ringp[c][r][1][0];
                                    }
                                }
                            } else {
                                float w8[1 + 2 * CG][8];
                                tmem_ld8(tm_ring + sl * RW, w8[0]);
    #pragma unroll
                                for (int c = 0; c < CG; ++c) {
                                    tmem_ld8(tm_ring + sl * RW + 8 + 16 * c, w8[1 + 2 * c]);
                                    tmem_ld8(tm_ring + sl * RW + 16 + 16 * c, w8[2 + 2 * c]);
                                }
                                tmem_wait_ld();
    #pragma unroll
                                for (int r = 0; r < 4; ++r) {
                                    lu[r] = make_float2(w8[0][2 * r], w8[0][2 * r + 1]);
    #pragma unroll
                                    for (int c = 0; c < CG; ++c) {
                                        const float* q8 = w8[1 + 2 * c + (r >> 1)] + 4 * (r & 1);
                                        lp[c][r][0] = make_float2(q8[0], q8[1]);
                                        lp[c][r][1] = make_float2(q8[2], q8[3]);
                                    }
                                }
                            }
    #pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                tu[r] = d == 0 ? A::mul2(a.taps_t[0], lu[r], zero2)
                                               : A::mac2(tu[r], a.taps_t[d], lu[r], one2, zero2);
    #pragma unroll
                                for (int c = 0; c < CG; ++c)
    #pragma unroll
                                    for (int j = 0; j < 2; ++j)
                                        tp[c][r][j] = d == 0 ? A::mul2(a.taps_t[0], lp[c][r][j], zero2)
                                                             : A::mac2(tp[c][r][j], a.taps_t[d], lp[c][r][j], one2, zero2);
                            }
                        }
                    }
    #pragma unroll
                    for (int r = 0; r < ((SFK_EXP & 18) ? 0 : 4); ++r) {
                        // t-pass (conv3d.cpp:147-165): planes oldest..newest take
                        // taps_t[0..2RT]; first = w * in, then +=
                        float2 zu;
                        if constexpr (TMR) {
                            zu = tu[r];
                        } else {
                            zu = A::mul2(a.taps_t[0], ringu[r][(S_ + 1) % KR], zero2);
    #pragma unroll
                            for (int d = 1; d < K; ++d)
                                zu = A::mac2(zu, a.taps_t[d], ringu[r][(S_ + 1 + d) % KR], one2, zero2);
                        }
                        const float2 spv = *reinterpret_cast<const float2*>(sl + r * TX);
                        float2 prev = make_float2(0.0f, 0.0f);
                        if constexpr (ACC) {  // y so far (earlier groups); 0 outside the volume
                            const int y = q.tile_y * TY + band * 4 + r, x = q.tile_x * TX + 2 * cp;
                            if (y < a.H && x < a.W) {
                                const float* op = a.out + static_cast<long long>(to - a.out_buf_t0) * a.H * a.pitch +
                                                  static_cast<long long>(y) * a.pitch + x;
                                prev.x = op[0];
                                if (x + 1 < a.W) prev.y = op[1];
                            }
                        }
                        float v[2];
    #pragma unroll
                        for (int c = 0; c < CG; ++c) {
                            const float2 fv = *reinterpret_cast<const float2*>(sl + (1 + c) * G::SLAB + r * TX);
    #pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                float2 z;
                                if constexpr (TMR) {
                                    z = tp[c][r][j];
                                } else {
                                    z = A::mul2(a.taps_t[0], ringp[c][r][j][(S_ + 1) % KR], zero2);
    #pragma unroll
                                    for (int d = 1; d < K; ++d)
                                        z = A::mac2(z, a.taps_t[d], ringp[c][r][j][(S_ + 1 + d) % KR], one2, zero2);
                                }
                                // engine.cpp:113-119, channel sum engine.cpp:157-162
                                const float term = A::recombine(j ? spv.y : spv.x, j ? fv.y : fv.x,
                                                                inv_alpha, j ? zu.y : zu.x, z.y, z.x);
                                v[j] = c > 0 ? xadd(v[j], term) : (ACC ? xadd(j ? prev.y : prev.x, term) : term);
                            }
                        }
                        v2[r] = make_float2(v[0], v[1]);
                        // each thread overwrites exactly the S^p values it read
                        *reinterpret_cast<float2*>(sl + r * TX) = v2[r];
                    }
                    // hand the slab to the TMA unit (generic-proxy writes -> async
                    // proxy; clipped at the volume edge)
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&a.tm_out, myslab + sb * G::NSF * G::SLAB, q.tile_x * TX,
                                     q.tile_y * TY + 8 * wb, to - a.out_buf_t0);
                        bulk_commit();
                    }
                    if (bt == 0) SFK_T(ecnt, 11);
                    if (bt == 224) SFK_T(ecnt, 12);
                    ++ecnt;
                    if (last && !(SFK_EXP & 18)) {
                        // canonical reduction (device_common.cuh), warp-local: a warp
                        // holds two whole bands (lanes 0-15 band 2w, 16-31 band 2w+1),
                        // lane l of a half holds columns 2l and 2l+1: column sums over
                        // the 4 rows, butterfly xor 8, 4, 2, 1 over the half-warp, then
                        // even + odd column inside the lane. EXACT sums in fp64; FAST
                        // in fp32 within the 4 x 32 block (fp64 above it).
                        double sum;
                        if constexpr (FMA) {
                            float2 cs = make_float2(0.0f, 0.0f);
    #pragma unroll
                            for (int r = 0; r < 4; ++r) cs = ffma2(v2[r], v2[r], cs);
    #pragma unroll
                            for (int o = 8; o >= 1; o >>= 1) {
                                const float2 t = make_float2(__shfl_xor_sync(0xffffffffu, cs.x, o),
                                                             __shfl_xor_sync(0xffffffffu, cs.y, o));
                                cs = make_float2(cs.x + t.x, cs.y + t.y);
                            }
                            sum = static_cast<double>(cs.x + cs.y);
                        } else {
                            double cs0 = 0.0, cs1 = 0.0;
    #pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                cs0 += static_cast<double>(v2[r].x) * static_cast<double>(v2[r].x);
                                cs1 += static_cast<double>(v2[r].y) * static_cast<double>(v2[r].y);
                            }
    #pragma unroll
                            for (int o = 8; o >= 1; o >>= 1) {
                                cs0 += __shfl_xor_sync(0xffffffffu, cs0, o);
                                cs1 += __shfl_xor_sync(0xffffffffu, cs1, o);
                            }
                            sum = cs0 + cs1;
                        }
                        float cmax = 0.0f;
    #pragma unroll
                        for (int r = 0; r < 4; ++r) cmax = fmaxf(cmax, fmaxf(v2[r].x, v2[r].y));
                        const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                        const int gb = q.tile_y * G::NBANDS + band;
                        if ((lane & 15) == 0 && gb < a.nbands && q.tile_x < a.nhalves)
                            a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves +
                                   q.tile_x] = sum;
                        if (lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
                    }
                }
                q.next();
            };
            using std::integral_constant;
            while (!q.done) {
                plane(integral_constant<int, 0>{});
                if constexpr (K > 1) { if (q.done) break; plane(integral_constant<int, (K > 1 ? 1 : 0)>{}); }
                if constexpr (K > 2) { if (q.done) break; plane(integral_constant<int, (K > 2 ? 2 : 0)>{}); }
                if constexpr (K > 3) { if (q.done) break; plane(integral_constant<int, (K > 3 ? 3 : 0)>{}); }
                if constexpr (K > 4) { if (q.done) break; plane(integral_constant<int, (K > 4 ? 4 : 0)>{}); }
                if constexpr (K > 5) { if (q.done) break; plane(integral_constant<int, (K > 5 ? 5 : 0)>{}); }
                if constexpr (K > 6) { if (q.done) break; plane(integral_constant<int, (K > 6 ? 6 : 0)>{}); }
                if constexpr (K > 7) { if (q.done) break; plane(integral_constant<int, (K > 7 ? 7 : 0)>{}); }
                if constexpr (K > 8) { if (q.done) break; plane(integral_constant<int, (K > 8 ? 8 : 0)>{}); }
            }
        }
        const int bt_end = tid - NA;
        if ((bt_end & 31) == 0) bulk_wait0();  // the output slabs are written before the CTA exits
        if constexpr (SFK_TMR != 0) {
            tmem_wait_st();
            tcgen05_fence_before();
            named_bar_sync(3, NB);
            tcgen05_fence_after();
            if (bt_end < 32) tmem_dealloc<256>(tmem_base_sh);
        }
    }
}

}  // namespace sfk
