// fused_ws.cuh — warp-specialised SFSeg power-iteration step for sm_100a, EXACT
// arithmetic (the reference's rounding, bit for bit), radii up to (2, 5, 5).
// FAST arithmetic runs fused_rs.cuh / fused_mc.cuh; EXACT at larger radii runs
// fused_mc.cuh's EXACT kind.
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
// F_c u and F_c^2 u of one column) run as one FFMA2, keeping the reference's
// rounding (product, then sum: two FFMA2 with runtime one/zero operands, so
// ptxas cannot contract them).
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "step_common.cuh"  // PlaneStream, Arith, ffma2, canonical_tree32
#include "sfseg_types.cuh"

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
    static constexpr size_t PROD_FLOATS = size_t(PBU) + size_t(CG) * PBP;
    static constexpr size_t XB_FLOATS = 2 * size_t(XBUF);
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
template <int RT, int R, int CG, int STAGES, int NWA = 8, bool ACC = false>
__global__ void __launch_bounds__(32 * NWA + 256, 1) fused_step_ws(const __grid_constant__ FusedArgs a) {
    using G = WsGeom<RT, R, CG, STAGES, NWA>;
    using A = Arith<false>;  // EXACT: every product and sum rounded on its own
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
    __shared__ int prod_count;

    const int tid = threadIdx.x;
    griddep_wait();  // PDL: the previous step / finalize has completed
    // an earlier iteration hit a zero norm, or the early-exit rule already held
    if (a.st->degenerate || a.st->stop) return;
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
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            const float* rs = raw + static_cast<size_t>(s) * NIN * FB;
            // products over the halo box (engine.cpp:92-100): thread -> (row
            // lane pr0, float4 column pc4), rows pr0, pr0 + NPR, ... (constant
            // offsets, no index arithmetic in the loop)
            if (pact) {
                const float4* rx = reinterpret_cast<const float4*>(rs) + pr0 * BW4 + pc4;
                float* du = produ + pr0 * BWU + 4 * pc4;
                float* dp = prodp + pr0 * BWP + 8 * pc4;
                // the double-precision load_norm needs more registers than A's
                // budget allows for an unrolled loop
#pragma unroll 1
                for (int k = 0; k < G::PPASS; ++k) {
                    if (k == G::PPASS - 1 && pr0 + k * G::NPR >= BH) break;
                    const int i = k * G::NPR * BW4;
                    const float4 yv = rx[i];
                    const float4 sv = rx[FB / 4 + i];
                    // the first F load goes out with the others (2% faster)
                    const float4 fpre = rx[2 * (FB / 4) + i];
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
                        const float4 fv = cg == 0 ? fpre : rx[(2 + cg) * (FB / 4) + i];
                        float4 p0, p1;  // (F S^p X, (F F) S^p X) per point
                        p0.x = A::mul(fv.x, u.x);
                        p0.z = A::mul(fv.y, u.y);
                        p1.x = A::mul(fv.z, u.z);
                        p1.z = A::mul(fv.w, u.w);
                        // engine.cpp:98: fi * fi * sx
                        p0.y = A::mul(A::mul(fv.x, fv.x), u.x);
                        p0.w = A::mul(A::mul(fv.y, fv.y), u.y);
                        p1.y = A::mul(A::mul(fv.z, fv.z), u.z);
                        p1.w = A::mul(A::mul(fv.w, fv.w), u.w);
                        float4* pp = reinterpret_cast<float4*>(dp + cg * PBP + k * G::NPR * BWP);
                        pp[0] = p0;
                        pp[1] = p1;
                    }
                }
            }
            named_bar_sync(1, NA);  // products ready; raw stage s fully read
            if (tid == 0) {
                fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_next();
            }
            // x-pass (conv3d.cpp:88-101) into the free x buffer
            const int b = cnt & 1;
            mbar_wait(&xb_empty[b], ((cnt >> 1) & 1) ^ 1);
            float* xbu = xb + b * XBUF;
            float* xbp = xbu + XBU;
            if (xw < G::NWU) {
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
            mbar_arrive(&xb_full[b]);  // release: this thread's x-pass stores
            named_bar_sync(1, NA);     // every A thread is done with the products
            ++cnt;
        }
    } else {
        // =====================================================================
        // B: y-pass ring, t-pass, recombination, store, reductions
        // =====================================================================
        setmaxnreg_inc<G::RB>();
        const int bt = tid - NA;
        const int band = bt >> 4;  // rows 4*band .. 4*band+3 of the tile
        const int cp = bt & 15;    // columns 2cp, 2cp+1
        const int lane = bt & 31;
        const float inv_alpha = a.inv_alpha;
        const bool last = a.last_group;

        constexpr int KR = K;  // register ring depth
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
        if (lane == 0) {
            eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
            issue_slab();
        }
        const int sloff = ((band & 1) * 4) * TX + 2 * cp;  // this thread's rows in a slab

        // one plane with ring slot S_; the caller unrolls K planes so every
        // ring index is a compile-time constant (no rotation moves)
        auto plane = [&](auto slot_c) {
            constexpr int S_ = decltype(slot_c)::value;
            constexpr int SR = S_;  // register slot of this plane
            const int tg = a.out_t0 + q.p;
            const bool valid = tg >= 0 && tg < a.T;
            const bool emit = q.p - RT >= q.ta;
            const int to = tg - RT;

            // y-pass (conv3d.cpp:113-135): first = w * in, then += (d ascending),
            // accumulated straight into this plane's ring slot
            if (valid) {
                const int b = cnt & 1;
                mbar_wait(&xb_full[b], (cnt >> 1) & 1);
                const float* xbu = xb + b * XBUF;
                const float* xbp = xbu + XBU;
                const float2* su = reinterpret_cast<const float2*>(xbu + (band * 4) * TXU) + cp;
#pragma unroll
                for (int j = 0; j < 4 + 2 * R; ++j) {
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
                for (int c = 0; c < CG; ++c) {
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
            if (emit) {
                if (lane == 0) {
                    // slab buffer of plane ecnt+1 = the one stored from at ecnt-1:
                    // once that store has read it, fetch the next operands
                    bulk_wait_read0();
                    issue_slab();
                }
                const int sb = ecnt & 1;
                float* sl = myslab + sb * G::NSF * G::SLAB + sloff;
                mbar_wait(&slab_full[2 * wb + sb], (ecnt >> 1) & 1);
                float2 v2[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    // t-pass (conv3d.cpp:147-165): planes oldest..newest take
                    // taps_t[0..2RT]; first = w * in, then +=
                    float2 zu = A::mul2(a.taps_t[0], ringu[r][(S_ + 1) % KR], zero2);
#pragma unroll
                    for (int d = 1; d < K; ++d)
                        zu = A::mac2(zu, a.taps_t[d], ringu[r][(S_ + 1 + d) % KR], one2, zero2);
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
                            float2 z = A::mul2(a.taps_t[0], ringp[c][r][j][(S_ + 1) % KR], zero2);
#pragma unroll
                            for (int d = 1; d < K; ++d)
                                z = A::mac2(z, a.taps_t[d], ringp[c][r][j][(S_ + 1 + d) % KR], one2, zero2);
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
                ++ecnt;
                if (last) {
                    // canonical reduction (device_common.cuh), warp-local: a warp
                    // holds two whole bands (lanes 0-15 band 2w, 16-31 band 2w+1),
                    // lane l of a half holds columns 2l and 2l+1: column sums over
                    // the 4 rows, butterfly xor 8, 4, 2, 1 over the half-warp, then
                    // even + odd column inside the lane, all in fp64.
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
                    const double sum = cs0 + cs1;
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
        const int bt_end = tid - NA;
        if ((bt_end & 31) == 0) bulk_wait0();  // the output slabs are written before the CTA exits
    }
}

}  // namespace sfk
