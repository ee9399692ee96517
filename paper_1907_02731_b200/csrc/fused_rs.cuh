// fused_rs.cuh — SFSeg power-iteration step, FAST arithmetic, with the
// products formed in registers inside the x-pass ("register-streamed").
//
// Same job as fused_step_ws (fused_ws.cuh): one launch per channel group per
// iteration does the products (engine.cpp:92-100), the three separable
// convolutions (conv3d.cpp:80-185), the recombination and channel sum
// (engine.cpp:107-120, 157-162) and the sum-of-squares / max scans of
// normalize_l2 / project_binary (engine.cpp:168-205).
//
// What changes against fused_step_ws, and why: there the A
// warps first wrote the product fields u, (F u, F^2 u) for the whole halo
// box to shared memory, barrier-synchronised, and then read them back for
// the x-pass. The shared-memory datapath is the binding resource of this
// stencil, and that round trip was ~1/4 of its traffic plus a serial phase
// on the A warps' critical path. Here an x-pass thread reads the raw TMA
// box (y_k, S^p, F) for its 8-output strip and forms u, F u, F^2 u in
// registers for the 8 + 2R inputs it convolves. The box width is an odd
// number of float4s so eight rows of one strip hit eight distinct 16-byte
// bank groups. The raw box now lives through the x-pass, so the TMA ring
// gets a third stage (the product tile's shared memory pays for it).
//
// FAST only: the normalisation 1/||y_k|| is applied to the output instead of
// to every input (the operator is linear: A(y s) = s A(y)), which takes one
// multiply off every one of the (8 + 2R) x 3 inputs a strip reads. Binarised
// iterations (mode 2) still apply the sigmoid per input. EXACT keeps
// fused_step_ws, whose on-load normalisation reproduces the reference's
// float(double(y) * inv) rounding.
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "step_common.cuh"  // PlaneStream, Arith, ffma2, canonical_tree32
#include "fused_ws.cuh"    // SFK_T timeline instrumentation
#include "sfseg_types.cuh"

#ifndef SFK_RS_EXP
#define SFK_RS_EXP 0
#endif
// SFK_RS_TMR=1: B keeps the t-pass ring of y-filtered planes in tensor
// memory (tcgen05.ld/st) instead of registers
#ifndef SFK_RS_TMR
#define SFK_RS_TMR 0
#endif
// SFK_RS_SPLIT=1: the B role is split in two warp groups that meet in a TMEM
// ring: B warps run the y-pass and store each y-filtered plane into tensor
// memory; C warps (same TMEM lane quadrants) run the t-pass from it, the
// recombination, the store and the reductions
#ifndef SFK_RS_SPLIT
#define SFK_RS_SPLIT 0
#endif
// SFK_RS_LSU=1: B fetches the recombination operands with plain loads one
// emitted plane ahead and stores y_{k+1} with plain stores, which leaves the
// per-SM TMA unit to the halo boxes alone (it is the busiest unit: ~32 B/clk)
#ifndef SFK_RS_LSU
#define SFK_RS_LSU 0
#endif
// SFK_RS_SPX=1 (with the TMEM ring): A passes S^p and F of the output points
// to B through the x-pass buffer (it reads them from the halo box anyway), B
// keeps them in the TMEM ring slot of their plane: no recombination operand
// loads at all, so the L2 -> SM traffic is the halo boxes alone
#ifndef SFK_RS_SPX
#define SFK_RS_SPX 0
#endif
// SFK_RS_STG=1: y_{k+1} leaves by plain coalesced stores instead of a TMA
// store; SFK_RS_PRODUCER: the A thread that issues the halo-box TMA loads
// (default thread 0; moving it to a one-block warp measured 2.7% slower)
#ifndef SFK_RS_STG
#define SFK_RS_STG 0
#endif
#ifndef SFK_RS_PRODUCER
#define SFK_RS_PRODUCER 0
#endif
// SFK_RS_DEFRED=1: the reductions of an emitted plane run at the start of
// the next plane's y-pass, so their shuffle chains overlap its FMAs
#ifndef SFK_RS_DEFRED
#define SFK_RS_DEFRED 0
#endif
// SFK_RS_WIDE=1: one CTA-wide TMA load of the S^p / F tile per emitted plane
// and one TMA store of the y tile (two B-wide barriers per plane) instead of a
// load pair and a store per B warp: 3 TMA operations per plane instead of 24
#ifndef SFK_RS_WIDE
#define SFK_RS_WIDE 1
#endif
// SFK_RS_RAWFENCE=0: no proxy fence before the producer refills a box stage
// (the stage's generic reads have completed: their values were consumed before
// the named barrier that precedes the refill)
// SFK_RS_WREDUCE=1 (WIDE): one B warp per plane finishes the column-sum
// butterflies from shared memory instead of every warp shuffling (238 us vs
// 214 us: the reducing warp delays the next barrier)
#ifndef SFK_RS_WREDUCE
#define SFK_RS_WREDUCE 0
#endif
#ifndef SFK_RS_RAWFENCE
#define SFK_RS_RAWFENCE 1
#endif
// SFK_RS_PSPLIT=1: the three halo boxes of a plane are issued by lane 0 of
// the last three A warps (one box each; the x box carries the expect_tx of
// all three) instead of one thread issuing all three: the issue (~1000
// cycles per plane) leaves warp 0, which also runs two x-pass blocks.
// Measured 206.4 us per c1 launch against 213.5 (timeline: warp 0's issue +
// loop 996 -> 339 cycles per plane), so on.
#ifndef SFK_RS_PSPLIT
#define SFK_RS_PSPLIT 1
#endif
// SFK_RS_CPA=1 (WIDE): each B warp fetches the S^p / F rows of its own
// outputs with cp.async (LSU path) one emitted plane ahead, which takes the
// operand tiles off the per-SM TMA unit (it then carries only the halo
// boxes and the y store). Measured 242 us against 206 (B waits ~1500 cycles
// per plane for the copies), so off.
#ifndef SFK_RS_CPA
#define SFK_RS_CPA 0
#endif
// SFK_RS_HALF=1: the x-pass rows beyond the first 8 NWA (the 2R halo rows
// below the tile) run as 4-wide strips spread over the first warps, so no
// A warp does two full 8-row passes per plane. Measured 207.4 us against
// 205.9 (warp 0's x-pass drops 2396 -> 2126 cycles per plane, the plane
// period does not move), so off.
#ifndef SFK_RS_HALF
#define SFK_RS_HALF 0
#endif
// SFK_RS_CPS: CTAs resident per SM (2 with a half-height tile: two
// independent pipelines per SM hide each other's barrier waits); the
// setmaxnreg budgets then share each SMSP's 512 registers per lane slot
// Measured: TY = 32, 4 + 4 warps, 2 stages, 2 CTAs per SM: 254.7 us
// against 206 (the 2R halo rows cost more than the second pipeline hides).
#ifndef SFK_RS_CPS
#define SFK_RS_CPS 1
#endif

namespace sfk {

// the 32-column xor-butterfly (16, 8, 4, 2, 1) of device_common.cuh evaluated
// serially on 32 column sums, in fp32: the same operands in the same order,
// so the same bits as the shuffle butterfly
__device__ __forceinline__ float tree32f_s4(const float* v, int i) {
    const float a = (v[i] + v[i + 16]) + (v[i + 8] + v[i + 24]);
    const float b = (v[i + 4] + v[i + 20]) + (v[i + 12] + v[i + 28]);
    return a + b;
}
__device__ __forceinline__ float tree32f(const float* v) {
    return (tree32f_s4(v, 0) + tree32f_s4(v, 2)) + (tree32f_s4(v, 1) + tree32f_s4(v, 3));
}

// TY: tile rows; BR: output rows per B thread (a B warp covers BR rows x 32
// columns, so there are TY / BR B warps)
template <int RT, int R, int NWA, int STAGES, int TY_ = 64, int BR_ = 8, bool TMR_ = (SFK_RS_TMR != 0)>
struct RsGeom {
    static constexpr bool TMR = TMR_;  // t-pass ring in tensor memory
    static constexpr int TY = TY_, TX = 32, BR = BR_;
    static constexpr bool SPLIT = SFK_RS_SPLIT != 0;
    static constexpr int NWB = TY / BR;
    static constexpr int NWC = SPLIT ? NWB : 0;
    static constexpr int NA = 32 * NWA, NB = 32 * NWB, NC = 32 * NWC, NT = NA + NB + NC;
    static constexpr int NS = 8;  // TMEM ring slots per thread (SPLIT)
    static constexpr int K = 2 * RT + 1;
    static constexpr int BH = TY + 2 * R;
    // x halos: the box must start on a 16-byte boundary (TMA faults on an
    // unaligned innermost coordinate), so the left halo HX is R rounded up to
    // whole float4s; the right halo HR >= R is chosen so the row is an odd
    // number of float4s, which makes float4 reads of 8 rows at one strip
    // conflict-free
    static constexpr int HX = (R + 3) / 4 * 4;
#ifndef SFK_RS_ODDBOX
#define SFK_RS_ODDBOX 1
#endif
    static constexpr int HR = (!SFK_RS_ODDBOX || ((TX + HX + (R + 3) / 4 * 4) / 4) % 2 == 1) ? (R + 3) / 4 * 4
                                                                                             : (R + 3) / 4 * 4 + 4;
    static constexpr int BW = TX + HX + HR;
    static constexpr int BW4 = BW / 4;
    static constexpr int XOFF = HX - R;  // first box column a strip reads
    static constexpr int FB = (BH * BW + 31) / 32 * 32;
    static constexpr int NIN = 3;  // raw fields: y_k, S^p, F
    // x-pass items: (row, 8-column strip); a warp pass = 8 rows x 4 strips
    static constexpr int SW = 8, NSTRIP = TX / SW;
    static constexpr int NINX = SW + 2 * R;            // inputs per strip
    static constexpr int NLD = (XOFF + NINX + 3) / 4;  // float4 loads per field
    static constexpr int RBLK = (BH + 7) / 8;          // 8-row blocks
    static constexpr int XPASS = (RBLK + NWA - 1) / NWA;
    // x-pass output, read by B: u [BH][TXU], (F u, F^2 u) pairs [BH][TXQ]
    static constexpr int TXU = TX + 4, TXQ = 2 * TX + 4;
    static constexpr int XBU = (BH * TXU + 31) / 32 * 32;
    static constexpr int XBP = (BH * TXQ + 31) / 32 * 32;
    static constexpr bool SPX = SFK_RS_SPX != 0 && TMR_ && (2 * RT + 1) * 5 * BR_ <= 256;
    static constexpr int XBS = SPX ? TY * TXU : 0;  // S^p rows of the output points (F follows)
    static constexpr int XBUF = XBU + XBP + 2 * XBS;
    static constexpr int NBANDS = TY / 4;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
#ifndef SFK_RS_NXB
#define SFK_RS_NXB 2
#endif
    static constexpr int NXB = SFK_RS_NXB;  // x-pass buffers between A and B
    static constexpr size_t XB_FLOATS = NXB * size_t(XBUF);
    // per B warp: S^p and F of its BR output rows (TMA, loaded one emitted
    // plane ahead) and the staging rows of y_{k+1} for the TMA store
    static constexpr int SLAB = BR * TX;
    static constexpr int SLW = SPX ? 1 : 3;  // per-warp slab rows: S^p, F, y staging (SPX: staging)
    static constexpr size_t SL_FLOATS = size_t(NWB) * SLW * SLAB;
    static constexpr int NBAR = STAGES + 2 * SFK_RS_NXB + NWB + (SPLIT ? 2 * NWB * NS : 0);
    static constexpr size_t SMEM_BYTES = (RAW_FLOATS + XB_FLOATS + SL_FLOATS) * sizeof(float) + NBAR * 8;
    // setmaxnreg budgets. Warp w runs on SMSP w % 4, whose register file
    // holds 512 registers per lane slot; the launch grants every warp
    // 512 / (most warps on one SMSP), and the budgets must fit every SMSP.
#ifndef SFK_RS_RA
#define SFK_RS_RA 64
#endif
    static constexpr int RA = SFK_RS_RA;
    static constexpr int NW = NWA + NWB + NWC;
    static constexpr int CPS = SFK_RS_CPS;
    static constexpr int SMSP_REGS = 512 / CPS;  // per lane slot, this CTA's share
    static constexpr int RPOOL = (SMSP_REGS / ((NW + 3) / 4)) / 8 * 8;
    // unsplit: the B warps take what A gives back. SPLIT: B keeps the launch
    // grant and the C warps take what A gives back.
    static constexpr int rb_for(int s) {
        int wa = 0, wb = 0, wk = 0;
        for (int w = 0; w < NW; ++w)
            if (w % 4 == s) {
                if (w < NWA) ++wa;
                else if (SPLIT && w < NWA + NWB) ++wk;
                else ++wb;
            }
        return wb ? (SMSP_REGS - wa * RA - wk * RPOOL) / wb : SMSP_REGS;
    }
    static constexpr int rb_min() {
        int m = SMSP_REGS;
        for (int s = 0; s < 4; ++s) m = rb_for(s) < m ? rb_for(s) : m;
        return m;
    }
    // and the CTA's launch pool: B takes no more than A gives back
    static constexpr int RB_POOL = RPOOL + (RPOOL - RA) * NWA / (SPLIT ? NWC : NWB);
    static constexpr int RB_CAP = rb_min() < RB_POOL ? rb_min() : RB_POOL;
    static constexpr int RB = (RB_CAP < 248 ? RB_CAP : 248) / 8 * 8;
    static_assert(BW4 % 2 == 1 || !SFK_RS_ODDBOX, "odd float4 box rows");
    static_assert((TXU / 4) % 2 == 1 && (TXQ / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert(RA <= RPOOL && RB >= RPOOL, "setmaxnreg: A gives, B takes");
    static_assert(NWA % 4 == 0 && NWB % 4 == 0, "setmaxnreg acts on whole warpgroups");
    static_assert(!SPLIT || (BR == 8 && NS * 3 * BR <= 256), "SPLIT: TMEM ring of one thread");
    static_assert(TY % BR == 0 && (BR == 4 || BR == 8), "B rows per thread");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// PEER: the time-sharded instantiation that also stores its edge planes into
// the neighbours' halo frames (a separate instantiation: the single-GPU
// kernel does not carry the extra epilogue code)
template <int RT, int R, int NWA, int STAGES, int TY_, int BR_, bool TMR_, bool ACC, bool PEER = false>
__global__ void __launch_bounds__(RsGeom<RT, R, NWA, STAGES, TY_, BR_, TMR_>::NT, SFK_RS_CPS)
    fused_step_rs(const __grid_constant__ FusedArgs a) {
    using G = RsGeom<RT, R, NWA, STAGES, TY_, BR_, TMR_>;
    using A = Arith<true>;
    constexpr int BR = G::BR, TY = G::TY, TX = G::TX, NA = G::NA, NB = G::NB, K = G::K, NWB = G::NWB;
    constexpr int BH = G::BH, BW = G::BW, FB = G::FB, BW4 = G::BW4, SW = G::SW;
    constexpr int TXU = G::TXU, TXQ = G::TXQ, XBU = G::XBU, XBUF = G::XBUF, SLAB = G::SLAB;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                    // [STAGES][3][FB]    TMA boxes
    constexpr int NXB = G::NXB;
    float* xb = raw + G::RAW_FLOATS;      // [NXB][XBUF]        x-pass output
    float* bsl = xb + G::XB_FLOATS;       // [NWB][3][BR][TX]   S^p, F, y_{k+1} rows
    uint64_t* mbar = reinterpret_cast<uint64_t*>(bsl + G::SL_FLOATS);
    uint64_t* raw_full = mbar;                // [STAGES]  TMA -> A
    uint64_t* xb_full = mbar + STAGES;              // [NXB]  A -> B (count NA)
    uint64_t* xb_empty = mbar + STAGES + NXB;       // [NXB]  B -> A (count NB)
    uint64_t* slab_full = mbar + STAGES + 2 * NXB;  // [NWB]  TMA -> B (C) warp
    uint64_t* ring_full = slab_full + NWB;          // [NWB][NS]  B -> C (SPLIT)
    uint64_t* ring_free = ring_full + NWB * G::NS;  // [NWB][NS]  C -> B (SPLIT)

    __shared__ IterState st;
    __shared__ PlaneStream prodq;
    __shared__ PlaneStream slabq[NWB];
    __shared__ int prod_count;
    __shared__ uint32_t tmem_base_sh;
    // WIDE: per-plane column sums of y^2 per 4-row band and per-warp maxima,
    // reduced by one B warp after the store barrier
    __shared__ float red_cols[SFK_RS_WIDE && SFK_RS_WREDUCE ? TY_ / 4 : 1][32];
    __shared__ float red_max[SFK_RS_WIDE && SFK_RS_WREDUCE ? TY_ / BR_ : 1];

    const int tid = threadIdx.x;
    griddep_wait();  // PDL: the previous step / finalize has completed
    if (a.st->degenerate && SFK_RS_EXP == 0) return;  // an earlier iteration hit a zero norm
    const int s0 = a.sched_off[blockIdx.x], s1 = a.sched_off[blockIdx.x + 1];
    if (s0 >= s1) return;

    if (tid == 0) {
        st = *a.st;
        for (int s = 0; s < STAGES; ++s) mbar_init(&raw_full[s], 1);
        for (int b = 0; b < NXB; ++b) {
            mbar_init(&xb_full[b], NA);
            mbar_init(&xb_empty[b], NB);
        }
        for (int w = 0; w < NWB; ++w) mbar_init(&slab_full[w], 1);
        if constexpr (G::SPLIT)
            for (int w = 0; w < 2 * NWB * G::NS; ++w) mbar_init(&ring_full[w], 32);
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        prefetch_tensormap(&a.tm_sp);
        prefetch_tensormap(&a.tm_f[0]);
        prefetch_tensormap(&a.tm_out);
        prefetch_tensormap(&a.tm_spc);
        prefetch_tensormap(&a.tm_fc[0]);
    }
    __syncthreads();

    const float2 zero2 = make_float2(0.0f, 0.0f);

    if (tid < NA) {
        // =====================================================================
        // A: TMA producer + x-pass with in-register products
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
            float* dst = raw + static_cast<size_t>(s) * 3 * FB;
            uint64_t* bar = &raw_full[s];
            mbar_arrive_expect_tx(bar, 3 * BH * BW * sizeof(float));
            const int bx = prodq.tile_x * TX - G::HX, by = prodq.tile_y * TY - R, bt = tg - a.buf_t0;
            tma_load_3d(dst, &a.tm_x, bar, bx, by, bt);
            tma_load_3d(dst + FB, &a.tm_sp, bar, bx, by, bt);
            tma_load_3d(dst + 2 * FB, &a.tm_f[0], bar, bx, by, bt);
            ++prod_count;
            prodq.next();
        };
        constexpr int PROD = SFK_RS_PRODUCER;
        constexpr bool PSPLIT = SFK_RS_PSPLIT != 0;
        constexpr bool HALF = SFK_RS_HALF != 0 && 8 * NWA <= BH && (BH - 8 * NWA) * (TX / 4) <= NA;
        // PSPLIT: box `pbox` of every plane is issued by lane 0 of warp
        // NWA - 3 + pbox, each with its own copy of the plane cursor
        const int pbox = (tid >> 5) - (NWA - 3);
        const bool pissuer = PSPLIT && (tid & 31) == 0 && pbox >= 0;
        PlaneStream pq;
        int pcount = 0;
        auto issue_box = [&]() {
            while (!pq.done) {
                const int tg = a.out_t0 + pq.p;
                if (tg >= 0 && tg < a.T) break;
                pq.next();
            }
            if (pq.done) return;
            const int tg = a.out_t0 + pq.p;
            const int s = pcount % STAGES;
            float* dst = raw + static_cast<size_t>(s) * 3 * FB;
            uint64_t* bar = &raw_full[s];
            const int bx = pq.tile_x * TX - G::HX, by = pq.tile_y * TY - R, bt = tg - a.buf_t0;
            if (pbox == 0) {
                mbar_arrive_expect_tx(bar, 3 * BH * BW * sizeof(float));
                tma_load_3d(dst, &a.tm_x, bar, bx, by, bt);
            } else if (pbox == 1) {
                tma_load_3d(dst + FB, &a.tm_sp, bar, bx, by, bt);
            } else {
                tma_load_3d(dst + 2 * FB, &a.tm_f[0], bar, bx, by, bt);
            }
            ++pcount;
            pq.next();
        };
        if (pissuer) {
            pq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            for (int s = 0; s < STAGES; ++s) issue_box();
        }
        if (!PSPLIT && tid == PROD) {
            prodq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            prod_count = 0;
            for (int s = 0; s < STAGES; ++s) issue_next();
        }
        const bool sigm = st.mode == 2;
        const int xw = tid >> 5, xl = tid & 31;  // warp; lane -> (row xl & 7, strip xl >> 3)

        // one x-pass item (conv3d.cpp:88-101): row r, strip sx (SW outputs).
        // u runs as column pairs (2k, 2k+1) with tap pairs (w[e], w[e-1]);
        // (F u, F^2 u) runs as a pair per column with a broadcast tap.
        // SWI: strip width (8; 4 for the HALF second pass)
        auto item = [&](auto sig_c, auto sw_c, const float* rs, float* xbu, float* xbp, int r, int sx) {
            constexpr bool SIG = decltype(sig_c)::value;
            constexpr int SW = decltype(sw_c)::value;
            constexpr int NINXI = SW + 2 * R, NLDI = (G::XOFF + NINXI + 3) / 4;
            const float4* py = reinterpret_cast<const float4*>(rs) + r * BW4 + sx * (SW / 4);
            float2 ou[SW / 2];
            float2 op[SW];
            float4 yv, sv, fv;
#pragma unroll
            for (int m4 = 0; m4 < NLDI * 4; ++m4) {
                if (m4 % 4 == 0) {
                    yv = py[m4 / 4];
                    sv = py[FB / 4 + m4 / 4];
                    fv = py[2 * (FB / 4) + m4 / 4];
                }
                const int m = m4 - G::XOFF;
                if (m < 0 || m >= NINXI) continue;
                const int c = m4 % 4;
                const float y = c == 0 ? yv.x : c == 1 ? yv.y : c == 2 ? yv.z : yv.w;
                const float s = c == 0 ? sv.x : c == 1 ? sv.y : c == 2 ? sv.z : sv.w;
                const float f = c == 0 ? fv.x : c == 1 ? fv.y : c == 2 ? fv.z : fv.w;
                const float x = SIG ? A::load_sigmoid(y, st) : y;
                const float u = s * x;  // engine.cpp:92-100 (FAST: F (F u))
                const float fu = f * u;
                const float2 pr = make_float2(fu, f * fu);
#pragma unroll
                for (int k = 0; k < SW / 2; ++k) {
                    const int e = m - 2 * k;
                    if (e < 0 || e > 2 * R + 1) continue;
                    ou[k] = ffma2(make_float2(u, u), a.tpair_x[e], e == 0 ? zero2 : ou[k]);
                }
#pragma unroll
                for (int j = 0; j < SW; ++j) {
                    const int d = m - j;
                    if (d < 0 || d > 2 * R) continue;
                    op[j] = ffma2(pr, make_float2(a.taps_x[d], a.taps_x[d]), d == 0 ? zero2 : op[j]);
                }
            }
            float4* du = reinterpret_cast<float4*>(xbu + r * TXU + sx * SW);
#pragma unroll
            for (int v = 0; v < SW / 4; ++v)
                du[v] = make_float4(ou[2 * v].x, ou[2 * v].y, ou[2 * v + 1].x, ou[2 * v + 1].y);
            float4* dp = reinterpret_cast<float4*>(xbp + r * TXQ + 2 * sx * SW);
#pragma unroll
            for (int v = 0; v < SW / 2; ++v)
                dp[v] = make_float4(op[2 * v].x, op[2 * v].y, op[2 * v + 1].x, op[2 * v + 1].y);
            if constexpr (G::SPX) {
                // S^p and F of this strip's output points (box columns HX ..)
                if (r >= R && r < R + TY) {
                    float4* ds = reinterpret_cast<float4*>(xbp + G::XBP + (r - R) * TXU + sx * SW);
#pragma unroll
                    for (int v = 0; v < SW / 4; ++v) {
                        ds[v] = py[FB / 4 + G::HX / 4 + v];
                        ds[G::XBS / 4 + v] = py[2 * (FB / 4) + G::HX / 4 + v];
                    }
                }
            }
        };

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;  // in-volume planes handled
        for (; !q.done; q.next()) {
            const int tg = a.out_t0 + q.p;
            if (tg < 0 || tg >= a.T) continue;  // planes outside the volume: B zero-fills
            const int s = cnt % STAGES;
            const int b = cnt % NXB;
            if (tid == 0 || tid == 64) SFK_T(cnt, tid ? 13 : 0);
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            if (tid == 0) SFK_T(cnt, 1);
            mbar_wait(&xb_empty[b], ((cnt / NXB) & 1) ^ 1);
            if (tid == 0) SFK_T(cnt, 2);
            const float* rs = raw + static_cast<size_t>(s) * 3 * FB;
            float* xbu = xb + b * XBUF;
            float* xbp = xbu + XBU;
            using W8 = std::integral_constant<int, 8>;
            using W4 = std::integral_constant<int, 4>;
            if constexpr (HALF) {
                // pass 1: box rows 8 xw .. 8 xw + 7, four 8-wide strips; pass 2:
                // the last BH - 8 NWA rows as 4-wide strips over the first warps
                if (!(SFK_RS_EXP & 1)) {
                    const int r = xw * 8 + (xl & 7);
                    if (sigm) item(std::true_type{}, W8{}, rs, xbu, xbp, r, xl >> 3);
                    else item(std::false_type{}, W8{}, rs, xbu, xbp, r, xl >> 3);
                    const int it2 = xw * 32 + xl;
                    if (it2 < (BH - 8 * NWA) * (TX / 4)) {
                        const int r2 = 8 * NWA + it2 / (TX / 4), s2 = it2 % (TX / 4);
                        if (sigm) item(std::true_type{}, W4{}, rs, xbu, xbp, r2, s2);
                        else item(std::false_type{}, W4{}, rs, xbu, xbp, r2, s2);
                    }
                }
            } else {
#pragma unroll
            for (int k = 0; k < G::XPASS; ++k) {
                const int blk = xw + k * NWA;
                if (blk >= G::RBLK) break;
                const int r = blk * 8 + (xl & 7);
                if (r >= BH || (SFK_RS_EXP & 1)) continue;
                if (sigm && !(SFK_RS_EXP & 4))
                    item(std::true_type{}, W8{}, rs, xbu, xbp, r, xl >> 3);
                else
                    item(std::false_type{}, W8{}, rs, xbu, xbp, r, xl >> 3);
            }
            }
            if (tid == 0 || tid == 64) SFK_T(cnt, tid ? 14 : 3);
            mbar_arrive(&xb_full[b]);  // release: this thread's x-pass stores
            named_bar_sync(1, NA);     // raw stage s fully read
            if (tid == 0) SFK_T(cnt, 4);
            if (!PSPLIT && tid == PROD) {
                if (SFK_RS_RAWFENCE) fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_next();
            }
            if (pissuer) {
                fence_proxy_async();
                issue_box();
            }
            ++cnt;
        }
    } else if constexpr (G::SPLIT) {
        // =====================================================================
        // SPLIT: B = y-pass into a TMEM ring; C = t-pass, recombination,
        // store, reductions. B warp i and C warp i share a TMEM lane quadrant.
        // =====================================================================
        constexpr int NS = G::NS, RW = 3 * BR;
        const int bt = tid - NA;
        const bool isC = bt >= NB;
        const int wi = (isC ? bt - NB : bt) >> 5;
        const int lane = bt & 31;
        if (bt < 32) tmem_alloc<512>(&tmem_base_sh);
        tcgen05_fence_before();
        named_bar_sync(2, NB + G::NC);
        tcgen05_fence_after();
        const int wq = (NA / 32 + (bt >> 5)) & 3;  // CTA warp id % 4 (same for B warp i and C warp i)
        const uint32_t ring = tmem_base_sh + (static_cast<uint32_t>(32 * wq) << 16) + static_cast<uint32_t>((wi >> 2) * 256);
        uint64_t* rfull = ring_full + wi * NS;
        uint64_t* rfree = ring_free + wi * NS;
        if (!isC) {
            // ---------------- B: y-pass (conv3d.cpp:113-135) ----------------
            PlaneStream q;
            q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            int cnt = 0;  // in-volume planes consumed
            for (int c = 0; !q.done; q.next(), ++c) {
                const int tg = a.out_t0 + q.p;
                float2 au[BR / 2], ap[BR];
#pragma unroll
                for (int k = 0; k < BR / 2; ++k) au[k] = zero2;
#pragma unroll
                for (int r = 0; r < BR; ++r) ap[r] = zero2;
                if (tg >= 0 && tg < a.T) {
                    const int b = cnt % NXB;
                    mbar_wait(&xb_full[b], (cnt / NXB) & 1);
                    const float* xbu = xb + b * XBUF + (BR * wi) * TXU + lane;
                    const float2* xbp = reinterpret_cast<const float2*>(xb + b * XBUF + XBU + (BR * wi) * TXQ) + lane;
#pragma unroll
                    for (int j = 0; j < BR + 2 * R; ++j) {
                        const float vin = xbu[j * TXU];
                        const float2 pv = xbp[j * (TXQ / 2)];
#pragma unroll
                        for (int k = 0; k < BR / 2; ++k) {
                            const int e = j - 2 * k;
                            if (e < 0 || e > 2 * R + 1) continue;
                            au[k] = ffma2(make_float2(vin, vin), a.tpair_y[e], au[k]);
                        }
#pragma unroll
                        for (int r = 0; r < BR; ++r) {
                            const int d = j - r;
                            if (d < 0 || d > 2 * R) continue;
                            ap[r] = ffma2(pv, make_float2(a.taps_y[d], a.taps_y[d]), ap[r]);
                        }
                    }
                    mbar_arrive(&xb_empty[b]);
                    ++cnt;
                }
                const int sl = c % NS;
                mbar_wait(&rfree[sl], ((c / NS) & 1) ^ 1);
                tcgen05_fence_after();
                float w[8];
#pragma unroll
                for (int k = 0; k < BR / 2; ++k) {
                    w[2 * k] = au[k].x;
                    w[2 * k + 1] = au[k].y;
                }
                tmem_st8(ring + sl * RW, w);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        w[2 * r] = ap[4 * h + r].x;
                        w[2 * r + 1] = ap[4 * h + r].y;
                    }
                    tmem_st8(ring + sl * RW + 8 + 8 * h, w);
                }
                tmem_wait_st();
                tcgen05_fence_before();
                mbar_arrive(&rfull[sl]);
            }
        } else {
            // ---------------- C: t-pass, recombination, store, reductions ----------------
            setmaxnreg_inc<G::RB>();
            const float inv_alpha = a.inv_alpha;
            const bool last = a.last_group;
            const float scale = st.mode == 1 ? st.inv_f : 1.0f;
            float* slab = bsl + wi * 3 * SLAB;
            uint64_t* sfull = &slab_full[wi];
            PlaneStream& eq = slabq[wi];  // lane 0 only
            auto issue_slab = [&]() {
                if (eq.done) return;
                mbar_arrive_expect_tx(sfull, 2 * SLAB * sizeof(float));
                const int x = eq.tile_x * TX, y = eq.tile_y * TY + BR * wi, t = a.out_t0 + eq.p - a.buf_t0;
                tma_load_3d(slab, &a.tm_spc, sfull, x, y, t);
                tma_load_3d(slab + SLAB, &a.tm_fc[0], sfull, x, y, t);
                eq.next();
            };
            if (lane == 0) {
                eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
                issue_slab();
            }
            PlaneStream q;
            q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            int ecnt = 0;
            for (int c = 0; !q.done; ++c) {
                const bool emit = q.p - RT >= q.ta;
                const bool seg_last = q.p + 1 >= q.tb + RT;
                const int to = a.out_t0 + q.p - RT;
                mbar_wait(&rfull[c % NS], (c / NS) & 1);
                tcgen05_fence_after();
                if (emit) {
                    // t-pass (conv3d.cpp:147-165): planes c - 2RT .. c take taps_t[0..2RT]
                    float2 tu[BR / 2], tp[BR];
#pragma unroll
                    for (int d = 0; d < K; ++d) {
                        float wv[3][8];
                        const int sl = (c - 2 * RT + d) % NS;
                        tmem_ld8(ring + sl * RW, wv[0]);
                        tmem_ld8(ring + sl * RW + 8, wv[1]);
                        tmem_ld8(ring + sl * RW + 16, wv[2]);
                        tmem_wait_ld();
                        const float2 w2 = make_float2(a.taps_t[d], a.taps_t[d]);
#pragma unroll
                        for (int k = 0; k < BR / 2; ++k)
                            tu[k] = ffma2(make_float2(wv[0][2 * k], wv[0][2 * k + 1]), w2, d == 0 ? zero2 : tu[k]);
#pragma unroll
                        for (int r = 0; r < BR; ++r)
                            tp[r] = ffma2(make_float2(wv[1 + r / 4][2 * (r % 4)], wv[1 + r / 4][2 * (r % 4) + 1]), w2,
                                          d == 0 ? zero2 : tp[r]);
                    }
                    mbar_wait(sfull, ecnt & 1);
                    float spv[BR], fv[BR];
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        spv[r] = slab[r * TX + lane];
                        fv[r] = slab[SLAB + r * TX + lane];
                    }
                    __syncwarp();
                    if (lane == 0) {
                        fence_proxy_async();
                        issue_slab();
                    }
                    float v[BR];
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        const float tur = (r & 1) ? tu[r / 2].y : tu[r / 2].x;
                        v[r] = A::recombine(spv[r] * scale, fv[r], inv_alpha, tur, tp[r].y, tp[r].x);
                    }
                    const int ox = q.tile_x * TX, oy = q.tile_y * TY + BR * wi;
                    if constexpr (ACC) {
                        const int nr = a.H - oy;
                        const float* po = a.out + (static_cast<size_t>(to - a.out_buf_t0) * a.H + oy) * a.pitch + ox + lane;
#pragma unroll
                        for (int r = 0; r < BR; ++r)
                            if (r < nr && ox + lane < a.W) v[r] += po[static_cast<size_t>(r) * a.pitch];
                    }
                    float* ost = slab + 2 * SLAB;
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < BR; ++r) ost[r * TX + lane] = v[r];
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&a.tm_out, ost, ox, oy, to - a.out_buf_t0);
                        bulk_commit();
                    }
                    ++ecnt;
                    if (last) {
#pragma unroll
                        for (int h = 0; h < BR / 4; ++h) {
                            float cs = 0.0f;
#pragma unroll
                            for (int r = 0; r < 4; ++r) cs = fmaf(v[4 * h + r], v[4 * h + r], cs);
#pragma unroll
                            for (int o = 16; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
                            const int gb = q.tile_y * G::NBANDS + (BR / 4) * wi + h;
                            if (lane == 0 && gb < a.nbands && q.tile_x < a.nhalves)
                                a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves + q.tile_x] =
                                    static_cast<double>(cs);
                        }
                        float cmax = 0.0f;
#pragma unroll
                        for (int r = 0; r < BR; ++r) cmax = fmaxf(cmax, v[r]);
                        const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                        if (lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
                    }
                }
                // release the ring slots no future output of this segment needs
                tcgen05_fence_before();
                if (emit) mbar_arrive(&rfree[(c - 2 * RT) % NS]);
                if (seg_last)
                    for (int d = 2 * RT - 1; d >= 0; --d) mbar_arrive(&rfree[(c - d) % NS]);
                q.next();
            }
            if (lane == 0) bulk_wait0();
        }
        tcgen05_fence_before();
        named_bar_sync(2, NB + G::NC);
        tcgen05_fence_after();
        if (bt < 32) tmem_dealloc<512>(tmem_base_sh);
    } else {
        // =====================================================================
        // B: y-pass ring, t-pass, recombination (x 1/||y_k||), store, reductions
        // =====================================================================
        setmaxnreg_inc<G::RB>();
        const int bt = tid - NA;
        // B thread = one column (its lane) x BR rows (BR wb .. BR wb + BR - 1);
        // u runs as row pairs (2k, 2k+1), (F u, F^2 u) as a pair per row
        const int lane = bt & 31;
        const int wb = bt >> 5;
        const float inv_alpha = a.inv_alpha;
        const bool last = a.last_group;
        // deferred normalisation: y_{k+1} = (1/||y_k||) A(y_k) (mode 1); the
        // sigmoid iterations (mode 2) normalised on load, iteration 1 has none
        const float scale = st.mode == 1 ? st.inv_f : 1.0f;

        constexpr bool TMR = G::TMR;
        constexpr bool LSU_MODE = SFK_RS_LSU != 0;
        constexpr int KR = TMR ? 1 : K;  // register ring depth
        float2 ringu[BR / 2][KR];  // u of rows (2k, 2k+1)
        float2 ringp[BR][KR];      // (F u, F^2 u) of row r
#pragma unroll
        for (int k = 0; k < KR; ++k) {
#pragma unroll
            for (int r = 0; r < BR / 2; ++r) ringu[r][k] = zero2;
#pragma unroll
            for (int r = 0; r < BR; ++r) ringp[r][k] = zero2;
        }
        // TMEM ring (TMR): slot = 3 BR words (u pairs, then (F u, F^2 u) per
        // row) in this thread's TMEM lane; warps w and w + 4 share a lane
        // quadrant and take the two column halves
        constexpr bool SPX = G::SPX;
        static_assert(!SPX || !LSU_MODE, "SPX and LSU are alternatives");
        constexpr int RW = (SPX ? 5 : 3) * BR;  // slot: u pairs, (F u, F^2 u) pairs [, S^p, F]
        constexpr int TCOLS = K * RW <= 128 ? 256 : 512;  // allocation; each warp takes half
        static_assert(!TMR || (BR == 8 && NWB == 8 && K * RW <= TCOLS / 2), "TMEM ring of one thread");
        static_assert(TMR || K <= 7, "register ring depth");
        uint32_t tm_ring = 0;
        int rslot = 0;  // TMR: ring slot of the current plane (runtime)
        if constexpr (TMR) {
            if (wb == 0) tmem_alloc<TCOLS>(&tmem_base_sh);
            tcgen05_fence_before();
            named_bar_sync(2, NB);
            tcgen05_fence_after();
            const int wq = (NWA + wb) & 3;  // CTA warp id % 4
            tm_ring = tmem_base_sh + (static_cast<uint32_t>(32 * wq) << 16) +
                      static_cast<uint32_t>((wb >> 2) * (TCOLS / 2));
        }
        auto ring_ld = [&](int slot, float2 (&lu)[BR / 2], float2 (&lp)[BR]) {
            float w[3][8];
            tmem_ld8(tm_ring + slot * RW, w[0]);
            tmem_ld8(tm_ring + slot * RW + 8, w[1]);
            tmem_ld8(tm_ring + slot * RW + 16, w[2]);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < BR / 2; ++k) lu[k] = make_float2(w[0][2 * k], w[0][2 * k + 1]);
#pragma unroll
            for (int r = 0; r < BR; ++r) lp[r] = make_float2(w[1 + r / 4][2 * (r % 4)], w[1 + r / 4][2 * (r % 4) + 1]);
        };

        // recombination operands S^p, F of this warp's BR rows: TMA, one
        // emitted plane ahead (cursor eq walks the output planes in schedule
        // order); zero-filled outside the volume, so those points come out as
        // exactly 0, add nothing to the sums, and the TMA store clips them
        constexpr bool WIDE = SFK_RS_WIDE != 0 && !TMR;
        constexpr bool WRED = WIDE && SFK_RS_WREDUCE != 0;
        static_assert(!WIDE || G::SLW == 3, "WIDE: S^p, F and y tiles");
        // WIDE: [S^p tile][F tile][y tile] of TY x TX; this warp's rows at BR wb
        float* slab = WIDE ? bsl + (BR * wb) * TX : bsl + wb * G::SLW * SLAB;
        constexpr int SLSTEP = WIDE ? TY * TX : SLAB;  // distance S^p -> F -> y rows
        uint64_t* sfull = WIDE ? &slab_full[0] : &slab_full[wb];
        PlaneStream& eq = slabq[WIDE ? 0 : wb];  // lane 0 (WIDE: thread bt == 0) only
        auto issue_slab = [&]() {
            if (eq.done) return;
            constexpr int NSL = WIDE ? TY * TX : SLAB;
            mbar_arrive_expect_tx(sfull, 2 * NSL * sizeof(float));
            const int x = eq.tile_x * TX, y = eq.tile_y * TY + (WIDE ? 0 : BR * wb),
                      t = a.out_t0 + eq.p - a.buf_t0;
            float* dst = WIDE ? bsl : slab;
            tma_load_3d(dst, &a.tm_spc, sfull, x, y, t);
            tma_load_3d(dst + NSL, &a.tm_fc[0], sfull, x, y, t);
            eq.next();
        };
        constexpr bool LSU = LSU_MODE;
        constexpr bool CPA = WIDE && SFK_RS_CPA != 0;
        PlaneStream cq;  // CPA: every B thread's cursor over the emitted planes
        auto issue_cpa = [&]() {
            if (cq.done) return;
            const int t = a.out_t0 + cq.p - a.buf_t0, x0 = cq.tile_x * TX, y0 = cq.tile_y * TY + BR * wb;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int ch = lane + 32 * j;  // 16-byte chunk: field ch / 64, row (ch % 64) / 8, float4 ch % 8
                const int fld = ch >> 6, row = (ch & 63) >> 3, c4 = ch & 7;
                const float* base = fld ? a.f[0] : a.sp;
                const bool in = y0 + row < a.H;
                const float* src =
                    in ? base + (static_cast<size_t>(t) * a.H + y0 + row) * a.pitch + x0 + 4 * c4 : base;
                cp_async16(slab + fld * SLSTEP + row * TX + 4 * c4, src, in ? 16 : 0);
            }
            cp_async_commit();
            cq.next();
        };
        if constexpr (CPA) {
            cq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
            issue_cpa();
        } else if ((WIDE ? bt == 0 : lane == 0) && !(SFK_RS_EXP & 16) && !LSU && !SPX) {
            eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
            issue_slab();
        }
        // LSU: operands of the next emitted plane in registers; one 64-bit
        // base per plane, then row increments; rows past H are predicated off
        // and columns past W read / write the pitch padding (S^p is 0 there)
        float nsp[BR], nf[BR];
        PlaneStream lq;
        const size_t rowstep = static_cast<size_t>(a.pitch);
        auto fetch = [&]() {
#pragma unroll
            for (int r = 0; r < BR; ++r) {
                nsp[r] = 0.0f;
                nf[r] = 0.0f;
            }
            if (lq.done) return;
            const int y0 = lq.tile_y * TY + BR * wb, nr = a.H - y0;
            const size_t off = (static_cast<size_t>(a.out_t0 + lq.p - a.buf_t0) * a.H + y0) * rowstep +
                               lq.tile_x * TX + lane;
            const float* ps = a.sp + off;
            const float* pf = a.f[0] + off;
#pragma unroll
            for (int r = 0; r < BR; ++r)
                if (r < nr) {
                    nsp[r] = __ldg(ps + r * rowstep);
                    nf[r] = __ldg(pf + r * rowstep);
                }
            lq.next();
        };
        if constexpr (LSU) {
            lq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
            fetch();
        }

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;   // in-volume planes consumed
        int ecnt = 0;  // output planes emitted

        // canonical reduction (device_common.cuh) of one emitted plane: BR / 4
        // blocks of 4 rows per warp, one column per lane, fp32 within a block
        constexpr bool DEFRED = SFK_RS_DEFRED != 0;
        float dv[BR];
        int d_to = 0, d_tx = 0, d_ty = 0;
        bool dpend = false;
        auto reduce_plane = [&](const float (&v)[BR], int to, int tx, int ty) {
#pragma unroll
            for (int h = 0; h < BR / 4; ++h) {
                float cs = 0.0f;
#pragma unroll
                for (int r = 0; r < 4; ++r) cs = fmaf(v[4 * h + r], v[4 * h + r], cs);
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
                const int gb = ty * G::NBANDS + (BR / 4) * wb + h;
                if (lane == 0 && gb < a.nbands && tx < a.nhalves)
                    a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves + tx] =
                        static_cast<double>(cs);
            }
            float cmax = 0.0f;
#pragma unroll
            for (int r = 0; r < BR; ++r) cmax = fmaxf(cmax, v[r]);
            const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
            if (lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
        };
        auto flush_red = [&]() {
            if (dpend) reduce_plane(dv, d_to, d_tx, d_ty);
            dpend = false;
        };

        auto plane = [&](auto slot_c) {
            constexpr int S_ = decltype(slot_c)::value;
            constexpr int SR = TMR ? 0 : S_;  // register slot of this plane
            const int slot = TMR ? rslot : S_;
            const int tg = a.out_t0 + q.p;
            const bool valid = tg >= 0 && tg < a.T;
            const bool emit = q.p - RT >= q.ta;
            const int to = tg - RT;

            // y-pass (conv3d.cpp:113-135) into this plane's ring slot
            float pso[SPX ? BR : 1], pfo[SPX ? BR : 1];  // SPX: S^p, F of this plane's points
#pragma unroll
            for (int r = 0; r < (SPX ? BR : 1); ++r) pso[r] = pfo[r] = 0.0f;
            if (valid) {
                const int b = cnt % NXB;
                if (bt == 0) SFK_T(cnt, 6);
                mbar_wait(&xb_full[b], (cnt / NXB) & 1);
                if (bt == 0) SFK_T(cnt, 7);
                if constexpr (DEFRED) flush_red();
                if constexpr (SPX) {
                    const float* xs = xb + b * XBUF + XBU + G::XBP + (BR * wb) * TXU + lane;
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        pso[r] = xs[r * TXU];
                        pfo[r] = xs[G::XBS + r * TXU];
                    }
                }
                const float* xbu = xb + b * XBUF + (BR * wb) * TXU + lane;
                const float2* xbp = reinterpret_cast<const float2*>(xb + b * XBUF + XBU + (BR * wb) * TXQ) + lane;
                if constexpr (TMR) {
                    // all BR + 2R input rows in registers first, then tap-major
                    // order: consecutive FFMA2s feed different accumulators
                    float vin[BR + 2 * R];
                    float2 pv[BR + 2 * R];
#pragma unroll
                    for (int j = 0; j < BR + 2 * R; ++j) {
                        vin[j] = xbu[j * TXU];
                        pv[j] = xbp[j * (TXQ / 2)];
                    }
#pragma unroll
                    for (int e = 0; e <= 2 * R + 1; ++e) {
#pragma unroll
                        for (int k = 0; k < BR / 2; ++k)
                            ringu[k][0] = ffma2(make_float2(vin[2 * k + e], vin[2 * k + e]), a.tpair_y[e],
                                                e == 0 ? zero2 : ringu[k][0]);
                        if (e <= 2 * R) {
#pragma unroll
                            for (int r = 0; r < BR; ++r)
                                ringp[r][0] = ffma2(pv[r + e], make_float2(a.taps_y[e], a.taps_y[e]),
                                                    e == 0 ? zero2 : ringp[r][0]);
                        }
                    }
                } else {
#pragma unroll
                for (int j = 0; j < ((SFK_RS_EXP & 2) ? 0 : BR + 2 * R); ++j) {
                    const float vin = xbu[j * TXU];
                    const float2 pv = xbp[j * (TXQ / 2)];
#pragma unroll
                    for (int k = 0; k < BR / 2; ++k) {
                        const int e = j - 2 * k;
                        if (e < 0 || e > 2 * R + 1) continue;
                        ringu[k][SR] = ffma2(make_float2(vin, vin), a.tpair_y[e], e == 0 ? zero2 : ringu[k][SR]);
                    }
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        const int d = j - r;
                        if (d < 0 || d > 2 * R) continue;
                        ringp[r][SR] = ffma2(pv, make_float2(a.taps_y[d], a.taps_y[d]), d == 0 ? zero2 : ringp[r][SR]);
                    }
                }
                }
                if (bt == 0) SFK_T(cnt, 8);
                mbar_arrive(&xb_empty[b]);
                ++cnt;
            } else {
#pragma unroll
                for (int r = 0; r < BR / 2; ++r) ringu[r][SR] = zero2;
#pragma unroll
                for (int r = 0; r < BR; ++r) ringp[r][SR] = zero2;
            }
            if (emit && !(SFK_RS_EXP & 8)) {
                // t-pass (conv3d.cpp:147-165): oldest..newest take taps_t[0..2RT]
                float2 tu[BR / 2], tp[BR];
                if constexpr (TMR) {
                    // planes oldest..newest: K - 1 TMEM slots, then this plane
                    tmem_wait_st();
#pragma unroll
                    for (int d = 0; d < K; ++d) {
                        float2 lu[BR / 2], lp[BR];
                        if (d == K - 1) {
#pragma unroll
                            for (int k = 0; k < BR / 2; ++k) lu[k] = ringu[k][0];
#pragma unroll
                            for (int r = 0; r < BR; ++r) lp[r] = ringp[r][0];
                        } else {
                            ring_ld((slot + 1 + d) % K, lu, lp);
                        }
                        const float2 w2 = make_float2(a.taps_t[d], a.taps_t[d]);
#pragma unroll
                        for (int k = 0; k < BR / 2; ++k) tu[k] = ffma2(lu[k], w2, d == 0 ? zero2 : tu[k]);
#pragma unroll
                        for (int r = 0; r < BR; ++r) tp[r] = ffma2(lp[r], w2, d == 0 ? zero2 : tp[r]);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < BR / 2; ++k) {
                        tu[k] = ffma2(ringu[k][(S_ + 1) % K], make_float2(a.taps_t[0], a.taps_t[0]), zero2);
#pragma unroll
                        for (int d = 1; d < K; ++d)
                            tu[k] = ffma2(ringu[k][(S_ + 1 + d) % K], make_float2(a.taps_t[d], a.taps_t[d]), tu[k]);
                    }
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        tp[r] = ffma2(ringp[r][(S_ + 1) % K], make_float2(a.taps_t[0], a.taps_t[0]), zero2);
#pragma unroll
                        for (int d = 1; d < K; ++d)
                            tp[r] = ffma2(ringp[r][(S_ + 1 + d) % K], make_float2(a.taps_t[d], a.taps_t[d]), tp[r]);
                    }
                }
                if (bt == 0) SFK_T(ecnt, 9);
                float spv[BR], fv[BR];
                if constexpr (SPX) {
                    // plane `to` sits RT slots after the oldest of the window
                    const int sl = (slot + 1 + RT) % K;
                    tmem_ld8(tm_ring + sl * RW + 3 * BR, spv);
                    tmem_ld8(tm_ring + sl * RW + 4 * BR, fv);
                    tmem_wait_ld();
                } else if constexpr (LSU) {
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        spv[r] = nsp[r];
                        fv[r] = nf[r];
                    }
                    fetch();  // the next emitted plane's operands
                } else if constexpr (CPA) {
                    cp_async_wait0();
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        spv[r] = slab[r * TX + lane];
                        fv[r] = slab[SLSTEP + r * TX + lane];
                    }
                    __syncwarp();
                    issue_cpa();                      // the next emitted plane's rows of this warp
                    if (bt == 0) bulk_wait_read0();  // the previous y tile store has read the staging
                    named_bar_sync(3, NB);
                } else if constexpr (WIDE) {
                    mbar_wait(sfull, ecnt & 1);
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        spv[r] = slab[r * TX + lane];
                        fv[r] = slab[SLSTEP + r * TX + lane];
                    }
                    if (bt == 0) bulk_wait_read0();  // the previous y tile store has read the staging
                    named_bar_sync(3, NB);            // every B warp has read the slab
                    if (bt == 0) {
                        fence_proxy_async();
                        issue_slab();
                    }
                } else {
                    if (!(SFK_RS_EXP & 16)) mbar_wait(sfull, ecnt & 1);
#pragma unroll
                    for (int r = 0; r < BR; ++r) {
                        spv[r] = slab[r * TX + lane];
                        fv[r] = slab[SLAB + r * TX + lane];
                    }
                    __syncwarp();
                    if (lane == 0 && !(SFK_RS_EXP & 16)) {
                        fence_proxy_async();  // the reads above before the next TMA write
                        issue_slab();
                    }
                }
                if (bt == 0) SFK_T(ecnt, 10);
                float v[BR];
#pragma unroll
                for (int r = 0; r < BR; ++r) {
                    const float tur = (r & 1) ? tu[r / 2].y : tu[r / 2].x;
                    // engine.cpp:113-119; channel sum engine.cpp:157-162
                    v[r] = A::recombine(spv[r] * scale, fv[r], inv_alpha, tur, tp[r].y, tp[r].x);
                }
                const int ox = q.tile_x * TX, oy = q.tile_y * TY + BR * wb;
                if constexpr (ACC) {  // y so far (earlier groups); rows past H read nothing
                    const int nr = a.H - oy;
                    const float* po = a.out + (static_cast<size_t>(to - a.out_buf_t0) * a.H + oy) * a.pitch + ox + lane;
#pragma unroll
                    for (int r = 0; r < BR; ++r)
                        if (r < nr && ox + lane < a.W) v[r] += po[static_cast<size_t>(r) * a.pitch];
                }
                if constexpr (LSU || SFK_RS_STG) {
                    const int nr = a.H - oy;
                    float* po = a.out + (static_cast<size_t>(to - a.out_buf_t0) * a.H + oy) * rowstep + ox + lane;
#pragma unroll
                    for (int r = 0; r < BR; ++r)
                        if (r < nr) po[r * rowstep] = v[r];
                } else if constexpr (WIDE) {
                    float* ost = slab + 2 * SLSTEP;
#pragma unroll
                    for (int r = 0; r < BR; ++r) ost[r * TX + lane] = v[r];
                    fence_proxy_async();
                    if (last && WRED) {
                        // column sums of this warp's 4-row bands and its max; the
                        // butterfly runs in one warp after the barrier
#pragma unroll
                        for (int h = 0; h < BR / 4; ++h) {
                            float cs = 0.0f;
#pragma unroll
                            for (int r = 0; r < 4; ++r) cs = fmaf(v[4 * h + r], v[4 * h + r], cs);
                            red_cols[(BR / 4) * wb + h][lane] = cs;
                        }
                        float cmax = 0.0f;
#pragma unroll
                        for (int r = 0; r < BR; ++r) cmax = fmaxf(cmax, v[r]);
                        const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                        if (lane == 0) red_max[wb] = __int_as_float(wm);
                    }
                    named_bar_sync(3, NB);
                    if (bt == 0) {
                        tma_store_3d(&a.tm_out, bsl + 2 * SLSTEP, ox, q.tile_y * TY, to - a.out_buf_t0);
                        bulk_commit();
                    }
                    if (last && WRED && wb == (ecnt % NWB)) {  // the reducing warp rotates per plane
                        if (lane < G::NBANDS) {
                            const int gb = q.tile_y * G::NBANDS + lane;
                            const float sb = tree32f(red_cols[lane]);
                            if (gb < a.nbands && q.tile_x < a.nhalves)
                                a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves + q.tile_x] =
                                    static_cast<double>(sb);
                        } else if (lane == 31) {
                            float m = 0.0f;
#pragma unroll
                            for (int w = 0; w < NWB; ++w) m = fmaxf(m, red_max[w]);
                            atomic_max_nonneg(a.frame_max + (to - a.part_t0), m);
                        }
                    }
                } else {
                    // y_{k+1} rows -> staging -> TMA store (clipped at the volume edge)
                    float* ost = slab + (G::SLW - 1) * SLAB;
                    if (lane == 0) bulk_wait_read0();  // the previous store has read the staging
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < BR; ++r) ost[r * TX + lane] = v[r];
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0 && !(SFK_RS_EXP & 16)) {
                        tma_store_3d(&a.tm_out, ost, ox, oy, to - a.out_buf_t0);
                        bulk_commit();
                    }
                }
                if (bt == 0) SFK_T(ecnt, 11);
                // time-sharded solve: the edge planes of this rank also go
                // straight into the neighbours' halo frames (peer memory,
                // coalesced 128-byte rows; rows past H are not written)
                if (PEER && last) {
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        float* pb = a.peer[side];
                        const bool edge = side == 0 ? to < a.out_t0 + a.peer_n : to >= a.out_t1 - a.peer_n;
                        if (!pb || !edge) continue;
                        const int oy = q.tile_y * TY + BR * wb, nr = a.H - oy;
                        float* po = pb + (static_cast<size_t>(to - a.peer_t0[side]) * a.H + oy) * a.pitch +
                                    q.tile_x * TX + lane;
#pragma unroll
                        for (int r = 0; r < BR; ++r)
                            if (r < nr) po[static_cast<size_t>(r) * a.pitch] = v[r];
                    }
                }
                ++ecnt;
                if (last && !WRED) {
                    if constexpr (DEFRED) {
                        flush_red();
#pragma unroll
                        for (int r = 0; r < BR; ++r) dv[r] = v[r];
                        d_to = to;
                        d_tx = q.tile_x;
                        d_ty = q.tile_y;
                        dpend = true;
                    } else if (!(SFK_RS_EXP & 32)) {
                        reduce_plane(v, to, q.tile_x, q.tile_y);
                    }
                }
            }
            if constexpr (TMR) {
                // this plane into slot S_ (it held a plane no longer needed)
                float w[8];
#pragma unroll
                for (int k = 0; k < BR / 2; ++k) {
                    w[2 * k] = ringu[k][0].x;
                    w[2 * k + 1] = ringu[k][0].y;
                }
                tmem_st8(tm_ring + slot * RW, w);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        w[2 * r] = ringp[4 * h + r][0].x;
                        w[2 * r + 1] = ringp[4 * h + r][0].y;
                    }
                    tmem_st8(tm_ring + slot * RW + 8 + 8 * h, w);
                }
                if constexpr (SPX) {
                    tmem_st8(tm_ring + slot * RW + 3 * BR, pso);
                    tmem_st8(tm_ring + slot * RW + 4 * BR, pfo);
                }
                rslot = rslot + 1 == K ? 0 : rslot + 1;
            }
            q.next();
        };
        using std::integral_constant;
        if constexpr (TMR) {
            while (!q.done) plane(integral_constant<int, 0>{});  // runtime slots
        } else while (!q.done) {
            plane(integral_constant<int, 0>{});
            if constexpr (K > 1) { if (q.done) break; plane(integral_constant<int, (K > 1 ? 1 : 0)>{}); }
            if constexpr (K > 2) { if (q.done) break; plane(integral_constant<int, (K > 2 ? 2 : 0)>{}); }
            if constexpr (K > 3) { if (q.done) break; plane(integral_constant<int, (K > 3 ? 3 : 0)>{}); }
            if constexpr (K > 4) { if (q.done) break; plane(integral_constant<int, (K > 4 ? 4 : 0)>{}); }
            if constexpr (K > 5) { if (q.done) break; plane(integral_constant<int, (K > 5 ? 5 : 0)>{}); }
            if constexpr (K > 6) { if (q.done) break; plane(integral_constant<int, (K > 6 ? 6 : 0)>{}); }
        }
        flush_red();
        if (lane == 0) bulk_wait0();  // the output rows are written before the CTA exits
        if constexpr (TMR) {
            tmem_wait_st();
            tcgen05_fence_before();
            named_bar_sync(2, NB);
            tcgen05_fence_after();
            if (wb == 0) tmem_dealloc<TCOLS>(tmem_base_sh);
        }
    }
}

}  // namespace sfk
