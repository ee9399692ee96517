// fused_mc.cuh — SFSeg power-iteration step for several feature channels,
// FAST arithmetic, in the (C + 2)-field form.
//
// Summing the per-channel recombination (engine.cpp:107-120) over the
// channels (engine.cpp:157-162) and using the linearity of the separable
// convolution G (conv3d.cpp:171-185) gives
//
//   sum_c X_c = S^p [ (C/alpha - Q) G(u) - G(Q u) + 2 sum_c f_c G(f_c u) ],
//   u = S^p x,  Q = sum_c f_c^2  (static: computed once per solve),
//
// so a step needs C + 2 convolved fields instead of the 1 + 2C of the
// per-channel form (c2, C = 8: 10 fields instead of 24; c4, C = 3: 5 instead
// of 9). All of them in one pass would need a t-pass ring of
// (2 RT + 1) x (C + 2) planes per output tile (c4: 368 KB for a 64 x 32 tile),
// more than the 256 KB of tensor memory, so the fields run in groups, each a
// single pass over the volume:
//
//   HEAD (first launch, NF = 2 or 3): raw boxes U, Q [, f_1]; fields u, Q u
//        [, f_1 u]; y = S^p ((C/alpha - Q) G(u) - G(Q u) [+ 2 f_1 G(f_1 u)])
//   TAIL (later launches, NF = 2; NF = 1 compiles but no grouping needs it): raw boxes U, f_a [, f_b]; fields
//        f_a u [, f_b u]; y += 2 S^p (f_a G(f_a u) + f_b G(f_b u))
//
// c4 (C = 3) is HEAD(3) + TAIL(2): two passes per iteration. An even channel
// count runs HEAD(2) + C/2 TAIL(2) (c2, C = 8: five passes, none of them a
// one-channel TAIL).
//
// U = S^p x is the u field itself. The last launch of a step writes, instead
// of y_{k+1}, U_{k+1} = S^p y_{k+1} (write_u) whenever the next iteration
// only normalises (FAST defers the 1/||y|| to the output, so u_{k+1} is
// exactly S^p y_{k+1}): the next step then reads one box (U) where it would
// read two (x, S^p), and HBM sees the same bytes per iteration. The first
// iteration, a sigmoid iteration (which needs the reduction first) and the
// last iteration of a solve (the caller reads y) go through y and k_make_u.
//
// The schedule, roles and pipeline are those of fused_step_rs (fused_rs.cuh)
// with its t-pass ring in tensor memory: one 512-thread CTA per SM walking
// (64 x 32 tile, frame range) segments; 8 A warps issue the halo-box TMA loads
// and run the x-pass with the products formed in registers; 8 B warps run the
// y-pass into a TMEM ring of the last 2RT+1 planes, the t-pass, the
// recombination (x 1/||y_k||, deferred as in FAST), the TMA store and, in the
// last launch, the canonical reductions. Every field is one "single" slot:
// two neighbouring outputs take one input with one FFMA2 and a tap pair
// (w[e], w[e-1]) — columns in the x-pass, rows in the y-pass.
//
// KIND 2 (EXACT, one launch per channel, the reference's own 1 + 2C form):
// boxes x, S^p, f; fields u, f u, (f f) u evaluated left to right
// (engine.cpp:92-100); every product and sum separately rounded in the
// reference's tap order (conv3d.cpp:88-165: paired FFMA2 with runtime
// zero / one operands, so no contraction), the normalisation and sigmoid
// applied on load in fp64 (engine.cpp:178, 196-203), the recombination and
// channel sum of engine.cpp:113-119, 157-162, and fp64 canonical reductions.
// A step is bit-identical to the reference's sfseg_step at the radii the
// warp-specialised EXACT kernel (fused_ws.cuh) has no room for (c2, c4).
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "step_common.cuh"  // PlaneStream, Arith, ffma2, canonical_tree32
#include "sfseg_types.cuh"


// ring slots fetched per tcgen05.wait::ld in the t-pass
#ifndef SFK_MC_TB
#define SFK_MC_TB 1
#endif

namespace sfk {

enum McKind { MC_HEAD = 0, MC_TAIL = 1, MC_EXACT = 2 };

template <int RT, int R, int NF, int KIND>
struct McGeom {
    static constexpr bool HEAD = KIND == MC_HEAD, EXACT = KIND == MC_EXACT;
    static constexpr int TY = 64, TX = 32, BR = 8, NWA = 8, NWB = TY / BR, STAGES = 2;
    static constexpr int NA = 32 * NWA, NB = 32 * NWB, NT = NA + NB;
    static constexpr int K = 2 * RT + 1;
    static constexpr int BH = TY + 2 * R;
    static constexpr int HX = (R + 3) / 4 * 4;  // left halo (16-byte aligned box start)
    static constexpr int HR = ((TX + HX + HX) / 4) % 2 == 1 ? HX : HX + 4;  // odd float4 rows
    static constexpr int BW = TX + HX + HR, BW4 = BW / 4;
    static constexpr int XOFF = HX - R;
    static constexpr int FB = (BH * BW + 31) / 32 * 32;
    // raw boxes: HEAD U, Q [, f_1]; TAIL U, f_a [, f_b]; EXACT x, S^p, f
    static constexpr int NR = EXACT ? 3 : HEAD ? NF : NF + 1;
    static constexpr int SW = 8;
    static constexpr int NINX = SW + 2 * R;
    static constexpr int NLD = (XOFF + NINX + 3) / 4;
    static constexpr int RBLK = (BH + 7) / 8;
    static constexpr int XPASS = (RBLK + NWA - 1) / NWA;
    static constexpr int TXU = TX + 4;
    static constexpr int XBU = (BH * TXU + 31) / 32 * 32;  // one field of the x-pass output
    static constexpr int NXB = 2;
    // recombination operands (TMA slabs, one emitted plane ahead): S^p, Q
    // [, f_1] | S^p, f_a [, f_b], y of the earlier launches
    // (EXACT: S^p, f, y of the earlier channels)
    static constexpr int NOP = HEAD ? NF : EXACT ? 3 : NF + 2;
    static constexpr int NFC = HEAD ? NF - 1 : EXACT ? 1 : NF;  // channel-type slabs after S^p
    static constexpr int SLAB = BR * TX;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NR * FB;
    static constexpr size_t XB_FLOATS = size_t(NXB) * NF * XBU;
    static constexpr size_t SL_FLOATS = size_t(NWB) * (NOP + 1) * SLAB;  // + y staging
    static constexpr int NBAR = STAGES + 2 * NXB + NWB;
    static constexpr size_t SMEM_BYTES = (RAW_FLOATS + XB_FLOATS + SL_FLOATS) * sizeof(float) + NBAR * 8;
    static constexpr int NBANDS = TY / 4;
    // TMEM ring: slot = NF x BR words (row pairs of each field) per thread;
    // warps w and w + 4 share a lane quadrant and take half the columns each
    static constexpr int RW = NF * BR;
    static constexpr int TCOLS = K * RW <= 128 ? 256 : 512;
    static constexpr int RA = EXACT ? 72 : 64;  // EXACT: three fields + separate roundings
    // setmaxnreg: every warp starts with the launch grant RPOOL (65536 / NT,
    // multiple of 8); an SMSP holds NWA / 4 A and NWB / 4 B warps, and B can
    // take only what A gives back (asking for more blocks forever)
    static constexpr int RPOOL = (65536 / NT) / 8 * 8 > 255 ? 248 : (65536 / NT) / 8 * 8;
    static constexpr int RB_ = ((NWA / 4 + NWB / 4) * RPOOL - (NWA / 4) * RA) / (NWB / 4) / 8 * 8;
    static constexpr int RB = RB_ > 248 ? 248 : RB_;
    static_assert(BW4 % 2 == 1, "odd float4 box rows (conflict-free strip reads)");
    static_assert((TXU / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert(K * RW <= TCOLS / 2, "TMEM ring of one thread");
    static_assert(EXACT ? NF == 3 : HEAD ? (NF == 2 || NF == 3) : (NF == 1 || NF == 2), "field groups");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
    static_assert(NWA % 4 == 0 && NWB % 4 == 0, "setmaxnreg acts on whole warpgroups");
};

template <int RT, int R, int NF, int KIND>
__global__ void __launch_bounds__(McGeom<RT, R, NF, KIND>::NT, 1)
    fused_step_mc(const __grid_constant__ FusedArgs a) {
    using G = McGeom<RT, R, NF, KIND>;
    constexpr bool HEAD = G::HEAD, EXACT = G::EXACT;
    using A = Arith<!EXACT>;
    constexpr int BR = G::BR, TY = G::TY, TX = G::TX, NA = G::NA, NB = G::NB, K = G::K, NWB = G::NWB;
    constexpr int BH = G::BH, BW = G::BW, FB = G::FB, BW4 = G::BW4, SW = G::SW, NR = G::NR;
    constexpr int TXU = G::TXU, XBU = G::XBU, SLAB = G::SLAB, NXB = G::NXB, STAGES = G::STAGES;
    constexpr int NOP = G::NOP, RW = G::RW;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                // [STAGES][NR][FB]
    float* xb = raw + G::RAW_FLOATS;  // [NXB][NF][XBU]
    float* bsl = xb + G::XB_FLOATS;   // [NWB][NOP + 1][BR][TX]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(bsl + G::SL_FLOATS);
    uint64_t* raw_full = mbar;                      // [STAGES]
    uint64_t* xb_full = mbar + STAGES;              // [NXB] (count NA)
    uint64_t* xb_empty = mbar + STAGES + NXB;       // [NXB] (count NB)
    uint64_t* slab_full = mbar + STAGES + 2 * NXB;  // [NWB]

    __shared__ IterState st;
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x;
    griddep_wait();  // PDL: the previous step / finalize has completed
    // an earlier iteration hit a zero norm, or the early-exit rule already held
    if (a.st->degenerate || a.st->stop) return;
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
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        if (EXACT) prefetch_tensormap(&a.tm_sp);
        prefetch_tensormap(&a.tm_f[0]);
        prefetch_tensormap(&a.tm_out);
        prefetch_tensormap(&a.tm_spc);
        prefetch_tensormap(&a.tm_fc[0]);
    }
    __syncthreads();
    const float2 zero2 = make_float2(0.0f, 0.0f);
    // EXACT: p = w x + 0 and acc = acc * 1 + p with run-time 0 / 1, so every
    // product and every sum is rounded on its own (no FMA contraction)
    const float2 zr2 = make_float2(a.zero, a.zero), one2 = make_float2(a.one, a.one);
    auto acc2 = [&](float2 acc, float2 x, float2 w, bool first) {
        if constexpr (EXACT) {
            const float2 pr = ffma2(x, w, zr2);
            return first ? pr : ffma2(acc, one2, pr);
        } else {
            return ffma2(x, w, first ? zero2 : acc);
        }
    };

    if (tid < NA) {
        // =====================================================================
        // A: TMA producer + x-pass (conv3d.cpp:88-101) with in-register products
        // =====================================================================
        setmaxnreg_dec<G::RA>();
        // box `pbox` (0 .. NR-1) of every plane is issued by lane 0 of warp
        // NWA - NR + pbox with its own plane cursor (warp 0 runs two x-pass
        // blocks; one issuer for all boxes costs ~1000 cycles per plane,
        // fused_rs.cuh SFK_RS_PSPLIT); box 0 carries the expect_tx of all
        const int pbox = (tid >> 5) - (G::NWA - NR);
        const bool pissuer = (tid & 31) == 0 && pbox >= 0;
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
            float* dst = raw + static_cast<size_t>(s) * NR * FB + pbox * FB;
            uint64_t* bar = &raw_full[s];
            const int bx = pq.tile_x * TX - G::HX, by = pq.tile_y * TY - R, bt = tg - a.buf_t0;
            if (pbox == 0) mbar_arrive_expect_tx(bar, NR * BH * BW * sizeof(float));
            const CUtensorMap* map = pbox == 0 ? &a.tm_x : EXACT ? (pbox == 1 ? &a.tm_sp : &a.tm_f[0])
                                                                 : &a.tm_f[pbox - 1];
            tma_load_3d(dst, map, bar, bx, by, bt);
            ++pcount;
            pq.next();
        };
        if (pissuer) {
            pq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            for (int s = 0; s < STAGES; ++s) issue_box();
        }
        // FAST reads U = S^p T(x) (k_make_u or the previous step's write_u)
        const bool sigm = EXACT && st.mode == 2;
        const bool norm = EXACT && st.mode == 1;  // EXACT normalises on load
        const int xw = tid >> 5, xl = tid & 31;  // lane -> (row xl & 7, strip xl >> 3)

        // one x-pass item: box row r, strip sx (SW outputs as column pairs)
        auto item = [&](auto sig_c, const float* rs, float* xbb, int r, int sx) {
            [[maybe_unused]] constexpr bool SIG = decltype(sig_c)::value == 2;
            [[maybe_unused]] constexpr bool NRM = decltype(sig_c)::value == 1;
            const float4* py = reinterpret_cast<const float4*>(rs) + r * BW4 + 2 * sx;
            float2 ou[NF][SW / 2];
            float4 v[NR];
#pragma unroll
            for (int m4 = 0; m4 < G::NLD * 4; ++m4) {
                if (m4 % 4 == 0) {
#pragma unroll
                    for (int i = 0; i < NR; ++i) v[i] = py[i * (FB / 4) + m4 / 4];
                }
                const int m = m4 - G::XOFF;
                if (m < 0 || m >= G::NINX) continue;
                const int c = m4 % 4;
                float e4[NR];
#pragma unroll
                for (int i = 0; i < NR; ++i) e4[i] = c == 0 ? v[i].x : c == 1 ? v[i].y : c == 2 ? v[i].z : v[i].w;
                float phi[NF];
                if constexpr (EXACT) {
                    const float x = SIG ? A::load_sigmoid(e4[0], st)
                                        : NRM ? A::load_norm(e4[0], st.inv, st.inv_f) : e4[0];
                    const float u = xmul(e4[1], x);  // engine.cpp:92-98, left to right
                    phi[0] = u;
                    phi[1] = xmul(e4[2], u);
                    phi[2] = xmul(xmul(e4[2], e4[2]), u);
                } else if constexpr (HEAD) {
                    const float u = e4[0];  // U = S^p x (engine.cpp:92-100)
                    phi[0] = u;
                    phi[1] = e4[1] * u;  // Q u
                    if constexpr (NF > 2) phi[2] = e4[2] * u;  // f_1 u
                } else {
#pragma unroll
                    for (int i = 0; i < NF; ++i) phi[i] = e4[1 + i] * e4[0];  // f_i u
                }
#pragma unroll
                for (int i = 0; i < NF; ++i) {
#pragma unroll
                    for (int k = 0; k < SW / 2; ++k) {
                        const int e = m - 2 * k;
                        if (e < 0 || e > 2 * R + 1) continue;
                        // x-pass starts from acc = 0 (conv3d.cpp:92): 0 + p = p
                        if constexpr (!EXACT) {
                            // the pair's two edge taps have a zero partner
                            // (w[-1], w[2R+1]): one scalar op instead of FFMA2
                            if (e == 0) {
                                ou[i][k] = make_float2(phi[i] * a.taps_x[0], 0.0f);
                                continue;
                            }
                            if (e == 2 * R + 1) {
                                ou[i][k].y = fmaf(phi[i], a.taps_x[2 * R], ou[i][k].y);
                                continue;
                            }
                        }
                        ou[i][k] = acc2(ou[i][k], make_float2(phi[i], phi[i]), a.tpair_x[e], e == 0);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < NF; ++i) {
                float4* du = reinterpret_cast<float4*>(xbb + i * XBU + r * TXU + sx * SW);
#pragma unroll
                for (int w = 0; w < SW / 4; ++w)
                    du[w] = make_float4(ou[i][2 * w].x, ou[i][2 * w].y, ou[i][2 * w + 1].x, ou[i][2 * w + 1].y);
            }
        };

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;
        for (; !q.done; q.next()) {
            const int tg = a.out_t0 + q.p;
            if (tg < 0 || tg >= a.T) continue;  // planes outside the volume: B zero-fills
            const int s = cnt % STAGES;
            const int b = cnt % NXB;
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            mbar_wait(&xb_empty[b], ((cnt / NXB) & 1) ^ 1);
            const float* rs = raw + static_cast<size_t>(s) * NR * FB;
            float* xbb = xb + static_cast<size_t>(b) * NF * XBU;
#pragma unroll
            for (int k = 0; k < G::XPASS; ++k) {
                const int blk = xw + k * G::NWA;
                if (blk >= G::RBLK) break;
                const int r = blk * 8 + (xl & 7);
                if (r >= BH) continue;
                using L0 = std::integral_constant<int, 0>;
                using L1 = std::integral_constant<int, 1>;
                using L2 = std::integral_constant<int, 2>;
                if (EXACT && sigm)
                    item(L2{}, rs, xbb, r, xl >> 3);
                else if (EXACT && norm)
                    item(L1{}, rs, xbb, r, xl >> 3);
                else
                    item(L0{}, rs, xbb, r, xl >> 3);
            }
            mbar_arrive(&xb_full[b]);  // release: this thread's x-pass stores
            named_bar_sync(1, NA);     // raw stage s fully read
            if (pissuer) {
                fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_box();
            }
            ++cnt;
        }
    } else {
        // =====================================================================
        // B: y-pass into the TMEM ring, t-pass, recombination, store, reductions
        // =====================================================================
        setmaxnreg_inc<G::RB>();
        const int bt = tid - NA;
        const int lane = bt & 31;
        const int wb = bt >> 5;
        const bool last = a.last_group;
        // deferred 1/||y_k|| (FAST; EXACT normalised on load)
        const float scale = (!EXACT && st.mode == 1) ? st.inv_f : 1.0f;
        const bool first = a.first_group;  // EXACT: no earlier channel to add
        constexpr int TCOLS = G::TCOLS;
        if (wb == 0) tmem_alloc<TCOLS>(&tmem_base_sh);
        tcgen05_fence_before();
        named_bar_sync(2, NB);
        tcgen05_fence_after();
        const int wq = (G::NWA + wb) & 3;  // CTA warp id % 4
        const uint32_t tm_ring = tmem_base_sh + (static_cast<uint32_t>(32 * wq) << 16) +
                                 static_cast<uint32_t>((wb >> 2) * (TCOLS / 2));

        float* slab = bsl + static_cast<size_t>(wb) * (NOP + 1) * SLAB;
        uint64_t* sfull = &slab_full[wb];
        // operands of output plane `tout` (global frame) of tile (tx, ty)
        auto issue_slab = [&](int tx, int ty, int tout) {
            const bool yprev = !HEAD && !(EXACT && first);
            mbar_arrive_expect_tx(sfull, (yprev ? NOP : NOP - (HEAD ? 0 : 1)) * SLAB * sizeof(float));
            const int x = tx * TX, y = ty * TY + BR * wb, t = tout - a.buf_t0;
            tma_load_3d(slab, &a.tm_spc, sfull, x, y, t);
#pragma unroll
            for (int i = 0; i < G::NFC; ++i)
                tma_load_3d(slab + (1 + i) * SLAB, &a.tm_fc[i], sfull, x, y, t);
            if (yprev)  // y so far: written by the previous launch (stream order)
                tma_load_3d(slab + (NOP - 1) * SLAB, &a.tm_out, sfull, x, y, t + a.buf_t0 - a.out_buf_t0);
        };

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        // the first output plane's operands; every emitted plane then fetches
        // the next one's: the following frame of the segment, or the first
        // frame of the next segment (no second plane cursor: the issue sits on
        // every B warp's chain)
        if (lane == 0 && !q.done) issue_slab(q.tile_x, q.tile_y, a.out_t0 + q.ta);
        int cnt = 0, ecnt = 0, rslot = 0;
        while (!q.done) {
            const int tg = a.out_t0 + q.p;
            const bool valid = tg >= 0 && tg < a.T;
            const bool emit = q.p - RT >= q.ta;
            const int to = tg - RT;
            float2 cur[NF][BR / 2];  // y-pass output of this plane, row pairs
            if (valid) {
                // y-pass (conv3d.cpp:113-135): rows BR wb .. + BR - 1 of column `lane`
                const int b = cnt % NXB;
                mbar_wait(&xb_full[b], (cnt / NXB) & 1);
#pragma unroll
                for (int i = 0; i < NF; ++i) {
                    const float* xc = xb + (static_cast<size_t>(b) * NF + i) * XBU + (BR * wb) * TXU + lane;
                    float vin[BR + 2 * R];
#pragma unroll
                    for (int j = 0; j < BR + 2 * R; ++j) vin[j] = xc[j * TXU];
#pragma unroll
                    for (int e = 0; e <= 2 * R + 1; ++e) {
#pragma unroll
                        for (int k = 0; k < BR / 2; ++k) {
                            const float vv = vin[2 * k + e];
                            if constexpr (!EXACT) {  // zero-partner edge taps as scalar ops
                                if (e == 0) {
                                    cur[i][k] = make_float2(vv * a.taps_y[0], 0.0f);
                                    continue;
                                }
                                if (e == 2 * R + 1) {
                                    cur[i][k].y = fmaf(vv, a.taps_y[2 * R], cur[i][k].y);
                                    continue;
                                }
                            }
                            cur[i][k] = acc2(cur[i][k], make_float2(vv, vv), a.tpair_y[e], e == 0);
                        }
                    }
                }
                mbar_arrive(&xb_empty[b]);
                ++cnt;
            } else {
#pragma unroll
                for (int i = 0; i < NF; ++i)
#pragma unroll
                    for (int k = 0; k < BR / 2; ++k) cur[i][k] = zero2;
            }
            if (emit) {
                // t-pass (conv3d.cpp:147-165): K - 1 ring slots (oldest first), then this plane
                float2 tacc[NF][BR / 2];
                tmem_wait_st();
                constexpr int TB = SFK_MC_TB;  // ring slots per tcgen05.wait::ld
#pragma unroll
                for (int d0 = 0; d0 < K; d0 += TB) {
                    float w[TB][NF][8];
#pragma unroll
                    for (int j = 0; j < TB; ++j) {
                        const int d = d0 + j;
                        if (d >= K - 1) continue;
                        int sl = rslot + 1 + d;
                        sl = sl >= K ? sl - K : sl;
#pragma unroll
                        for (int i = 0; i < NF; ++i) tmem_ld8(tm_ring + sl * RW + 8 * i, w[j][i]);
                    }
                    if (d0 < K - 1) tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < TB; ++j) {
                        const int d = d0 + j;
                        if (d >= K) continue;
                        const float2 w2 = make_float2(a.taps_t[d], a.taps_t[d]);
#pragma unroll
                        for (int i = 0; i < NF; ++i)
#pragma unroll
                            for (int k = 0; k < BR / 2; ++k) {
                                const float2 lu = d == K - 1
                                                      ? cur[i][k]
                                                      : make_float2(w[j][i][2 * k], w[j][i][2 * k + 1]);
                                tacc[i][k] = acc2(tacc[i][k], lu, w2, d == 0);
                            }
                    }
                }
                mbar_wait(sfull, ecnt & 1);
                float opv[NOP][BR];
#pragma unroll
                for (int o = 0; o < NOP; ++o)
#pragma unroll
                    for (int r = 0; r < BR; ++r) opv[o][r] = slab[o * SLAB + r * TX + lane];
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async();  // the reads above before the next TMA write
                    if (q.p + 1 < q.tb + RT) {
                        issue_slab(q.tile_x, q.tile_y, to + 1);
                    } else if (q.i + 1 < q.n) {
                        const int4 sg = q.seg[q.i + 1];
                        const int ny = sg.x / q.tiles_x;
                        issue_slab(sg.x - ny * q.tiles_x, ny, a.out_t0 + sg.y);
                    }
                }
                const int ox = q.tile_x * TX, oy = q.tile_y * TY + BR * wb;
                float v[BR];
#pragma unroll
                for (int r = 0; r < BR; ++r) {
                    float g[NF];
#pragma unroll
                    for (int i = 0; i < NF; ++i) g[i] = (r & 1) ? tacc[i][r / 2].y : tacc[i][r / 2].x;
                    if constexpr (EXACT) {
                        // engine.cpp:113-119 (u, F u, F^2 u convolved), channel sum :157-162
                        const float term = A::recombine(opv[0][r], opv[1][r], a.inv_alpha, g[0], g[2], g[1]);
                        v[r] = first ? term : xadd(opv[2][r], term);
                    } else if constexpr (HEAD) {
                        // S^p ((C/alpha - Q) G(u) - G(Q u) [+ 2 f_1 G(f_1 u)])
                        float h = (a.c_inv_alpha - opv[1][r]) * g[0] - g[1];
                        if constexpr (NF > 2) h = fmaf(2.0f * opv[2][r], g[2], h);
                        v[r] = (opv[0][r] * scale) * h;
                    } else {
                        // 2 S^p sum_i f_i G(f_i u)
                        float sfg = opv[1][r] * g[0];
                        if constexpr (NF > 1) sfg = fmaf(opv[2][r], g[1], sfg);
                        v[r] = (2.0f * opv[0][r] * scale) * sfg;
                    }
                }
                if constexpr (KIND == MC_TAIL) {  // y of the earlier launches (zero-filled past the edge)
#pragma unroll
                    for (int r = 0; r < BR; ++r) v[r] += opv[NOP - 1][r];
                }
                // y_{k+1} rows (or U_{k+1} = S^p y_{k+1}) -> staging -> TMA
                // store (clipped at the volume edge)
                float* ost = slab + NOP * SLAB;
                if (lane == 0) bulk_wait_read0();  // the previous store has read the staging
                __syncwarp();
                const bool wu = !EXACT && last && a.write_u;
#pragma unroll
                for (int r = 0; r < BR; ++r) ost[r * TX + lane] = wu ? opv[0][r] * v[r] : v[r];
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&a.tm_out, ost, ox, oy, to - a.out_buf_t0);
                    bulk_commit();
                }
                ++ecnt;
                if (last) {  // launch-uniform: the earlier launches of a step skip it
                    // canonical reduction (device_common.cuh): 4-row blocks, column
                    // sums (fp32 in FAST, fp64 in EXACT as fused_ws.cuh), xor-butterfly
                    // over the 32 columns. The warp's two blocks share one butterfly:
                    // after the first exchange lanes 0-15 hold block 0's pair sums
                    // c_i + c_{i+16} and lanes 16-31 block 1's — the values the
                    // per-block xor-16 step leaves there — and the xor 8, 4, 2, 1
                    // steps stay inside each half: same bits, half the shuffles.
                    static_assert(BR == 8, "two 4-row blocks per warp");
                    using RT_ = std::conditional_t<EXACT, double, float>;
                    RT_ cs0 = 0, cs1 = 0;
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        cs0 += static_cast<RT_>(v[r]) * static_cast<RT_>(v[r]);
                        cs1 += static_cast<RT_>(v[4 + r]) * static_cast<RT_>(v[4 + r]);
                    }
                    const bool lo = lane < 16;
                    RT_ cs = (lo ? cs0 : cs1) + __shfl_xor_sync(0xffffffffu, lo ? cs1 : cs0, 16);
#pragma unroll
                    for (int o = 8; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
                    float cmax = 0.0f;
#pragma unroll
                    for (int r = 0; r < BR; ++r) cmax = fmaxf(cmax, v[r]);
                    const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
                    const int gb = q.tile_y * G::NBANDS + (BR / 4) * wb + (lo ? 0 : 1);
                    if ((lane & 15) == 0 && gb < a.nbands && q.tile_x < a.nhalves)
                        a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves + q.tile_x] =
                            static_cast<double>(cs);
                    if (lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
                }
            }
            // this plane into ring slot rslot (it held a plane no longer needed)
#pragma unroll
            for (int i = 0; i < NF; ++i) {
                float w[8];
#pragma unroll
                for (int k = 0; k < BR / 2; ++k) {
                    w[2 * k] = cur[i][k].x;
                    w[2 * k + 1] = cur[i][k].y;
                }
                tmem_st8(tm_ring + rslot * RW + 8 * i, w);
            }
            rslot = rslot + 1 == K ? 0 : rslot + 1;
            q.next();
        }
        if (lane == 0) bulk_wait0();  // the output rows are written before the CTA exits
        tmem_wait_st();
        tcgen05_fence_before();
        named_bar_sync(2, NB);
        tcgen05_fence_after();
        if (wb == 0) tmem_dealloc<TCOLS>(tmem_base_sh);
    }
}

}  // namespace sfk
