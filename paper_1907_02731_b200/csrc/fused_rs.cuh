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
#include "fused_step.cuh"  // PlaneStream, Arith, ffma2
#include "sfseg_types.cuh"

#ifndef SFK_RS_EXP
#define SFK_RS_EXP 0
#endif

namespace sfk {

template <int RT, int R, int NWA, int STAGES>
struct RsGeom {
    static constexpr int TY = 64, TX = 32;
    static constexpr int NA = 32 * NWA, NB = 256, NT = NA + NB;
    static constexpr int NWB = NB / 32;
    static constexpr int K = 2 * RT + 1;
    static constexpr int BH = TY + 2 * R;
    // x halos: the box must start on a 16-byte boundary (TMA faults on an
    // unaligned innermost coordinate), so the left halo HX is R rounded up to
    // whole float4s; the right halo HR >= R is chosen so the row is an odd
    // number of float4s, which makes float4 reads of 8 rows at one strip
    // conflict-free
    static constexpr int HX = (R + 3) / 4 * 4;
    static constexpr int HR = ((TX + HX + (R + 3) / 4 * 4) / 4) % 2 == 1 ? (R + 3) / 4 * 4 : (R + 3) / 4 * 4 + 4;
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
    static constexpr int XBUF = XBU + XBP;
    static constexpr int NBANDS = TY / 4;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
    static constexpr size_t XB_FLOATS = 2 * size_t(XBUF);
    static constexpr size_t SMEM_BYTES = (RAW_FLOATS + XB_FLOATS) * sizeof(float) + 256;
    // setmaxnreg budgets: warp w runs on SMSP w % 4 and each SMSP has 512
    // registers per lane slot; the fullest SMSP bounds the budgets
    static constexpr int WA_MAX = (NWA + 3) / 4;            // A warps on the fullest SMSP
#ifndef SFK_RS_RA
#define SFK_RS_RA 64
#endif
    static constexpr int RA = SFK_RS_RA;
    static constexpr int WMAX = (NWA + NWB + 3) / 4;
    // B warps NWA..NWA+7: SMSPs hold WA_s A warps and WB_s B warps; take the
    // tightest SMSP
    static constexpr int rb_for(int s) {
        const int wa = NWA / 4 + (s < NWA % 4 ? 1 : 0);
        int wb = 0;
        for (int w = NWA; w < NWA + NWB; ++w) wb += (w % 4 == s) ? 1 : 0;
        return wb ? (512 - wa * RA) / wb : 512;
    }
    static constexpr int RB_RAW = rb_for(0) < rb_for(1) ? (rb_for(0) < rb_for(2) ? (rb_for(0) < rb_for(3) ? rb_for(0) : rb_for(3)) : (rb_for(2) < rb_for(3) ? rb_for(2) : rb_for(3)))
                                                        : (rb_for(1) < rb_for(2) ? (rb_for(1) < rb_for(3) ? rb_for(1) : rb_for(3)) : (rb_for(2) < rb_for(3) ? rb_for(2) : rb_for(3)));
    static constexpr int RPOOL = (65536 / NT) / 8 * 8;  // launch grant per thread
    static constexpr int RB_POOL = (NT * RPOOL - NA * RA) / NB;
    static constexpr int RB_MIN = RB_RAW < RB_POOL ? RB_RAW : RB_POOL;
    static constexpr int RB = (RB_MIN < 248 ? RB_MIN : 248) / 8 * 8;
    static_assert(BW4 % 2 == 1, "odd float4 box rows");
    static_assert((TXU / 4) % 2 == 1 && (TXQ / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert(RA <= RPOOL && RB >= RPOOL, "setmaxnreg: A gives, B takes");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

template <int RT, int R, int NWA, int STAGES, bool ACC>
__global__ void __launch_bounds__(32 * NWA + 256, 1) fused_step_rs(const __grid_constant__ FusedArgs a) {
    using G = RsGeom<RT, R, NWA, STAGES>;
    using A = Arith<true>;
    constexpr int TY = G::TY, TX = G::TX, NA = G::NA, NB = G::NB, K = G::K;
    constexpr int BH = G::BH, BW = G::BW, FB = G::FB, BW4 = G::BW4;
    constexpr int TXU = G::TXU, TXQ = G::TXQ, XBU = G::XBU, XBUF = G::XBUF;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                   // [STAGES][3][FB]   TMA boxes
    float* xb = raw + G::RAW_FLOATS;     // [2][XBUF]         x-pass output
    uint64_t* mbar = reinterpret_cast<uint64_t*>(xb + G::XB_FLOATS);
    uint64_t* raw_full = mbar;               // [STAGES]  TMA -> A
    uint64_t* xb_full = mbar + STAGES;       // [2]       A -> B (count NA)
    uint64_t* xb_empty = mbar + STAGES + 2;  // [2]       B -> A (count NB)

    __shared__ IterState st;
    __shared__ PlaneStream prodq;
    __shared__ int prod_count;

    const int tid = threadIdx.x;
    if (a.st->degenerate) return;  // an earlier iteration hit a zero norm
    const int s0 = a.sched_off[blockIdx.x], s1 = a.sched_off[blockIdx.x + 1];
    if (s0 >= s1) return;

    if (tid == 0) {
        st = *a.st;
        for (int s = 0; s < STAGES; ++s) mbar_init(&raw_full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xb_full[b], NA);
            mbar_init(&xb_empty[b], NB);
        }
        fence_barrier_init();
        prefetch_tensormap(&a.tm_x);
        prefetch_tensormap(&a.tm_sp);
        prefetch_tensormap(&a.tm_f[0]);
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
        if (tid == 0) {
            prodq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            prod_count = 0;
            for (int s = 0; s < STAGES; ++s) issue_next();
        }
        const bool sigm = st.mode == 2;
        const int xw = tid >> 5, xl = tid & 31;  // warp; lane -> (row xl & 7, strip xl >> 3)

        // one x-pass item: row r, strip sx; SIG applies the sigmoid to y_k
        auto item = [&](auto sig_c, const float* rs, float* xbu, float* xbp, int r, int sx) {
            constexpr bool SIG = decltype(sig_c)::value;
            const float4* py = reinterpret_cast<const float4*>(rs) + r * BW4 + 2 * sx;
            float ou[G::SW];
            float2 op[G::SW];
            float4 yv, sv, fv;
#pragma unroll
            for (int m4 = 0; m4 < G::NLD * 4; ++m4) {
                if (m4 % 4 == 0) {
                    yv = py[m4 / 4];
                    sv = py[FB / 4 + m4 / 4];
                    fv = py[2 * (FB / 4) + m4 / 4];
                }
                const int m = m4 - G::XOFF;
                if (m < 0 || m >= G::NINX) continue;
                const int c = m4 % 4;
                const float y = c == 0 ? yv.x : c == 1 ? yv.y : c == 2 ? yv.z : yv.w;
                const float s = c == 0 ? sv.x : c == 1 ? sv.y : c == 2 ? sv.z : sv.w;
                const float f = c == 0 ? fv.x : c == 1 ? fv.y : c == 2 ? fv.z : fv.w;
                const float x = SIG ? A::load_sigmoid(y, st) : y;
                const float u = s * x;  // engine.cpp:92-100 (FAST: F (F u))
                const float fu = f * u;
                const float2 pr = make_float2(fu, f * fu);
#pragma unroll
                for (int j = 0; j < G::SW; ++j) {
                    const int d = m - j;
                    if (d < 0 || d > 2 * R) continue;
                    if (d == 0) {
                        ou[j] = a.taps_x[0] * u;
                        op[j] = ffma2(pr, make_float2(a.taps_x[0], a.taps_x[0]), zero2);
                    } else {
                        ou[j] = fmaf(a.taps_x[d], u, ou[j]);
                        op[j] = ffma2(pr, make_float2(a.taps_x[d], a.taps_x[d]), op[j]);
                    }
                }
            }
            float4* du = reinterpret_cast<float4*>(xbu + r * TXU + sx * G::SW);
#pragma unroll
            for (int v = 0; v < G::SW / 4; ++v)
                du[v] = make_float4(ou[4 * v], ou[4 * v + 1], ou[4 * v + 2], ou[4 * v + 3]);
            float4* dp = reinterpret_cast<float4*>(xbp + r * TXQ + 2 * sx * G::SW);
#pragma unroll
            for (int v = 0; v < G::SW / 2; ++v)
                dp[v] = make_float4(op[2 * v].x, op[2 * v].y, op[2 * v + 1].x, op[2 * v + 1].y);
        };

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;  // in-volume planes handled
        for (; !q.done; q.next()) {
            const int tg = a.out_t0 + q.p;
            if (tg < 0 || tg >= a.T) continue;  // planes outside the volume: B zero-fills
            const int s = cnt % STAGES;
            const int b = cnt & 1;
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            mbar_wait(&xb_empty[b], ((cnt >> 1) & 1) ^ 1);
            const float* rs = raw + static_cast<size_t>(s) * 3 * FB;
            float* xbu = xb + b * XBUF;
            float* xbp = xbu + XBU;
#pragma unroll
            for (int k = 0; k < G::XPASS; ++k) {
                const int blk = xw + k * NWA;
                if (blk >= G::RBLK) break;
                const int r = blk * 8 + (xl & 7);
                if (r >= BH || (SFK_RS_EXP & 1)) continue;
                if (sigm && !(SFK_RS_EXP & 4))
                    item(std::true_type{}, rs, xbu, xbp, r, xl >> 3);
                else
                    item(std::false_type{}, rs, xbu, xbp, r, xl >> 3);
            }
            mbar_arrive(&xb_full[b]);  // release: this thread's x-pass stores
            named_bar_sync(1, NA);     // raw stage s fully read
            if (tid == 0) {
                fence_proxy_async();  // generic reads of stage s before the TMA overwrite
                issue_next();
            }
            ++cnt;
        }
    } else {
        // =====================================================================
        // B: y-pass ring, t-pass, recombination (x 1/||y_k||), store, reductions
        // =====================================================================
        setmaxnreg_inc<G::RB>();
        const int bt = tid - NA;
        // B thread = one column (its lane) x 8 rows (8 wb .. 8 wb + 7) of the tile
        const int lane = bt & 31;
        const int wb = bt >> 5;
        const float inv_alpha = a.inv_alpha;
        const bool last = a.last_group;
        // deferred normalisation: y_{k+1} = (1/||y_k||) A(y_k) (mode 1); the
        // sigmoid iterations (mode 2) normalised on load, iteration 1 has none
        const float scale = st.mode == 1 ? st.inv_f : 1.0f;

        float ringu[8][K];       // u
        float2 ringp[8][K];      // (F u, F^2 u)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                ringu[r][k] = 0.0f;
                ringp[r][k] = zero2;
            }

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;   // in-volume planes consumed
        // recombination operands S^p, F of this thread's 8 output points,
        // loaded one emitted plane ahead (cursor eq walks the output planes in
        // schedule order); rows / columns outside the volume read as 0, so
        // those points come out as exactly 0 and add nothing to the sums
        float nsp[8], nf[8];
        PlaneStream eq;
        eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
        auto fetch = [&]() {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                nsp[r] = 0.0f;
                nf[r] = 0.0f;
            }
            if (eq.done) return;
            // one 64-bit address per plane, then row increments; rows past H
            // are predicated off (columns past W read the zero pitch padding)
            const int y0 = eq.tile_y * TY + 8 * wb, nr = a.H - y0;
            const size_t off = (static_cast<size_t>(a.out_t0 + eq.p - a.buf_t0) * a.H + y0) * a.pitch +
                               eq.tile_x * TX + lane;
            const float* ps = a.sp + off;
            const float* pf = a.f[0] + off;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (r < nr) {
                    nsp[r] = __ldg(ps);
                    nf[r] = __ldg(pf);
                }
                ps += a.pitch;
                pf += a.pitch;
            }
            eq.next();
        };
        fetch();

        auto plane = [&](auto slot_c) {
            constexpr int S_ = decltype(slot_c)::value;
            const int tg = a.out_t0 + q.p;
            const bool valid = tg >= 0 && tg < a.T;
            const bool emit = q.p - RT >= q.ta;
            const int to = tg - RT;

            // y-pass (conv3d.cpp:113-135) into this plane's ring slot
            if (valid) {
                const int b = cnt & 1;
                mbar_wait(&xb_full[b], (cnt >> 1) & 1);
                const float* xbu = xb + b * XBUF + (8 * wb) * TXU + lane;
                const float2* xbp = reinterpret_cast<const float2*>(xb + b * XBUF + XBU + (8 * wb) * TXQ) + lane;
#pragma unroll
                for (int j = 0; j < ((SFK_RS_EXP & 2) ? 0 : 8 + 2 * R); ++j) {
                    const float vin = xbu[j * TXU];
                    const float2 pv = xbp[j * (TXQ / 2)];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int d = j - r;
                        if (d < 0 || d > 2 * R) continue;
                        if (d == 0) {
                            ringu[r][S_] = a.taps_y[0] * vin;
                            ringp[r][S_] = ffma2(pv, make_float2(a.taps_y[0], a.taps_y[0]), zero2);
                        } else {
                            ringu[r][S_] = fmaf(a.taps_y[d], vin, ringu[r][S_]);
                            ringp[r][S_] = ffma2(pv, make_float2(a.taps_y[d], a.taps_y[d]), ringp[r][S_]);
                        }
                    }
                }
                mbar_arrive(&xb_empty[b]);
                ++cnt;
            } else {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    ringu[r][S_] = 0.0f;
                    ringp[r][S_] = zero2;
                }
            }
            if (emit) {
                // columns past W land in the pitch padding as exact zeros (S^p
                // is 0 there); rows past H are predicated off
                const int y0 = q.tile_y * TY + 8 * wb, nr = a.H - y0;
                float* po = a.out + (static_cast<size_t>(to - a.out_buf_t0) * a.H + y0) * a.pitch +
                            q.tile_x * TX + lane;
                float v[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    // t-pass (conv3d.cpp:147-165): oldest..newest take taps_t[0..2RT]
                    float tu = a.taps_t[0] * ringu[r][(S_ + 1) % K];
                    float2 tp = ffma2(ringp[r][(S_ + 1) % K], make_float2(a.taps_t[0], a.taps_t[0]), zero2);
#pragma unroll
                    for (int d = 1; d < K; ++d) {
                        tu = fmaf(a.taps_t[d], ringu[r][(S_ + 1 + d) % K], tu);
                        tp = ffma2(ringp[r][(S_ + 1 + d) % K], make_float2(a.taps_t[d], a.taps_t[d]), tp);
                    }
                    // engine.cpp:113-119; channel sum engine.cpp:157-162
                    const float term = A::recombine(nsp[r] * scale, nf[r], inv_alpha, tu, tp.y, tp.x);
                    if constexpr (ACC)  // y so far (earlier groups)
                        v[r] = r < nr ? *po + term : 0.0f;
                    else
                        v[r] = term;
                    if (r < nr) *po = v[r];
                    po += a.pitch;
                }
                fetch();  // the next emitted plane's operands
                if (last) {
                    // canonical reduction (device_common.cuh): two 4-row blocks per
                    // warp, one column per lane, fp32 within a block (FAST)
                    double sum[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float cs = 0.0f;
#pragma unroll
                        for (int r = 0; r < 4; ++r) cs = fmaf(v[4 * h + r], v[4 * h + r], cs);
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
                        sum[h] = static_cast<double>(cs);
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
        }
    }
}

}  // namespace sfk
