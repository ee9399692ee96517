// fused_rs.cuh — SFSeg power-iteration step for one feature channel, FAST
// arithmetic, with the products formed in registers inside the x-pass
// ("register-streamed").
//
// One launch per iteration does the products (engine.cpp:92-100), the three
// separable convolutions of u, F u, F^2 u (conv3d.cpp:80-185), the
// recombination (engine.cpp:107-120) and the sum-of-squares / max scans of
// normalize_l2 / project_binary (engine.cpp:168-205).
//
// Inputs. The u field is read as it is: U = S^p x (the previous step's
// write_u store, or k_make_u for iteration 1 and binarised iterations), so an
// x-pass thread reads two halo boxes, U and F, for its 8-output strip and
// forms F u and F^2 u = F (F u) in registers. With the x box and the S^p box
// replaced by one U box, the L2 -> SM traffic per output drops from 3 to 2
// halo boxes. The last launch of a solve stores y_{k+1} (the
// caller reads it); earlier ones store U_{k+1} = S^p y_{k+1} (a.write_u).
//
// FAST: the normalisation 1/||y_k|| is applied to the output instead of to
// every input (the operator is linear: A(y s) = s A(y)).
//
// Roles (one 512-thread CTA per SM, persistent over (64 x 32 tile, frame
// range) segments): 8 A warps issue the halo-box TMA loads (box b of a plane
// by lane 0 of warp 6 + b) and run the x-pass; 8 B warps run the y-pass, the
// t-pass (register variants: 2RT pending outputs kept as running sums, each
// y-filtered plane scattered into them; RT >= 3: a ring of the last 2RT+1
// planes in tensor memory, gathered at emission), the recombination, the
// store and the canonical reductions. A and B meet at two mbarrier pairs per
// x-pass buffer.
#pragma once

#include <type_traits>

#include "device_common.cuh"
#include "sfseg_types.cuh"
#include "step_common.cuh"  // PlaneStream, Arith, ffma2

namespace sfk {

template <int RT, int R, int STAGES, bool TMR_>
struct RsGeom {
    static constexpr bool TMR = TMR_;  // t-pass ring in tensor memory
    static constexpr int TY = 64, TX = 32, BR = 8, NWA = 8;
    static constexpr int NWB = TY / BR;
    static constexpr int NA = 32 * NWA, NB = 32 * NWB, NT = NA + NB;
    static constexpr int K = 2 * RT + 1;
    static constexpr int BH = TY + 2 * R;
    // x halos: the box must start on a 16-byte boundary (TMA faults on an
    // unaligned innermost coordinate), so the left halo HX is R rounded up to
    // whole float4s; the right halo HR >= R makes the row an odd number of
    // float4s, so float4 reads of 8 rows at one strip are conflict-free
    static constexpr int HX = (R + 3) / 4 * 4;
    static constexpr int HR = ((TX + 2 * HX) / 4) % 2 == 1 ? HX : HX + 4;
    static constexpr int BW = TX + HX + HR;
    static constexpr int BW4 = BW / 4;
    static constexpr int XOFF = HX - R;  // first box column a strip reads
    static constexpr int FB = (BH * BW + 31) / 32 * 32;
    static constexpr int NIN = 2;  // raw boxes: U, F
    // x-pass items: (row, 8-column strip); a warp pass = 8 rows x 4 strips
    static constexpr int SW = 8;
    static constexpr int NINX = SW + 2 * R;            // inputs per strip
    static constexpr int NLD = (XOFF + NINX + 3) / 4;  // float4 loads per field
    static constexpr int RBLK = (BH + 7) / 8;          // 8-row blocks
    static constexpr int XPASS = (RBLK + NWA - 1) / NWA;
    // x-pass output, read by B: u [BH][TXU], (F u, F^2 u) pairs [BH][TXQ]
    static constexpr int TXU = TX + 4, TXQ = 2 * TX + 4;
    static constexpr int XBU = (BH * TXU + 31) / 32 * 32;
    static constexpr int XBP = (BH * TXQ + 31) / 32 * 32;
    static constexpr int XBUF = XBU + XBP;
    static constexpr int NXB = 2;  // x-pass buffers between A and B
    static constexpr int NBANDS = TY / 4;
    static constexpr size_t RAW_FLOATS = size_t(STAGES) * NIN * FB;
    static constexpr size_t XB_FLOATS = NXB * size_t(XBUF);
    // recombination operands S^p, F and the y_{k+1} staging: register-ring
    // variants move CTA-wide TY x TX tiles (3 TMA operations per plane);
    // TMEM-ring variants move one BR x TX slab per B warp
    static constexpr int SLAB = BR * TX;
    static constexpr size_t SL_FLOATS = size_t(3) * TY * TX;
    static constexpr int NBAR = STAGES + 2 * NXB + NWB;
    static constexpr size_t SMEM_BYTES = (RAW_FLOATS + XB_FLOATS + SL_FLOATS) * sizeof(float) + NBAR * 8;
    // setmaxnreg: every warp starts with 65536 / NT registers per thread; A
    // gives back down to RA and B takes what A released (an SMSP holds two
    // A and two B warps)
    static constexpr int RA = 64;
    static constexpr int RPOOL = (65536 / NT) / 8 * 8;
    static constexpr int RB_ = (2 * RPOOL - RA) / 8 * 8;
    static constexpr int RB = RB_ > 248 ? 248 : RB_;
    static_assert(BW4 % 2 == 1, "odd float4 box rows");
    static_assert((TXU / 4) % 2 == 1 && (TXQ / 4) % 2 == 1, "conflict-free x-pass rows");
    static_assert(BW <= 256 && BH <= 256, "TMA box limit");
    static_assert(TMR || K <= 7, "register ring depth");
    static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// PEER: the time-sharded instantiation that also stores its edge planes into
// the neighbours' halo frames (a separate instantiation: the single-GPU
// kernel does not carry the extra epilogue code)
template <int RT, int R, int STAGES, bool TMR_, bool PEER = false>
__global__ void __launch_bounds__(RsGeom<RT, R, STAGES, TMR_>::NT, 1)
    fused_step_rs(const __grid_constant__ FusedArgs a) {
    using G = RsGeom<RT, R, STAGES, TMR_>;
    using A = Arith<true>;
    constexpr int BR = G::BR, TY = G::TY, TX = G::TX, NA = G::NA, NB = G::NB, K = G::K, NWB = G::NWB;
    constexpr int BH = G::BH, FB = G::FB, BW4 = G::BW4, SW = G::SW, NXB = G::NXB;
    constexpr int TXU = G::TXU, TXQ = G::TXQ, XBU = G::XBU, XBUF = G::XBUF, SLAB = G::SLAB;
    constexpr bool TMR = G::TMR;

    extern __shared__ __align__(128) float smem[];
    float* raw = smem;                // [STAGES][2][FB]    TMA boxes U, F
    float* xb = raw + G::RAW_FLOATS;  // [NXB][XBUF]        x-pass output
    float* bsl = xb + G::XB_FLOATS;   // S^p, F, y_{k+1} tiles (or per-warp slabs)
    uint64_t* mbar = reinterpret_cast<uint64_t*>(bsl + G::SL_FLOATS);
    uint64_t* raw_full = mbar;                      // [STAGES]  TMA -> A
    uint64_t* xb_full = mbar + STAGES;              // [NXB]  A -> B (count NA)
    uint64_t* xb_empty = mbar + STAGES + NXB;       // [NXB]  B -> A (count NB)
    uint64_t* slab_full = mbar + STAGES + 2 * NXB;  // [NWB]  TMA -> B

    __shared__ IterState st;
    __shared__ PlaneStream slabq[NWB];
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
        prefetch_tensormap(&a.tm_f[0]);
        prefetch_tensormap(&a.tm_out);
        prefetch_tensormap(&a.tm_spc);
        prefetch_tensormap(&a.tm_fc[0]);
    }
    __syncthreads();

    const float2 zero2 = make_float2(0.0f, 0.0f);

    if (tid < NA) {
        // =====================================================================
        // A: TMA producer + x-pass (conv3d.cpp:88-101), products in registers
        // =====================================================================
        setmaxnreg_dec<G::RA>();
        // box `pbox` of every plane is issued by lane 0 of warp NWA - 2 + pbox
        // with its own plane cursor (one issuer for all boxes cost ~1000
        // cycles per plane on a warp that also runs x-pass blocks); box 0
        // carries the expect_tx of both
        const int pbox = (tid >> 5) - (G::NWA - G::NIN);
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
            float* dst = raw + static_cast<size_t>(s) * G::NIN * FB + pbox * FB;
            uint64_t* bar = &raw_full[s];
            const int bx = pq.tile_x * TX - G::HX, by = pq.tile_y * TY - R, bt = tg - a.buf_t0;
            if (pbox == 0) mbar_arrive_expect_tx(bar, G::NIN * BH * G::BW * sizeof(float));
            tma_load_3d(dst, pbox == 0 ? &a.tm_x : &a.tm_f[0], bar, bx, by, bt);
            ++pcount;
            pq.next();
        };
        if (pissuer) {
            pq.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
            for (int s = 0; s < STAGES; ++s) issue_box();
        }
        const int xw = tid >> 5, xl = tid & 31;  // warp; lane -> (row xl & 7, strip xl >> 3)

        // one x-pass item: box row r, strip sx (SW outputs). u runs as column
        // pairs (2k, 2k+1) with tap pairs (w[e], w[e-1]); (F u, F^2 u) as a
        // pair per column with a broadcast tap
        auto item = [&](const float* rs, float* xbu, float* xbp, int r, int sx) {
            const float4* py = reinterpret_cast<const float4*>(rs) + r * BW4 + sx * (SW / 4);
            float2 ou[SW / 2];
            float2 op[SW];
            float4 uv, fv;
#pragma unroll
            for (int m4 = 0; m4 < G::NLD * 4; ++m4) {
                if (m4 % 4 == 0) {
                    uv = py[m4 / 4];
                    fv = py[FB / 4 + m4 / 4];
                }
                const int m = m4 - G::XOFF;
                if (m < 0 || m >= G::NINX) continue;
                const int c = m4 % 4;
                const float u = c == 0 ? uv.x : c == 1 ? uv.y : c == 2 ? uv.z : uv.w;
                const float f = c == 0 ? fv.x : c == 1 ? fv.y : c == 2 ? fv.z : fv.w;
                const float fu = f * u;  // engine.cpp:92-100 (FAST: F (F u))
                const float2 pr = make_float2(fu, f * fu);
#pragma unroll
                for (int k = 0; k < SW / 2; ++k) {
                    const int e = m - 2 * k;
                    if (e < 0 || e > 2 * R + 1) continue;
                    // the pair's edge taps have a zero partner (w[-1], w[2R+1])
                    if (e == 0)
                        ou[k] = make_float2(u * a.taps_x[0], 0.0f);
                    else if (e == 2 * R + 1)
                        ou[k].y = fmaf(u, a.taps_x[2 * R], ou[k].y);
                    else
                        ou[k] = ffma2(make_float2(u, u), a.tpair_x[e], ou[k]);
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
        };

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;  // in-volume planes handled
        for (; !q.done; q.next()) {
            const int tg = a.out_t0 + q.p;
            if (tg < 0 || tg >= a.T) continue;  // planes outside the volume: B zero-fills
            const int s = cnt % STAGES;
            const int b = cnt % NXB;
            mbar_wait(&raw_full[s], (cnt / STAGES) & 1);
            mbar_wait(&xb_empty[b], ((cnt / NXB) & 1) ^ 1);
            const float* rs = raw + static_cast<size_t>(s) * G::NIN * FB;
            float* xbu = xb + b * XBUF;
            float* xbp = xbu + XBU;
#pragma unroll
            for (int k = 0; k < G::XPASS; ++k) {
                const int blk = xw + k * G::NWA;
                if (blk >= G::RBLK) break;
                const int r = blk * 8 + (xl & 7);
                if (r < BH) item(rs, xbu, xbp, r, xl >> 3);
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
        const bool wu = a.write_u != 0;
        // deferred normalisation: y_{k+1} = (1/||y_k||) A(y_k) (mode 1);
        // binarised iterations (mode 2) come normalised in U
        const float scale = st.mode == 1 ? st.inv_f : 1.0f;

        // t-pass in scatter form (register variants): instead of a ring of the
        // last K y-filtered planes summed at emission, KA = K - 1 pending
        // outputs are kept as running sums. Plane p completes output p - RT
        // with its last tap (the only t-pass work between the y-pass and the
        // recombination), starts output p + RT with tap 0 in the freed slot
        // and adds to the K - 2 outputs in between; those updates have no
        // consumer until later planes, so they sit in the epilogue's latency
        // shadows. An output still receives taps 0..2RT in plane order: the
        // same FMA sequence, the same bits as the gather form. A slot is
        // re-initialised (tap 0) before its output's other taps arrive, so
        // nothing carries over between schedule segments.
        constexpr int KA = TMR ? 1 : K - 1;
        static_assert(TMR || RT >= 1, "scatter t-pass needs a temporal radius");
        float2 yu[BR / 2], yp[BR];  // y-filtered current plane: u of rows (2k, 2k+1); (F u, F^2 u) of row r
        float2 accu[BR / 2][KA];
        float2 accp[BR][KA];
#pragma unroll
        for (int k = 0; k < KA; ++k) {
#pragma unroll
            for (int r = 0; r < BR / 2; ++r) accu[r][k] = zero2;
#pragma unroll
            for (int r = 0; r < BR; ++r) accp[r][k] = zero2;
        }
        // TMEM ring: slot = 3 BR words (u pairs, then (F u, F^2 u) per row) in
        // this thread's TMEM lane; warps w and w + 4 share a lane quadrant
        // and take the two column halves
        constexpr int RW = 3 * BR;
        constexpr int TCOLS = K * RW <= 128 ? 256 : 512;
        static_assert(!TMR || K * RW <= TCOLS / 2, "TMEM ring of one thread");
        uint32_t tm_ring = 0;
        int rslot = 0;  // TMR: ring slot of the current plane
        if constexpr (TMR) {
            if (wb == 0) tmem_alloc<TCOLS>(&tmem_base_sh);
            tcgen05_fence_before();
            named_bar_sync(2, NB);
            tcgen05_fence_after();
            const int wq = (G::NWA + wb) & 3;  // CTA warp id % 4
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

        // recombination operands S^p, F: TMA, one emitted plane ahead (cursor
        // eq walks the output planes in schedule order); zero-filled outside
        // the volume, so those points come out as exactly 0, add nothing to
        // the sums, and the TMA store clips them. WIDE (register ring): one
        // CTA-wide tile pair per plane and one y-tile store, two B-wide
        // barriers per plane; TMEM ring: a slab pair and a store per B warp.
        constexpr bool WIDE = !TMR;
        float* slab = WIDE ? bsl + (BR * wb) * TX : bsl + wb * 3 * SLAB;
        constexpr int SLSTEP = WIDE ? TY * TX : SLAB;  // distance S^p -> F -> y rows
        uint64_t* sfull = WIDE ? &slab_full[0] : &slab_full[wb];
        PlaneStream& eq = slabq[WIDE ? 0 : wb];  // issuing thread only
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
        if (WIDE ? bt == 0 : lane == 0) {
            eq.init(a.sched + s0, s1 - s0, 0, a.tiles_x);
            issue_slab();
        }

        PlaneStream q;
        q.init(a.sched + s0, s1 - s0, RT, a.tiles_x);
        int cnt = 0;   // in-volume planes consumed
        int ecnt = 0;  // output planes emitted

        // canonical reduction (device_common.cuh) of one emitted plane: BR / 4
        // blocks of 4 rows per warp, one column per lane, fp32 within a block.
        // The two blocks of a warp share one butterfly: after the first
        // exchange lanes 0-15 hold block 0's pair sums c_i + c_{i+16} and lanes
        // 16-31 block 1's, exactly the values the per-block xor-16 step leaves
        // in those lanes (addition commutes), and the xor 8, 4, 2, 1 steps stay
        // inside each half: same operands, same order, same bits, half the
        // shuffles. `doit` predicates the stores (no branch), and the call sits
        // before the staging stores, so the shuffle latency overlaps them
        // (measured: 203.0 -> 192.3 us per c1 launch).
        static_assert(BR == 8, "two 4-row blocks per warp");
        auto reduce_plane = [&](const float (&v)[BR], int to, int tx, int ty, bool doit) {
            float cs0 = 0.0f, cs1 = 0.0f;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                cs0 = fmaf(v[r], v[r], cs0);
                cs1 = fmaf(v[4 + r], v[4 + r], cs1);
            }
            const bool lo = lane < 16;
            float cs = (lo ? cs0 : cs1) + __shfl_xor_sync(0xffffffffu, lo ? cs1 : cs0, 16);
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
            float cmax = 0.0f;
#pragma unroll
            for (int r = 0; r < BR; ++r) cmax = fmaxf(cmax, v[r]);
            const int wm = __reduce_max_sync(0xffffffffu, __float_as_int(cmax));
            const int gb = ty * G::NBANDS + (BR / 4) * wb + (lo ? 0 : 1);
            if (doit && (lane & 15) == 0 && gb < a.nbands && tx < a.nhalves)
                a.part[(static_cast<size_t>(to - a.part_t0) * a.nbands + gb) * a.nhalves + tx] =
                    static_cast<double>(cs);
            if (doit && lane == 0) atomic_max_nonneg(a.frame_max + (to - a.part_t0), __int_as_float(wm));
        };

        auto plane = [&](auto slot_c) {
            constexpr int S_ = decltype(slot_c)::value;  // register variants: the emitting slot
            [[maybe_unused]] const int slot = rslot;     // TMEM ring: slot of this plane
            const int tg = a.out_t0 + q.p;
            const bool valid = tg >= 0 && tg < a.T;
            const bool emit = q.p - RT >= q.ta;
            const int to = tg - RT;

            // y-pass (conv3d.cpp:113-135) of this plane
            if (valid) {
                const int b = cnt % NXB;
                mbar_wait(&xb_full[b], (cnt / NXB) & 1);
                const float* xbu = xb + b * XBUF + (BR * wb) * TXU + lane;
                const float2* xbp = reinterpret_cast<const float2*>(xb + b * XBUF + XBU + (BR * wb) * TXQ) + lane;
                // all BR + 2R input rows first, then tap-major order:
                // consecutive FFMA2s feed different accumulators
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
                    for (int k = 0; k < BR / 2; ++k) {
                        const float vv = vin[2 * k + e];
                        if (e == 0)  // zero-partner edge taps as scalar ops
                            yu[k] = make_float2(vv * a.taps_y[0], 0.0f);
                        else if (e == 2 * R + 1)
                            yu[k].y = fmaf(vv, a.taps_y[2 * R], yu[k].y);
                        else
                            yu[k] = ffma2(make_float2(vv, vv), a.tpair_y[e], yu[k]);
                    }
                    if (e <= 2 * R) {
#pragma unroll
                        for (int r = 0; r < BR; ++r)
                            yp[r] = ffma2(pv[r + e], make_float2(a.taps_y[e], a.taps_y[e]), e == 0 ? zero2 : yp[r]);
                    }
                }
                mbar_arrive(&xb_empty[b]);
                ++cnt;
            } else {
#pragma unroll
                for (int r = 0; r < BR / 2; ++r) yu[r] = zero2;
#pragma unroll
                for (int r = 0; r < BR; ++r) yp[r] = zero2;
            }
            // scatter step j of this plane (register variants): j = 0 starts
            // the output RT planes ahead in the slot the emission freed, j >= 1
            // adds tap K - 1 - j to the output emitted j planes from now
            [[maybe_unused]] auto scatter = [&](auto jc) {
                constexpr int J = decltype(jc)::value;
                if constexpr (!TMR && J < KA) {
                    constexpr int SJ = (S_ + J) % KA;
                    const float2 w2 = make_float2(a.taps_t[J == 0 ? 0 : K - 1 - J], a.taps_t[J == 0 ? 0 : K - 1 - J]);
#pragma unroll
                    for (int k = 0; k < BR / 2; ++k) accu[k][SJ] = ffma2(yu[k], w2, J == 0 ? zero2 : accu[k][SJ]);
#pragma unroll
                    for (int r = 0; r < BR; ++r) accp[r][SJ] = ffma2(yp[r], w2, J == 0 ? zero2 : accp[r][SJ]);
                }
            };
            using std::integral_constant;
            if (emit) {
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
                            for (int k = 0; k < BR / 2; ++k) lu[k] = yu[k];
#pragma unroll
                            for (int r = 0; r < BR; ++r) lp[r] = yp[r];
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
                    // the last tap completes the output in slot S_
                    const float2 wl = make_float2(a.taps_t[K - 1], a.taps_t[K - 1]);
#pragma unroll
                    for (int k = 0; k < BR / 2; ++k) tu[k] = ffma2(yu[k], wl, accu[k][S_]);
#pragma unroll
                    for (int r = 0; r < BR; ++r) tp[r] = ffma2(yp[r], wl, accp[r][S_]);
                }
                float spv[BR], fv[BR];
                mbar_wait(sfull, ecnt & 1);
#pragma unroll
                for (int r = 0; r < BR; ++r) {
                    spv[r] = slab[r * TX + lane];
                    fv[r] = slab[SLSTEP + r * TX + lane];
                }
                scatter(integral_constant<int, 0>{});
                scatter(integral_constant<int, 1>{});
                if constexpr (WIDE) {
                    if (bt == 0) bulk_wait_read0();  // the previous y tile store has read the staging
                    named_bar_sync(3, NB);            // every B warp has read the tiles
                    if (bt == 0) {
                        fence_proxy_async();
                        issue_slab();
                    }
                } else {
                    __syncwarp();
                    if (lane == 0) {
                        fence_proxy_async();  // the reads above before the next TMA write
                        issue_slab();
                    }
                }
                float v[BR], o[BR];
#pragma unroll
                for (int r = 0; r < BR; ++r) {
                    const float tur = (r & 1) ? tu[r / 2].y : tu[r / 2].x;
                    // engine.cpp:113-119
                    v[r] = A::recombine(spv[r] * scale, fv[r], inv_alpha, tur, tp[r].y, tp[r].x);
                    o[r] = wu ? spv[r] * v[r] : v[r];  // U_{k+1} = S^p y_{k+1} or y_{k+1}
                }
                const int ox = q.tile_x * TX, oy = q.tile_y * TY + BR * wb;
                reduce_plane(v, to, q.tile_x, q.tile_y, last);
                scatter(integral_constant<int, 2>{});
                scatter(integral_constant<int, 3>{});
                scatter(integral_constant<int, 4>{});
                scatter(integral_constant<int, 5>{});
                if constexpr (WIDE) {
                    float* ost = slab + 2 * SLSTEP;
#pragma unroll
                    for (int r = 0; r < BR; ++r) ost[r * TX + lane] = o[r];
                    fence_proxy_async();
                    named_bar_sync(3, NB);
                    if (bt == 0) {
                        tma_store_3d(&a.tm_out, bsl + 2 * SLSTEP, ox, q.tile_y * TY, to - a.out_buf_t0);
                        bulk_commit();
                    }
                } else {
                    // rows -> staging -> TMA store (clipped at the volume edge)
                    float* ost = slab + 2 * SLAB;
                    if (lane == 0) bulk_wait_read0();  // the previous store has read the staging
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < BR; ++r) ost[r * TX + lane] = o[r];
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_3d(&a.tm_out, ost, ox, oy, to - a.out_buf_t0);
                        bulk_commit();
                    }
                }
                // time-sharded solve: the edge planes of this rank also go
                // straight into the neighbours' halo frames (peer memory,
                // coalesced 128-byte rows; rows past H are not written)
                if (PEER && last) {
#pragma unroll
                    for (int side = 0; side < 2; ++side) {
                        float* pb = a.peer[side];
                        const bool edge = side == 0 ? to < a.out_t0 + a.peer_n : to >= a.out_t1 - a.peer_n;
                        if (!pb || !edge) continue;
                        const int nr = a.H - oy;
                        float* po = pb + (static_cast<size_t>(to - a.peer_t0[side]) * a.H + oy) * a.pitch +
                                    q.tile_x * TX + lane;
#pragma unroll
                        for (int r = 0; r < BR; ++r)
                            if (r < nr) po[static_cast<size_t>(r) * a.pitch] = o[r];
                    }
                }
                ++ecnt;
            } else {
                // the first 2RT planes of a segment emit nothing
                scatter(integral_constant<int, 0>{});
                scatter(integral_constant<int, 1>{});
                scatter(integral_constant<int, 2>{});
                scatter(integral_constant<int, 3>{});
                scatter(integral_constant<int, 4>{});
                scatter(integral_constant<int, 5>{});
            }
            if constexpr (TMR) {
                // this plane into its slot (it held a plane no longer needed)
                float w[8];
#pragma unroll
                for (int k = 0; k < BR / 2; ++k) {
                    w[2 * k] = yu[k].x;
                    w[2 * k + 1] = yu[k].y;
                }
                tmem_st8(tm_ring + slot * RW, w);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        w[2 * r] = yp[4 * h + r].x;
                        w[2 * r + 1] = yp[4 * h + r].y;
                    }
                    tmem_st8(tm_ring + slot * RW + 8 + 8 * h, w);
                }
                rslot = rslot + 1 == K ? 0 : rslot + 1;
            }
            q.next();
        };
        using std::integral_constant;
        if constexpr (TMR) {
            while (!q.done) plane(integral_constant<int, 0>{});  // runtime slots
        } else while (!q.done) {
            // pending-output slots: the index must be a compile-time constant
            plane(integral_constant<int, 0>{});
            if constexpr (KA > 1) { if (q.done) break; plane(integral_constant<int, (KA > 1 ? 1 : 0)>{}); }
            if constexpr (KA > 2) { if (q.done) break; plane(integral_constant<int, (KA > 2 ? 2 : 0)>{}); }
            if constexpr (KA > 3) { if (q.done) break; plane(integral_constant<int, (KA > 3 ? 3 : 0)>{}); }
            if constexpr (KA > 4) { if (q.done) break; plane(integral_constant<int, (KA > 4 ? 4 : 0)>{}); }
            if constexpr (KA > 5) { if (q.done) break; plane(integral_constant<int, (KA > 5 ? 5 : 0)>{}); }
        }
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
