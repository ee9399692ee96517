// sfseg_types.cuh — structures shared between the host driver and kernels.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace sfk {

constexpr int kMaxCG = 4;      // feature channels fused into one stencil pass
constexpr int kMaxTapsXY = 32;  // 2*R+1 for R <= 15
constexpr int kMaxTapsT = 16;   // 2*RT+1 for RT <= 7

// Scalars carried from one iteration to the next, written on the device by
// finalize_total and read by the next stencil launch (no host round trip).
struct IterState {
    double inv;        // 1 / ||y_k||                      (engine.cpp:178)
    double theta;      // threshold_frac * max(x_unit)     (engine.cpp:191)
    double lambda;     // slope0 * growth^(k - start)      (engine.cpp:192-193)
    double norm;       // ||y_k||
    int32_t mode;      // 0: x = y (iteration 1); 1: normalise; 2: normalise + sigmoid
    int32_t degenerate;  // sticky: some ||y_k|| == 0      (engine.cpp:174-175)
    float max_raw;     // max(0, max y_k)
    float max_unit;    // max(0, max x_unit)
    float inv_f, theta_f, lambda_f;  // float copies for the FAST arithmetic
    // sfseg_solve_until: set on the device by k_conv_final once the stopping
    // rule holds (> 0: the iteration it held at; < 0: the rule is undefined, a
    // zero vector). While it is set, every kernel of the later iterations
    // already in the stream returns at once, so the iterate stays put.
    int32_t stop;
};

// Arguments of one fused stencil launch (one channel group of one step).
struct FusedArgs {
    CUtensorMap tm_x;           // iterate source y_k (or S / x0 at iteration 1)
    CUtensorMap tm_sp;          // S^p
    CUtensorMap tm_f[kMaxCG];   // feature channels of this group
    CUtensorMap tm_out;         // y_{k+1}, box = one warp's 8-row output slab (TMA store)
    CUtensorMap tm_spc;         // S^p, box = one 8-row slab (recombination operands)
    CUtensorMap tm_fc[kMaxCG];  // F_c, box = one 8-row slab
    const float* sp;            // pitched S^p (recombination reload)
    const float* f[kMaxCG];
    float* out;                 // pitched y_{k+1}
    double* part;               // canonical partial sums [Tout][nbands][nhalves]
    float* frame_max;           // [Tout] max(0, y_{k+1}) per frame (int-ordered)
    int part_t0;                // global frame of part/frame_max entry 0
    const IterState* st;
    float taps_x[kMaxTapsXY];
    float taps_y[kMaxTapsXY];
    float taps_t[kMaxTapsT];
    // FAST kernel (fused_rs.cuh): tap pairs (w[e], w[e-1]), w[-1] = w[2R+1] = 0,
    // so two neighbouring outputs take one input with one FFMA2
    float2 tpair_x[kMaxTapsXY + 1];
    float2 tpair_y[kMaxTapsXY + 1];
    float inv_alpha;
    float c_inv_alpha;  // C / alpha (fused_mc.cuh HEAD launch)
    int write_u;        // fused_mc.cuh last launch: store U_{k+1} = S^p y_{k+1} instead of y_{k+1}
    // time-sharded solve with peer-memory halos (fused_rs.cuh, last group):
    // output planes [out_t0, out_t0 + peer_n) also go to peer[0] (rank-1's
    // iterate buffer, frame origin peer_t0[0]) and [out_t1 - peer_n, out_t1)
    // to peer[1]; nullptr = no neighbour / not pushed by the kernel
    float* peer[2];
    int peer_t0[2];
    int peer_n;
    float one, zero;  // 1.0f / 0.0f at run time (keeps ptxas from contracting EXACT FFMA2 pairs)
    int T, H, W, pitch;
    int buf_t0;      // global frame of input buffer frame 0
    int out_t0, out_t1;  // global output frames [out_t0, out_t1)
    int out_buf_t0;  // global frame of output buffer frame 0
    int tiles_x, tiles_y;
    const int4* sched;   // segments (tile, ta, tb, 0), ta/tb relative to out_t0
    const int* sched_off;  // CTA b walks sched[sched_off[b] .. sched_off[b+1])
    int first_group, last_group;
    int nbands, nhalves;
};

}  // namespace sfk
