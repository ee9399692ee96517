// sfseg_api.cu — host driver of the B200 SFSeg library and implementation of
// the C ABI declared in include/sfseg_cuda.h.
//
// Per iteration of Algorithm 1 (engine.cpp:284-341) the context launches, on
// its own stream: the fused stencil kernel once per channel group
// (fused_rs.cuh / fused_ws.cuh / fused_mc.cuh) and k_finalize. No host
// synchronisation happens inside the loop; norms and the projection scalars
// stay on the device (IterState) until the solve ends.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sfseg_cuda.h"
#include "aux_kernels.cuh"
#include "step_common.cuh"
#include "fused_ws.cuh"
#include "fused_rs.cuh"
#include "fused_mc.cuh"
#include "affinity.cuh"

namespace {

using sfk::FusedArgs;
using sfk::IterState;
using sfk::Vol;

thread_local std::string g_err;
std::atomic<uint64_t> g_conv_count{0};

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what);

// After every launch: launch errors always; with SFSEG_DEBUG_SYNC=1 also a
// stream sync so an asynchronous fault is attributed to the right kernel.
void launched(cudaStream_t s, const char* what) {
    static const bool dbg = [] {
        const char* v = std::getenv("SFSEG_DEBUG_SYNC");
        return v && *v && *v != '0';
    }();
    ck(cudaGetLastError(), what);
    if (dbg) ck(cudaStreamSynchronize(s), what);
}

void ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation)
        fail(SFSEG_ERR_CAPACITY, std::string(what) + ": " + cudaGetErrorString(e));
    fail(SFSEG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return SFSEG_OK;
    } catch (const Fail& f) {
        g_err = f.msg;
        return f.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SFSEG_ERR_STATE;
    }
}

// ---- taps: make_gaussian_kernel (conv3d.cpp:23-58), fp64 on the host ------
std::vector<double> raw_taps(double sigma, int r) {
    std::vector<double> t(2 * r + 1);
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (int i = -r; i <= r; ++i) t[i + r] = std::exp(-static_cast<double>(i) * i * inv);
    return t;
}

struct HostKernel {
    std::vector<double> t, y, x;
    int rt, ry, rx;
};

HostKernel make_kernel(const int32_t radii[3], const double sigmas[3]) {
    for (int a = 0; a < 3; ++a)
        if (!(sigmas[a] > 0.0)) fail(SFSEG_ERR_PARAMETER, "kernel sigma must be positive");
    for (int a = 0; a < 3; ++a)
        if (radii[a] < 0) fail(SFSEG_ERR_PARAMETER, "kernel radius must be nonnegative");
    HostKernel k;
    k.rt = radii[0];
    k.ry = radii[1];
    k.rx = radii[2];
    k.t = raw_taps(sigmas[0], radii[0]);
    k.y = raw_taps(sigmas[1], radii[1]);
    k.x = raw_taps(sigmas[2], radii[2]);
    auto sum = [](const std::vector<double>& v) {
        double s = 0.0;
        for (double a : v) s += a;
        return s;
    };
    const double total = sum(k.t) * sum(k.y) * sum(k.x);
    for (double& a : k.t) a /= total;
    return k;
}

// FAST arithmetic, opt-in (sfseg_ctx_set_tap_trim / SFSEG_FAST_TRIM=1): the
// outermost taps of an axis whose magnitude is at most 2^-24 of the axis's
// largest tap are dropped symmetrically, and the step runs the kernel of the
// remaining support. Such a tap moves an fp32 sum of the axis by less than
// half an ulp of the largest term; the operator changes by at most
// 2 (r - r') 2^-24 relative per axis, below the fp32 rounding FAST already
// differs from the reference by. BASELINE c4 (radii 4,10,10 with sigmas
// 0.5,1.5,1.5: exp(-9^2/4.5) = 1.5e-8, exp(-3^2/0.5) = 1.5e-8) runs as
// (2,8,8): 25% fewer FMAs; the other configs keep every tap. The taps are not
// renormalised (conv3d.cpp:52-55 normalises the full product kernel), EXACT
// never trims, and halos / peer pushes keep the requested temporal radius.
HostKernel trim_kernel(const HostKernel& k) {
    auto eff = [](const std::vector<double>& w, int r) {
        double mx = 0.0;
        for (double a : w) mx = std::max(mx, std::fabs(a));
        const double cut = std::ldexp(mx, -24);
        int re = r;
        while (re > 0 && std::fabs(w[r - re]) <= cut && std::fabs(w[r + re]) <= cut) --re;
        return re;
    };
    auto slice = [](const std::vector<double>& w, int r, int re) {
        return std::vector<double>(w.begin() + (r - re), w.begin() + (r + re + 1));
    };
    HostKernel t;
    t.rt = eff(k.t, k.rt);
    t.ry = eff(k.y, k.ry);
    t.rx = eff(k.x, k.rx);
    t.t = slice(k.t, k.rt, t.rt);
    t.y = slice(k.y, k.ry, t.ry);
    t.x = slice(k.x, k.rx, t.rx);
    return t;
}

void validate_params(const sfseg_params* c) {
    if (!c) fail(SFSEG_ERR_PARAMETER, "null params");
    // engine.cpp:21-42, same order and messages
    if (!(c->alpha > 0.0)) fail(SFSEG_ERR_PARAMETER, "alpha must be positive");
    if (c->p < 0.0) fail(SFSEG_ERR_PARAMETER, "p must be nonnegative");
    if (c->iterations < 1) fail(SFSEG_ERR_PARAMETER, "iterations must be at least 1");
    if (c->binarize_start < 1) fail(SFSEG_ERR_PARAMETER, "binarize_start must be at least 1");
    if (!(c->sigmoid_slope0 > 0.0)) fail(SFSEG_ERR_PARAMETER, "sigmoid_slope0 must be positive");
    if (!(c->slope_growth >= 1.0)) fail(SFSEG_ERR_PARAMETER, "slope_growth must be >= 1");
    if (!(c->threshold_frac > 0.0 && c->threshold_frac < 1.0))
        fail(SFSEG_ERR_PARAMETER, "threshold_frac must lie in (0,1)");
    if (!(c->final_threshold > 0.0 && c->final_threshold < 1.0))
        fail(SFSEG_ERR_PARAMETER, "final_threshold must lie in (0,1)");
    for (int a = 0; a < 3; ++a)
        if (!(c->sigmas[a] > 0.0)) fail(SFSEG_ERR_PARAMETER, "kernel sigma must be positive");
    for (int a = 0; a < 3; ++a)
        if (c->radii[a] < 0) fail(SFSEG_ERR_PARAMETER, "kernel radius must be nonnegative");
    if (c->temporal_window >= 0 && c->temporal_window < c->radii[0])
        fail(SFSEG_ERR_PARAMETER, "temporal_window must cover the kernel time radius");
    if (!c->allow_negative_affinity && c->alpha > 1.0)
        fail(SFSEG_ERR_PARAMETER,
             "alpha > 1 can produce negative affinities; enable allow_negative_affinity or "
             "reduce alpha");
    if (c->arith != SFSEG_ARITH_EXACT && c->arith != SFSEG_ARITH_FAST)
        fail(SFSEG_ERR_PARAMETER, "arith must be SFSEG_ARITH_EXACT or SFSEG_ARITH_FAST");
}

// ---- TMA descriptor encoding via the driver entry point -------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) fail(SFSEG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap encode_tmap(const float* base, int frames, int H, int W, int pitch, int box_w,
                        int box_h) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                                static_cast<cuuint64_t>(frames)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch) * 4,
                                   static_cast<cuuint64_t>(pitch) * H * 4};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                   const_cast<float*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SFSEG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

// A solve encodes the same few descriptors every iteration (the two iterate
// buffers alternate; S^p and the channels never change): a small per-thread
// cache keyed by every encoded field. A descriptor holds only the address
// and the geometry, so an entry stays valid when the buffer is reallocated
// at the same address. Small solves are host-bound without it (c0: ~15 us of
// kernels per iteration against five driver calls).
CUtensorMap make_tmap(const float* base, int frames, int H, int W, int pitch, int box_w,
                      int box_h) {
    struct Key {
        const float* base;
        int frames, H, W, pitch, box_w, box_h;
        bool operator==(const Key& o) const {
            return base == o.base && frames == o.frames && H == o.H && W == o.W && pitch == o.pitch &&
                   box_w == o.box_w && box_h == o.box_h;
        }
    };
    struct Entry {
        Key k;
        CUtensorMap m;
    };
    constexpr int kSlots = 64;  // direct-mapped
    thread_local std::vector<Entry> cache(kSlots, Entry{Key{nullptr, 0, 0, 0, 0, 0, 0}, CUtensorMap{}});
    const Key k{base, frames, H, W, pitch, box_w, box_h};
    size_t h = reinterpret_cast<uintptr_t>(base) >> 8;
    h = h * 0x9e3779b97f4a7c15ull + static_cast<size_t>(box_w) * 131 + static_cast<size_t>(box_h) * 31 +
        static_cast<size_t>(frames);
    Entry& e = cache[(h >> 20) % kSlots];
    if (!(e.k == k)) {
        e.m = encode_tmap(base, frames, H, W, pitch, box_w, box_h);
        e.k = k;
    }
    return e.m;
}

// ---- fused kernel registry -------------------------------------------------
// Each instantiation covers radii up to (RT, R) by zero-padding the taps:
// zero taps add +0 to the float sums, which leaves every value unchanged.
struct FusedVariant {
    int rt, r, ty, tx;
    bool fma;
    size_t smem;
    int threads;
    void (*kernel)(FusedArgs);
    void (*kernel_acc)(FusedArgs);  // later channel groups (y += terms); may equal kernel
    int box_w, box_h;
    int slab_h = 8;  // rows of the recombination-operand / output TMA boxes
    bool rs = false;      // fused_rs.cuh (stores the sharded solve's edge planes to the peers)
    void (*kernel_peer)(FusedArgs) = nullptr;  // rs: single-group step + peer edge stores
};

#ifndef SFK_NWA
#define SFK_NWA 8
#endif
template <int RT, int R, int NWA = SFK_NWA>
FusedVariant variant_ws() {
#ifndef SFK_STAGES
#define SFK_STAGES 2
#endif
    using G = sfk::WsGeom<RT, R, 1, SFK_STAGES, NWA>;
    FusedVariant v;
    v.rt = RT;
    v.r = R;
    v.ty = G::TY;
    v.tx = G::TX;
    v.fma = false;  // EXACT only (fused_ws.cuh)
    v.smem = G::SMEM_BYTES;
    v.threads = G::NT;
    v.kernel = sfk::fused_step_ws<RT, R, 1, SFK_STAGES, NWA, false>;
    v.kernel_acc = sfk::fused_step_ws<RT, R, 1, SFK_STAGES, NWA, true>;
    v.box_w = G::BW;
    v.box_h = G::BH;
    return v;
}

#ifndef SFK_RS_STAGES
#define SFK_RS_STAGES 3
#endif
// FAST, one channel: products formed in registers inside the x-pass, u read
// as U = S^p x (fused_rs.cuh)
template <int RT, int R, int ST = SFK_RS_STAGES, bool TMR = false>
FusedVariant variant_rs() {
    using G = sfk::RsGeom<RT, R, ST, TMR>;
    FusedVariant v;
    v.rt = RT;
    v.r = R;
    v.ty = G::TY;
    v.tx = G::TX;
    v.fma = true;
    v.smem = G::SMEM_BYTES;
    v.threads = G::NT;
    v.slab_h = TMR ? 8 : G::TY;  // TMEM-ring variants: per-warp slabs; else CTA-wide tiles
    v.rs = true;
    v.kernel = sfk::fused_step_rs<RT, R, ST, TMR>;
    v.kernel_acc = nullptr;  // FAST with C > 1 runs fused_mc.cuh (every rs radius has an mc variant)
    v.kernel_peer = sfk::fused_step_rs<RT, R, ST, TMR, true>;
    v.box_w = G::BW;
    v.box_h = G::BH;
    return v;
}

// radii beyond (2, 5) (BASELINE c2: 3,7,7; c4: 4,10,10): the t-pass ring in
// tensor memory (a 7- or 9-plane register ring does not fit)
#define SFK_VARIANTS_RS()                                                                  \
    variant_rs<1, 2>(), variant_rs<1, 3>(), variant_rs<2, 4>(), variant_rs<2, 5>(),       \
        variant_rs<3, 7, 2, true>(), variant_rs<4, 10, 2, true>()

// FAST, C > 1: (C + 2)-field launches (fused_mc.cuh): a HEAD (u, Q u, f_1 u)
// and TAILs of one or two channels (f_a u [, f_b u])
struct McVariant {
    int rt, r;
    int threads, box_w, box_h;
    size_t smem[4];          // head (u, Q u, f_1 u), tail of 2 channels, EXACT per channel, head (u, Q u)
    void (*kernel[4])(FusedArgs);
};
// channels folded into the HEAD launch: f_1 for an odd channel count (c4:
// HEAD(3) + one TAIL(2)); none for an even one, where the same number of
// launches then needs no one-channel TAIL (c2: HEAD(2) + four TAIL(2))
constexpr int head_channels(int C) { return C % 2; }

template <int RT, int R>
McVariant variant_mc() {
    McVariant v;
    v.rt = RT;
    v.r = R;
    using GH = sfk::McGeom<RT, R, 3, sfk::MC_HEAD>;
    using G2 = sfk::McGeom<RT, R, 2, sfk::MC_TAIL>;
    using GE = sfk::McGeom<RT, R, 3, sfk::MC_EXACT>;
    using GH2 = sfk::McGeom<RT, R, 2, sfk::MC_HEAD>;
    v.threads = GH::NT;
    v.box_w = GH::BW;
    v.box_h = GH::BH;
    v.smem[0] = GH::SMEM_BYTES;
    v.smem[1] = G2::SMEM_BYTES;
    v.smem[2] = GE::SMEM_BYTES;
    v.kernel[0] = sfk::fused_step_mc<RT, R, 3, sfk::MC_HEAD>;
    v.kernel[1] = sfk::fused_step_mc<RT, R, 2, sfk::MC_TAIL>;
    v.kernel[2] = sfk::fused_step_mc<RT, R, 3, sfk::MC_EXACT>;
    v.smem[3] = GH2::SMEM_BYTES;
    v.kernel[3] = sfk::fused_step_mc<RT, R, 2, sfk::MC_HEAD>;
    return v;
}

const std::vector<McVariant>& mc_variants() {
    // (2, 8): BASELINE c4 with its sub-resolution taps trimmed (trim_kernel)
    static const std::vector<McVariant> v = {variant_mc<2, 5>(), variant_mc<2, 8>(), variant_mc<3, 7>(),
                                             variant_mc<4, 10>()};
    return v;
}

#define SFK_VARIANTS_WS() variant_ws<1, 2>(), variant_ws<1, 3>(), variant_ws<2, 4>(), variant_ws<2, 5>()

// EXACT runs the warp-specialised kernel (fused_ws.cuh), FAST the
// register-streamed one (fused_rs.cuh).
const std::vector<FusedVariant>& variants() {
    static const std::vector<FusedVariant> v = {SFK_VARIANTS_WS(), SFK_VARIANTS_RS()};
    return v;
}

// Host scheduler for the persistent stencil grid: G CTAs, ntiles tiles of
// Tout output frames. Round 1 gives every CTA floor(ntiles/G) whole tiles
// (CTA b: tiles b, b+G, ...), so at any time the CTAs sweep neighbouring
// tiles at the same frame and the halo rows each tile shares with its
// neighbours are served from L2. The R = ntiles mod G remaining tiles are cut
// into c = floor(G/R) time chunks; CTA b takes tile (b mod R) chunk (b div R).
struct Schedule {
    std::vector<int4> seg;
    std::vector<int> off;
};

Schedule build_schedule(int ntiles, int tout, int G) {
    Schedule s;
    std::vector<std::vector<int4>> per(G);
    const int k1 = ntiles / G, rem = ntiles % G;
    for (int b = 0; b < G; ++b)
        for (int j = 0; j < k1; ++j) per[b].push_back(make_int4(j * G + b, 0, tout, 0));
    if (rem > 0) {
        int c = std::max(1, std::min(G / rem, tout));
        const int L = (tout + c - 1) / c;
        c = (tout + L - 1) / L;
        for (int b = 0; b < rem * c && b < G; ++b) {
            const int r = b % rem, k = b / rem;
            const int t0 = k * L, t1 = std::min(tout, (k + 1) * L);
            if (t0 < t1) per[b].push_back(make_int4(k1 * G + r, t0, t1, 0));
        }
    }
    s.off.push_back(0);
    for (int b = 0; b < G; ++b) {
        for (const auto& e : per[b]) s.seg.push_back(e);
        s.off.push_back(static_cast<int>(s.seg.size()));
    }
    return s;
}

bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}

const FusedVariant* pick_variant(int rt, int ry, int rx, bool fma) {
    static const bool force_generic = env_flag("SFSEG_FORCE_GENERIC");
    if (force_generic) return nullptr;
    const int r = std::max(ry, rx);
    const FusedVariant* best = nullptr;
    for (const auto& v : variants())
        if (v.fma == fma && v.rt >= rt && v.r >= r) {
            const long cost = (2L * v.rt + 1) * (2L * v.r + 1);
            if (!best || cost < (2L * best->rt + 1) * (2L * best->r + 1)) best = &v;
        }
    return best;
}

const McVariant* pick_mc(int rt, int ry, int rx) {
    if (env_flag("SFSEG_FORCE_GENERIC")) return nullptr;
    const int r = std::max(ry, rx);
    const McVariant* best = nullptr;
    for (const auto& v : mc_variants())
        if (v.rt >= rt && v.r >= r &&
            (!best || (2L * v.rt + 1) * (2L * v.r + 1) < (2L * best->rt + 1) * (2L * best->r + 1)))
            best = &v;
    return best;
}

// Programmatic dependent launch for the per-iteration chain step -> finalize
// -> step: the next kernel is scheduled while the previous one drains and
// waits in griddep_wait() (every fused kernel and k_finalize call it before
// touching the predecessor's results). SFSEG_PDL=0 turns it off.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SFSEG_PDL");
        return !(e && *e == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t stream,
                Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

}  // namespace

// ---------------------------------------------------------------------------
struct sfseg_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    // resident problem. T = frames in the device buffers; for a time shard
    // the buffer holds global frames [buf_t0, buf_t0 + T) of a Tg-frame
    // problem and the rank outputs frames [out_t0, out_t1).
    int T = 0, H = 0, W = 0, P = 0, C = 0;
    int Tg = 0, buf_t0 = 0, out_t0 = 0, out_t1 = 0, halo = 0;
    bool loaded = false;    // buffers allocated for (T, H, W, C)
    bool resident = false;  // a problem from sfseg_load is in S/F/x0
    bool has_x0 = false;
    float* S = nullptr;
    float* sp = nullptr;
    std::vector<float*> F;       // raw channels as uploaded
    std::vector<float*> Fw;      // guard-rescaled working copies (may alias F)
    bool guard_applied = false;  // Fw reflects the allow_negative_affinity=false guard
    float* x0 = nullptr;
    float* y[2] = {nullptr, nullptr};
    int cur = -1;                // index into y of the current raw iterate (-1: none)
    bool cur_u = false;          // y[cur] holds U = S^p y (fused_mc.cuh write_u), not y
    double sp_p = NAN;           // p that sp was computed for
    // scratch
    double* part = nullptr;
    size_t part_elems = 0;
    double* frame_sum = nullptr;
    float* frame_max = nullptr;
    unsigned int* ticket = nullptr;  // k_finalize's last-block counter (0 between launches)
    IterState* st = nullptr;     // solve state
    IterState* st_aux = nullptr; // stateless operators
    double* norms = nullptr;
    int norms_cap = 0;
    int* flags = nullptr;
    float* scratch_f = nullptr;  // 2 floats + block min/max
    float* bminmax = nullptr;
    double* acc3 = nullptr;
    unsigned long long* cnt2 = nullptr;
    double* conv_part = nullptr;     // convergence statistics (solve_until)
    IterState* st_prev = nullptr;
    // persistent-grid schedule (device copy, keyed by ntiles/Tout/G)
    int4* sched_seg = nullptr;
    int* sched_off = nullptr;
    long long sched_key = -1;
    int sched_busy = 0;  // CTAs with work: a prefix of the grid (build_schedule)
    // generic-path temporaries (allocated lazily)
    std::vector<float*> tmp;
    void* pin[2] = {nullptr, nullptr};  // sfseg_load_files: pinned file-read buffers
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    bool pin_used[2] = {false, false};  // pin_ev[b] marks a DMA still reading pin[b]
    // peer-memory halo exchange (sfseg_shard_set_peers): the neighbours' two
    // iterate buffers, their buffer frame origin, and whether we opened them by IPC
    float* peer_y[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [lo, hi][y index]
    int peer_buf_t0[2] = {0, 0};
    bool peer_ipc[2] = {false, false};
    int peer_push_dst = -1;         // y index the current shard step writes (-1: not a shard step)
    bool pushed_in_kernel = false;  // the step kernel already stored the edge planes to the peers
    float* q = nullptr;              // Q = sum_c f_c^2 of the channel set q_for (fused_mc.cuh)
    std::vector<float*> q_for;
    // dense staging for host transfers (one contiguous DMA, re-pitched on the
    // device) and the device mask of downloads
    float* stage = nullptr;
    size_t stage_elems = 0;
    // pipelined host uploads (load_impl): a copy stream DMAs row chunks into a
    // two-slot staging ring while the library stream re-pitches and validates
    cudaStream_t cstream = nullptr;
    float* ring[2] = {nullptr, nullptr};
    size_t ring_elems = 0;
    cudaEvent_t ring_up[2] = {nullptr, nullptr};  // chunk landed in ring[b]
    cudaEvent_t ring_rp[2] = {nullptr, nullptr};  // ring[b] consumed by its re-pitch
    int* vflags = nullptr;  // per-volume validation flags of a load
    int vflags_n = 0;
    uint8_t* dmask = nullptr;
    size_t dmask_elems = 0;
    // timing
    bool timing = false;
    bool tap_trim = false;  // FAST: drop taps below fp32 resolution (trim_kernel)
    sfseg_timing last_timing{};
    std::vector<cudaEvent_t> ev;
    std::mutex mu;
    sfseg_ctx* scratch = nullptr;  // stateless operators (scratch_ctx)
    std::mutex scratch_mu;
    // sfseg_step on small host volumes: the S / F it uploaded last (host
    // copies), so a caller stepping the same features again (bench.cpp's conv
    // loop, acceptance.cpp check 5) skips their upload and S^p
    uint64_t alloc_gen = 0;  // set_shape reallocations
    bool in_valid = false;
    uint64_t in_gen = 0;
    std::vector<std::vector<float>> in_host;  // S, F_0 .. F_{C-1}
    void* pin_small = nullptr;  // pinned arena of small host transfers (pin_slot)
    size_t pin_small_cap = 0, pin_small_used = 0;

    // volume buffers are allocated with cap_elems >= vol_elems() floats: a
    // context that loads problems of several shapes (sfseg_run_batch, a clip
    // after a clip) reallocates only when a problem outgrows them
    size_t cap_elems = 0;
    int frames_cap = 0;
    size_t vol_elems() const { return static_cast<size_t>(T) * H * P; }
    Vol vol(float* p) const { return Vol{p, T, H, W, P}; }
    int Tout() const { return out_t1 - out_t0; }
    // the rank's output frames inside a buffer
    Vol out_vol(float* p) const {
        return Vol{p + static_cast<size_t>(out_t0 - buf_t0) * H * P, Tout(), H, W, P};
    }
    int nbands() const { return (H + 3) / 4; }
    int nhalves() const { return (W + 31) / 32; }
};

namespace {

// SFSEG_DEBUG_GUARD=1 (tests/test_gpu_guardbands.py; the pool's GPUs refuse
// compute-sanitizer): every volume buffer gets a guard band of kGuard floats
// on either side, bands AND interior are filled with a NaN pattern instead of
// zeros, and sfseg_debug_check_guards counts band words that changed. An
// out-of-bounds store lands in a band; a read of memory no kernel wrote (or
// of the pitch padding) puts a NaN in the result.
constexpr size_t kGuard = 16384;            // floats per band (64 KiB, keeps 128-B alignment)
constexpr uint32_t kPoison = 0x7fc0dead;    // a quiet NaN
bool guard_mode() {
    static const bool on = env_flag("SFSEG_DEBUG_GUARD");
    return on;
}
std::mutex g_guard_mu;
std::vector<std::pair<float*, size_t>> g_guarded;  // (user pointer, floats) of live guarded buffers

__global__ void k_fill_u32(uint32_t* p, size_t n, uint32_t v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}
void poison_fill(float* p, size_t n, cudaStream_t s) {
    k_fill_u32<<<1184, 256, 0, s>>>(reinterpret_cast<uint32_t*>(p), n, kPoison);
    launched(s, "k_fill_u32");
}

void dfree(float*& p) {
    if (p) {
        if (guard_mode()) {
            std::lock_guard<std::mutex> lk(g_guard_mu);
            for (size_t i = 0; i < g_guarded.size(); ++i)
                if (g_guarded[i].first == p) {
                    g_guarded.erase(g_guarded.begin() + i);
                    break;
                }
            cudaFree(p - kGuard);
        } else {
            cudaFree(p);
        }
    }
    p = nullptr;
}

float* dalloc_vol(sfseg_ctx* c) {
    float* p = nullptr;
    const size_t n = std::max(c->cap_elems, c->vol_elems());
    if (guard_mode()) {
        ck(cudaMalloc(&p, (n + 2 * kGuard) * sizeof(float)), "cudaMalloc volume");
        poison_fill(p, n + 2 * kGuard, c->stream);
        std::lock_guard<std::mutex> lk(g_guard_mu);
        g_guarded.emplace_back(p + kGuard, n);
        return p + kGuard;
    }
    ck(cudaMalloc(&p, n * sizeof(float)), "cudaMalloc volume");
    // zero the pitch padding once; kernels never read past W, TMA treats it as OOB
    ck(cudaMemsetAsync(p, 0, n * sizeof(float), c->stream), "memset");
    return p;
}

// forget the neighbours' iterate buffers (sfseg_shard_set_peers)
void drop_peers(sfseg_ctx* c) {
    for (int side = 0; side < 2; ++side) {
        for (int b = 0; b < 2; ++b) {
            if (c->peer_ipc[side] && c->peer_y[side][b]) cudaIpcCloseMemHandle(c->peer_y[side][b]);
            c->peer_y[side][b] = nullptr;
        }
        c->peer_ipc[side] = false;
    }
}

void release_problem(sfseg_ctx* c) {
    if (c->guard_applied)
        for (size_t i = 0; i < c->Fw.size(); ++i)
            if (c->Fw[i] != c->F[i]) dfree(c->Fw[i]);
    c->Fw.clear();
    for (auto*& f : c->F) dfree(f);
    c->F.clear();
    dfree(c->S);
    dfree(c->sp);
    dfree(c->x0);
    dfree(c->y[0]);
    dfree(c->y[1]);
    for (auto*& t : c->tmp) dfree(t);
    c->tmp.clear();
    dfree(c->q);
    c->q_for.clear();
    drop_peers(c);
    if (c->stage) cudaFree(c->stage);
    if (c->dmask) cudaFree(c->dmask);
    c->stage = nullptr;
    c->stage_elems = 0;
    c->dmask = nullptr;
    c->dmask_elems = 0;
    if (c->part) cudaFree(c->part);
    if (c->frame_sum) cudaFree(c->frame_sum);
    if (c->frame_max) cudaFree(c->frame_max);
    c->part = nullptr;
    c->frame_sum = nullptr;
    c->frame_max = nullptr;
    c->part_elems = 0;
    c->frames_cap = 0;
    c->cap_elems = 0;
    c->loaded = false;
    c->resident = false;
    c->cur = -1;
    c->cur_u = false;
    c->sp_p = NAN;
    c->guard_applied = false;
}

// VolumeShape::validate (volume.cpp:39-52) plus this library's own limits:
// each axis, the pitched volume size (overflow-checked: the product of three
// 32-bit extents does not fit 64 bits) and the per-frame reduction blocks
// (an int in the kernels)
void check_shape(uint32_t T, uint32_t H, uint32_t W) {
    if (T == 0 || H == 0 || W == 0) fail(SFSEG_ERR_VALIDATION, "volume shape has an empty axis");
    if (T > (1u << 30) || H > (1u << 20) || W > (1u << 20))
        fail(SFSEG_ERR_CAPACITY, "volume shape exceeds the supported extent");
    const unsigned __int128 bytes = static_cast<unsigned __int128>(T) * H *
                                    ((static_cast<uint64_t>(W) + 31) / 32 * 32) * sizeof(float);
    if (bytes > (static_cast<unsigned __int128>(1) << 40))
        fail(SFSEG_ERR_CAPACITY, "volume exceeds the supported size (1 TiB per field)");
    const uint64_t blocks = (static_cast<uint64_t>(H) + 3) / 4 * ((static_cast<uint64_t>(W) + 31) / 32);
    if (blocks > static_cast<uint64_t>(INT32_MAX) / 64)
        fail(SFSEG_ERR_CAPACITY, "frame exceeds the supported size");
}

void set_shape(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C, int Tg = -1,
               int buf_t0 = 0, int out_t0 = 0, int out_t1 = -1, int halo = 0) {
    if (Tg < 0) Tg = static_cast<int>(T);
    if (out_t1 < 0) out_t1 = Tg;
    if (c->loaded && c->T == (int)T && c->H == (int)H && c->W == (int)W && c->C == C &&
        c->Tg == Tg && c->buf_t0 == buf_t0 && c->out_t0 == out_t0 && c->out_t1 == out_t1)
        return;
    // the buffers of an earlier problem are kept when this one fits in them
    // (same channel count, no more floats per volume): no cudaFree/cudaMalloc
    // (both synchronise the device) between the clips of a batch
    const int P = round_up(static_cast<int>(W), 32);
    const size_t need = static_cast<size_t>(T) * H * P;
    const bool reuse = c->loaded && c->C == C && need <= c->cap_elems;
    const bool same_rows = reuse && c->W == (int)W && c->P == P;
    if (reuse) {
        if (c->guard_applied)
            for (size_t i = 0; i < c->Fw.size(); ++i)
                if (c->Fw[i] != c->F[i]) dfree(c->Fw[i]);
        c->Fw = c->F;
        c->guard_applied = false;
        c->q_for.clear();
        drop_peers(c);
        c->resident = false;
        c->cur = -1;
        c->cur_u = false;
        c->sp_p = NAN;
    } else {
        release_problem(c);
        c->cap_elems = need;
    }
    c->Tg = Tg;
    c->buf_t0 = buf_t0;
    c->out_t0 = out_t0;
    c->out_t1 = out_t1;
    c->halo = halo;
    c->T = T;
    c->H = H;
    c->W = W;
    c->P = P;
    c->C = C;
    ++c->alloc_gen;
    c->in_valid = false;
    if (!reuse) {
        c->S = dalloc_vol(c);
        c->sp = dalloc_vol(c);
        for (int i = 0; i < C; ++i) c->F.push_back(dalloc_vol(c));
        c->Fw = c->F;
        c->y[0] = dalloc_vol(c);
        c->y[1] = dalloc_vol(c);
    } else if (!same_rows) {
        // a different row layout: the pitch padding (columns W .. P-1 of every
        // row) must read as zero again
        auto zero = [&](float* p) {
            if (!p) return;
            if (guard_mode()) {  // keep the padding poisoned (see dalloc_vol)
                poison_fill(p, need, c->stream);
                return;
            }
            ck(cudaMemsetAsync(p, 0, need * sizeof(float), c->stream), "memset");
        };
        zero(c->S);
        zero(c->sp);
        for (float* f : c->F) zero(f);
        zero(c->y[0]);
        zero(c->y[1]);
        zero(c->x0);
        zero(c->q);
        for (float* t : c->tmp) zero(t);
    }
    const int tout = c->Tout();
    const size_t parts = static_cast<size_t>(tout) * c->nbands() * c->nhalves();
    if (parts > c->part_elems) {
        if (c->part) cudaFree(c->part);
        c->part = nullptr;
        c->part_elems = 0;
        ck(cudaMalloc(&c->part, parts * sizeof(double)), "cudaMalloc partials");
        c->part_elems = parts;
    }
    const int frames = std::max(tout, Tg);
    if (frames > c->frames_cap) {
        if (c->frame_sum) cudaFree(c->frame_sum);
        if (c->frame_max) cudaFree(c->frame_max);
        c->frame_sum = nullptr;
        c->frame_max = nullptr;
        c->frames_cap = 0;
        ck(cudaMalloc(&c->frame_sum, frames * sizeof(double)), "cudaMalloc frame sums");
        ck(cudaMalloc(&c->frame_max, frames * sizeof(float)), "cudaMalloc frame max");
        c->frames_cap = frames;
    }
    ck(cudaMemsetAsync(c->frame_max, 0, frames * sizeof(float), c->stream), "memset");
    c->loaded = true;
}

// dense (T,H,W) host/device -> pitched device
float* stage_buf(sfseg_ctx* c) {
    const size_t n = static_cast<size_t>(c->T) * c->H * c->W;
    if (c->stage_elems < n) {
        if (c->stage) cudaFree(c->stage);
        c->stage = nullptr;
        c->stage_elems = 0;
        ck(cudaMalloc(&c->stage, n * sizeof(float)), "cudaMalloc staging");
        c->stage_elems = n;
    }
    return c->stage;
}

// Host volumes move as one dense DMA through a staging buffer and are
// (re)pitched on the device at HBM speed; a 2-D copy of W-float rows would
// run the DMA engine one short row at a time.
// Small host volumes (up to kSmall voxels) are laid out with the device
// pitch in a pinned host buffer and cross the bus as ONE contiguous DMA, no
// re-pitch kernel: at these sizes a kernel launch and a pageable copy cost
// more than the transfer. Slots of the pinned arena are handed out per call
// (every stateless operator ends with a stream synchronisation).
constexpr size_t kSmall = size_t(1) << 18;

float* pin_slot(sfseg_ctx* c, size_t floats) {
    const size_t bytes = (floats * sizeof(float) + 255) / 256 * 256;
    if (c->pin_small_used + bytes > c->pin_small_cap) {
        // wrap (or grow): after a synchronisation nothing in flight uses it
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->pin_small_used = 0;
        if (bytes > c->pin_small_cap) {
            if (c->pin_small) cudaFreeHost(c->pin_small);
            c->pin_small = nullptr;
            c->pin_small_cap = 0;
            const size_t cap = std::max<size_t>(4 * bytes, size_t(4) << 20);
            ck(cudaHostAlloc(&c->pin_small, cap, cudaHostAllocDefault), "cudaHostAlloc");
            std::memset(c->pin_small, 0, cap);  // pitch padding stays 0
            c->pin_small_cap = cap;
        }
    }
    float* p = reinterpret_cast<float*>(static_cast<char*>(c->pin_small) + c->pin_small_used);
    c->pin_small_used += bytes;
    return p;
}

void upload(sfseg_ctx* c, float* dst, const float* src, int32_t mem) {
    const size_t rows = static_cast<size_t>(c->T) * c->H;
    if (mem == SFSEG_MEM_HOST && rows * c->W <= kSmall) {
        float* pin = pin_slot(c, rows * c->P);
        for (size_t r = 0; r < rows; ++r) std::memcpy(pin + r * c->P, src + r * c->W, c->W * sizeof(float));
        ck(cudaMemcpyAsync(dst, pin, rows * c->P * sizeof(float), cudaMemcpyHostToDevice, c->stream),
           "upload volume");
        return;
    }
    if (mem == SFSEG_MEM_DEVICE || c->P == c->W) {
        ck(cudaMemcpy2DAsync(dst, c->P * sizeof(float), src, c->W * sizeof(float), c->W * sizeof(float),
                             rows, mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             c->stream),
           "upload volume");
        return;
    }
    float* st = stage_buf(c);
    ck(cudaMemcpyAsync(st, src, rows * c->W * sizeof(float), cudaMemcpyHostToDevice, c->stream),
       "upload volume");
    sfk::k_repitch<<<c->num_sms * 8, 256, 0, c->stream>>>(st, c->W, dst, c->P, rows, c->W);
    launched(c->stream, "k_repitch");
}

// (small host volumes: synchronous, see pin_slot)
void download(sfseg_ctx* c, float* dst, const float* src, int32_t mem) {
    const size_t rows = static_cast<size_t>(c->T) * c->H;
    if (mem == SFSEG_MEM_HOST && rows * c->W <= kSmall) {
        float* pin = pin_slot(c, rows * c->P);
        ck(cudaMemcpyAsync(pin, src, rows * c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
           "download volume");
        ck(cudaStreamSynchronize(c->stream), "download");
        for (size_t r = 0; r < rows; ++r) std::memcpy(dst + r * c->W, pin + r * c->P, c->W * sizeof(float));
        return;
    }
    if (mem == SFSEG_MEM_DEVICE || c->P == c->W) {
        ck(cudaMemcpy2DAsync(dst, c->W * sizeof(float), src, c->P * sizeof(float), c->W * sizeof(float),
                             rows, mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             c->stream),
           "download volume");
        return;
    }
    float* st = stage_buf(c);
    sfk::k_repitch<<<c->num_sms * 8, 256, 0, c->stream>>>(src, c->P, st, c->W, rows, c->W);
    launched(c->stream, "k_repitch");
    ck(cudaMemcpyAsync(dst, st, rows * c->W * sizeof(float), cudaMemcpyDeviceToHost, c->stream),
       "download volume");
}

int aux_grid(sfseg_ctx* c) { return c->num_sms * 8; }

void validate_vol(sfseg_ctx* c, float* v, bool nonneg, const char* what) {
    ck(cudaMemsetAsync(c->flags, 0, sizeof(int), c->stream), "memset flags");
    sfk::k_validate<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(v), nonneg, c->flags);
    launched(c->stream, "k_validate");
    int h = 0;
    ck(cudaMemcpyAsync(&h, c->flags, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "flags");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (h & 1) fail(SFSEG_ERR_VALIDATION, std::string(what) + " contains a non-finite value");
    if (h & 2)
        fail(SFSEG_ERR_VALIDATION,
             std::string(what) + ": unary/solution volume contains a negative value");
}

// S^p for the resident S (cached per p)
void ensure_sp(sfseg_ctx* c, double p) {
    if (c->sp_p == p) return;
    sfk::k_pow<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->S), c->vol(c->sp), p);
    launched(c->stream, "k_pow");
    c->sp_p = p;
}

// guard rescale of the pairwise channels (engine.cpp:255-259)
void ensure_guard(sfseg_ctx* c, bool guard) {
    if (!guard) {
        if (c->guard_applied) {
            for (size_t i = 0; i < c->Fw.size(); ++i)
                if (c->Fw[i] != c->F[i]) dfree(c->Fw[i]);
            c->Fw = c->F;
            c->guard_applied = false;
        }
        return;
    }
    if (c->guard_applied) return;
    const int nb = aux_grid(c);
    for (int i = 0; i < c->C; ++i) {
        sfk::k_minmax_blocks<<<nb, sfk::kAuxThreads, 0, c->stream>>>(
            c->vol(c->F[i]), c->bminmax, c->bminmax + nb);
        sfk::k_minmax_final<<<1, sfk::kAuxThreads, 0, c->stream>>>(c->bminmax, c->bminmax + nb,
                                                                 nb, c->scratch_f);
        float lohi[2];
        ck(cudaMemcpyAsync(lohi, c->scratch_f, sizeof lohi, cudaMemcpyDeviceToHost, c->stream),
           "minmax");
        ck(cudaStreamSynchronize(c->stream), "sync");
        if (lohi[0] >= 0.0f && lohi[1] <= 1.0f) continue;  // bits untouched
        float* w = dalloc_vol(c);
        ck(cudaMemcpyAsync(w, c->F[i], c->vol_elems() * sizeof(float), cudaMemcpyDeviceToDevice,
                           c->stream),
           "copy channel");
        sfk::k_unit_range<<<nb, sfk::kAuxThreads, 0, c->stream>>>(c->vol(w), c->scratch_f);
        launched(c->stream, "k_unit_range");
        c->Fw[i] = w;
    }
    c->guard_applied = true;
}

void upload_schedule(sfseg_ctx* c, int ntiles, int tout, int G) {
    const long long key = (static_cast<long long>(ntiles) << 40) ^
                          (static_cast<long long>(tout) << 16) ^ G;
    if (key == c->sched_key) return;
    const Schedule s = build_schedule(ntiles, tout, G);
    c->sched_busy = 0;
    for (int b = 0; b < G; ++b)
        if (s.off[b + 1] > s.off[b]) c->sched_busy = b + 1;
    if (c->sched_seg) cudaFree(c->sched_seg);
    if (c->sched_off) cudaFree(c->sched_off);
    c->sched_seg = nullptr;
    c->sched_off = nullptr;
    ck(cudaMalloc(&c->sched_seg, std::max<size_t>(1, s.seg.size()) * sizeof(int4)), "malloc");
    ck(cudaMalloc(&c->sched_off, s.off.size() * sizeof(int)), "malloc");
    ck(cudaMemcpyAsync(c->sched_seg, s.seg.data(), s.seg.size() * sizeof(int4),
                       cudaMemcpyHostToDevice, c->stream),
       "schedule");
    ck(cudaMemcpyAsync(c->sched_off, s.off.data(), s.off.size() * sizeof(int),
                       cudaMemcpyHostToDevice, c->stream),
       "schedule");
    ck(cudaStreamSynchronize(c->stream), "schedule");
    c->sched_key = key;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to a device's context:
// set once per (device, kernel), thread-safe, before the first launch
void ensure_smem_attr(sfseg_ctx* c, void (*fn)(FusedArgs), size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<int, void (*)(FusedArgs)>> done;
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& d : done)
        if (d.first == c->device && d.second == fn) return;
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    done.emplace_back(c->device, fn);
}

void fill_taps(FusedArgs& a, const HostKernel& k, const FusedVariant& v) {
    std::memset(a.taps_x, 0, sizeof a.taps_x);
    std::memset(a.taps_y, 0, sizeof a.taps_y);
    std::memset(a.taps_t, 0, sizeof a.taps_t);
    // centre the real taps inside the variant's support; outer taps stay 0
    for (int i = 0; i <= 2 * k.rx; ++i) a.taps_x[v.r - k.rx + i] = static_cast<float>(k.x[i]);
    for (int i = 0; i <= 2 * k.ry; ++i) a.taps_y[v.r - k.ry + i] = static_cast<float>(k.y[i]);
    for (int i = 0; i <= 2 * k.rt; ++i) a.taps_t[v.rt - k.rt + i] = static_cast<float>(k.t[i]);
    for (int e = 0; e <= 2 * v.r + 1 && e <= sfk::kMaxTapsXY; ++e) {
        const float x0 = e <= 2 * v.r ? a.taps_x[e] : 0.0f, x1 = e >= 1 ? a.taps_x[e - 1] : 0.0f;
        const float y0 = e <= 2 * v.r ? a.taps_y[e] : 0.0f, y1 = e >= 1 ? a.taps_y[e - 1] : 0.0f;
        a.tpair_x[e] = make_float2(x0, x1);
        a.tpair_y[e] = make_float2(y0, y1);
    }
}

float* tmp_vol(sfseg_ctx* c, size_t i) {
    while (c->tmp.size() <= i) c->tmp.push_back(dalloc_vol(c));
    return c->tmp[i];
}

// Q = sum_c f_c^2 for the channel set Fch (cached until the channels change)
float* ensure_q(sfseg_ctx* c, const std::vector<float*>& Fch) {
    if (c->q && c->q_for == Fch) return c->q;
    if (!c->q) c->q = dalloc_vol(c);
    for (size_t i = 0; i < Fch.size(); ++i)
        sfk::k_sq_acc<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->q), c->vol(Fch[i]),
                                                                      i == 0);
    launched(c->stream, "k_sq_acc");
    c->q_for = Fch;
    return c->q;
}

// FAST step for C > 1 channels in the (C + 2)-field form (fused_mc.cuh): a
// HEAD launch (u, Q u, f_1 u) and ceil((C - 1) / 2) TAIL launches of one or
// two channels accumulating into y; the last launch emits the reductions and
// stores U_{k+1} = S^p y_{k+1} instead of y_{k+1} when write_u. The u field
// is read from x_src when src_is_u (the previous step stored U), else made
// by k_make_u. EXACT (exact = true): one launch per channel, the reference's
// per-channel form.
void launch_step_mc(sfseg_ctx* c, const HostKernel& k, double alpha, const float* x_src,
                    const IterState* st, float* out, const std::vector<float*>& Fch,
                    const McVariant& v, bool exact, bool src_is_u, bool write_u) {
    float* q = exact ? nullptr : ensure_q(c, Fch);
    const float* u = x_src;
    if (!exact && !src_is_u) {
        float* ub = tmp_vol(c, 0);
        launch_pdl(sfk::k_make_u, aux_grid(c), sfk::kAuxThreads, 0, c->stream, c->vol(const_cast<float*>(x_src)),
                   c->vol(c->sp), c->vol(ub), st);
        launched(c->stream, "k_make_u");
        u = ub;
    }
    FusedVariant fv;  // taps / tensor-map geometry
    fv.rt = v.rt;
    fv.r = v.r;
    fv.ty = 64;
    fv.tx = 32;
    FusedArgs a;
    std::memset(&a, 0, sizeof a);
    a.tm_sp = make_tmap(c->sp, c->T, c->H, c->W, c->P, v.box_w, v.box_h);
    a.tm_out = make_tmap(out, c->T, c->H, c->W, c->P, fv.tx, 8);
    a.tm_spc = make_tmap(c->sp, c->T, c->H, c->W, c->P, fv.tx, 8);
    a.sp = c->sp;
    a.out = out;
    a.part = c->part;
    a.frame_max = c->frame_max;
    a.part_t0 = c->out_t0;
    a.st = st;
    fill_taps(a, k, fv);
    a.inv_alpha = static_cast<float>(1.0 / alpha);
    a.c_inv_alpha = static_cast<float>(static_cast<double>(Fch.size()) / alpha);
    a.one = 1.0f;
    a.zero = 0.0f;
    a.T = c->Tg;
    a.H = c->H;
    a.W = c->W;
    a.pitch = c->P;
    a.buf_t0 = c->buf_t0;
    a.out_t0 = c->out_t0;
    a.out_t1 = c->out_t1;
    a.out_buf_t0 = c->buf_t0;
    a.tiles_x = (c->W + fv.tx - 1) / fv.tx;
    a.tiles_y = (c->H + fv.ty - 1) / fv.ty;
    a.nbands = c->nbands();
    a.nhalves = c->nhalves();
    const int grid_n = c->num_sms;
    upload_schedule(c, a.tiles_x * a.tiles_y, c->Tout(), grid_n);
    a.sched = c->sched_seg;
    a.sched_off = c->sched_off;
    for (int i = 0; i < 4; ++i) ensure_smem_attr(c, v.kernel[i], v.smem[i]);
    const int C = static_cast<int>(Fch.size());
    const int hc = head_channels(C);
    const int ntail = exact ? C - 1 : (C - hc + 1) / 2;
    for (int g = 0; g <= ntail; ++g) {
        int kind = 0;
        if (exact) {  // one launch per channel: boxes x, S^p, f_g; operands S^p, f_g, y
            kind = 2;
            a.tm_x = make_tmap(x_src, c->T, c->H, c->W, c->P, v.box_w, v.box_h);
            a.tm_f[0] = make_tmap(Fch[g], c->T, c->H, c->W, c->P, v.box_w, v.box_h);
            a.tm_fc[0] = make_tmap(Fch[g], c->T, c->H, c->W, c->P, fv.tx, 8);
        } else if (g == 0) {  // boxes U, Q [, f_1]; operands S^p, Q [, f_1]
            kind = hc ? 0 : 3;
            a.tm_x = make_tmap(u, c->T, c->H, c->W, c->P, v.box_w, v.box_h);
            a.tm_f[0] = make_tmap(q, c->T, c->H, c->W, c->P, v.box_w, v.box_h);
            a.tm_fc[0] = make_tmap(q, c->T, c->H, c->W, c->P, fv.tx, 8);
            if (hc) {
                a.tm_f[1] = make_tmap(Fch[0], c->T, c->H, c->W, c->P, v.box_w, v.box_h);
                a.tm_fc[1] = make_tmap(Fch[0], c->T, c->H, c->W, c->P, fv.tx, 8);
            }
        } else {  // boxes U, f_a, f_b; operands S^p, f_a, f_b, y (C - hc is even: always two channels)
            const int c0 = hc + 2 * (g - 1), n = 2;
            kind = 1;
            for (int i = 0; i < n; ++i) {
                a.tm_f[i] = make_tmap(Fch[c0 + i], c->T, c->H, c->W, c->P, v.box_w, v.box_h);
                a.tm_fc[i] = make_tmap(Fch[c0 + i], c->T, c->H, c->W, c->P, fv.tx, 8);
            }
        }
        a.first_group = g == 0;
        a.last_group = g == ntail;
        a.write_u = !exact && g == ntail && write_u;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->timing) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, c->stream);
        }
        launch_pdl(v.kernel[kind], c->sched_busy, v.threads, v.smem[kind], c->stream, a);
        launched(c->stream, "fused_step_mc launch");
        if (c->timing) {
            cudaEventRecord(e1, c->stream);
            c->ev.push_back(e0);
            c->ev.push_back(e1);
        }
    }
}

// One step y_out = sum_c step_c(T(x_src)) with fused kernels or the generic
// multi-pass path; emits canonical partials + frame max into c->part /
// c->frame_max for the whole volume.
// src_is_u: x_src holds U = S^p x (a previous FAST multi-channel step stored
// it); write_u: the step may store U_{k+1} instead of y_{k+1}. Returns
// whether it did (only the multi-channel FAST path does).
bool launch_step(sfseg_ctx* c, const HostKernel& k_full, double alpha, const float* x_src,
                 const IterState* st, float* out, const std::vector<float*>& Fch, bool fma,
                 bool src_is_u = false, bool write_u = false) {
    const HostKernel k_trim = (fma && c->tap_trim) ? trim_kernel(k_full) : HostKernel();
    const HostKernel& k = (fma && c->tap_trim) ? k_trim : k_full;
    const float inv_alpha = static_cast<float>(1.0 / alpha);
    const FusedVariant* v = pick_variant(k.rt, k.ry, k.rx, fma);
    g_conv_count.fetch_add(3ull * Fch.size(), std::memory_order_relaxed);
    c->pushed_in_kernel = false;
    const McVariant* mc = (fma && Fch.size() > 1) ? pick_mc(k.rt, k.ry, k.rx) : nullptr;
    if (mc) {
        launch_step_mc(c, k, alpha, x_src, st, out, Fch, *mc, false, src_is_u, write_u);
        return write_u;
    }
    if (src_is_u && !(v && v->rs)) fail(SFSEG_ERR_STATE, "iterate stored as S^p y for another step path");
    // EXACT beyond the warp-specialised instantiations (c2, c4 radii): the
    // per-channel EXACT launches of fused_mc.cuh
    const McVariant* mce = (!fma && !v) ? pick_mc(k.rt, k.ry, k.rx) : nullptr;
    if (mce) {
        launch_step_mc(c, k, alpha, x_src, st, out, Fch, *mce, true, false, false);
        return false;
    }
    if (v) {
        // the FAST kernel (fused_rs.cuh) reads u = S^p x as a volume: the
        // previous step's U store, or k_make_u; it stores U_{k+1} on request
        const float* xin = x_src;
        const bool wu = v->rs && write_u;
        if (v->rs && !src_is_u) {
            float* ub = tmp_vol(c, 0);
            launch_pdl(sfk::k_make_u, aux_grid(c), sfk::kAuxThreads, 0, c->stream,
                       c->vol(const_cast<float*>(x_src)), c->vol(c->sp), c->vol(ub), st);
            launched(c->stream, "k_make_u");
            xin = ub;
        }
        FusedArgs a;
        std::memset(&a, 0, sizeof a);
        a.write_u = wu;
        a.tm_x = make_tmap(xin, c->T, c->H, c->W, c->P, v->box_w, v->box_h);
        a.tm_sp = make_tmap(c->sp, c->T, c->H, c->W, c->P, v->box_w, v->box_h);
        a.tm_out = make_tmap(out, c->T, c->H, c->W, c->P, v->tx, v->slab_h);
        a.tm_spc = make_tmap(c->sp, c->T, c->H, c->W, c->P, v->tx, v->slab_h);
        a.sp = c->sp;
        a.out = out;
        a.part = c->part;
        a.frame_max = c->frame_max;
        a.part_t0 = c->out_t0;
        a.st = st;
        fill_taps(a, k, *v);
        a.inv_alpha = inv_alpha;
        a.one = 1.0f;
        a.zero = 0.0f;
        a.T = c->Tg;
        a.H = c->H;
        a.W = c->W;
        a.pitch = c->P;
        a.buf_t0 = c->buf_t0;
        a.out_t0 = c->out_t0;
        a.out_t1 = c->out_t1;
        a.out_buf_t0 = c->buf_t0;
        a.tiles_x = (c->W + v->tx - 1) / v->tx;
        a.tiles_y = (c->H + v->ty - 1) / v->ty;
        a.nbands = c->nbands();
        a.nhalves = c->nhalves();
        const int ntiles = a.tiles_x * a.tiles_y;
        const int grid_n = c->num_sms;
        upload_schedule(c, ntiles, c->Tout(), grid_n);
        a.sched = c->sched_seg;
        a.sched_off = c->sched_off;
        for (auto kfn : {v->kernel, v->kernel_acc, v->kernel_peer})
            if (kfn) ensure_smem_attr(c, kfn, v->smem);
        // the FAST stencil (fused_rs.cuh) pushes the sharded solve's edge
        // planes to the peers itself; other kernels leave it to k_halo_push
        c->pushed_in_kernel = false;
        if (fma && c->peer_push_dst >= 0 && v->kernel_peer && Fch.size() == 1) {
            const int nh = std::min(c->halo, c->Tout());
            for (int side = 0; side < 2; ++side) {
                a.peer[side] = c->peer_y[side][c->peer_push_dst];
                a.peer_t0[side] = c->peer_buf_t0[side];
            }
            a.peer_n = nh;
            c->pushed_in_kernel = a.peer[0] || a.peer[1];
        }
        if (Fch.size() > 1 && !v->kernel_acc) fail(SFSEG_ERR_STATE, "no accumulating kernel for this variant");
        for (size_t g = 0; g < Fch.size(); ++g) {
            a.tm_f[0] = make_tmap(Fch[g], c->T, c->H, c->W, c->P, v->box_w, v->box_h);
            a.tm_fc[0] = make_tmap(Fch[g], c->T, c->H, c->W, c->P, v->tx, v->slab_h);
            a.f[0] = Fch[g];
            a.first_group = g == 0;
            a.last_group = g + 1 == Fch.size();
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (c->timing) {
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0, c->stream);
            }
            launch_pdl(c->pushed_in_kernel ? v->kernel_peer : g == 0 ? v->kernel : v->kernel_acc, c->sched_busy,
                       v->threads, v->smem, c->stream, a);
            launched(c->stream, "fused_step launch");
            if (c->timing) {
                cudaEventRecord(e1, c->stream);
                c->ev.push_back(e0);
                c->ev.push_back(e1);
            }
        }
        return wu;
    }
    // generic multi-pass path (radii beyond the fused instantiations)
    sfk::Taps tp;
    std::memset(&tp, 0, sizeof tp);
    if (k.rt > 31 || k.ry > 31 || k.rx > 31) fail(SFSEG_ERR_CAPACITY, "kernel radius above 31");
    for (int i = 0; i <= 2 * k.rt; ++i) tp.t[i] = static_cast<float>(k.t[i]);
    for (int i = 0; i <= 2 * k.ry; ++i) tp.y[i] = static_cast<float>(k.y[i]);
    for (int i = 0; i <= 2 * k.rx; ++i) tp.x[i] = static_cast<float>(k.x[i]);
    tp.rt = k.rt;
    tp.ry = k.ry;
    tp.rx = k.rx;
    const int g = aux_grid(c), bt = sfk::kAuxThreads;
    float *u = tmp_vol(c, 0), *fu = tmp_vol(c, 1), *f2u = tmp_vol(c, 2);
    float *ca = tmp_vol(c, 3), *cb = tmp_vol(c, 4), *cc = tmp_vol(c, 5);
    float *t0 = tmp_vol(c, 6), *t1 = tmp_vol(c, 7);
    Vol xs = c->vol(const_cast<float*>(x_src));
    for (size_t ch = 0; ch < Fch.size(); ++ch) {
        sfk::k_products<<<g, bt, 0, c->stream>>>(xs, c->vol(c->sp), c->vol(Fch[ch]), c->vol(u),
                                                 c->vol(fu), c->vol(f2u), st);
        const float* srcs[3] = {u, f2u, fu};
        float* dsts[3] = {ca, cb, cc};
        for (int q = 0; q < 3; ++q) {
            sfk::k_pass_x<<<g, bt, 0, c->stream>>>(c->vol(const_cast<float*>(srcs[q])), c->vol(t0), tp);
            sfk::k_pass_y<<<g, bt, 0, c->stream>>>(c->vol(t0), c->vol(t1), tp);
            sfk::k_pass_t<<<g, bt, 0, c->stream>>>(c->vol(t1), c->vol(dsts[q]), tp);
        }
        sfk::k_recombine<<<g, bt, 0, c->stream>>>(c->vol(ca), c->vol(cb), c->vol(cc),
                                                  c->vol(c->sp), c->vol(Fch[ch]), c->vol(out),
                                                  inv_alpha, ch == 0);
        launched(c->stream, "generic step");
    }
    const long long warps = static_cast<long long>(c->Tout()) * c->nbands() * c->nhalves();
    sfk::k_partials<<<static_cast<int>((warps * 32 + 255) / 256), 256, 0, c->stream>>>(
        c->out_vol(out), c->part, c->frame_max, c->nbands(), c->nhalves(), 0);
    launched(c->stream, "k_partials");
    return false;
}

void frame_sums(sfseg_ctx* c) {
    const int per_frame = c->nbands() * c->nhalves();
    launch_pdl(sfk::k_finalize_frames, c->Tout(), sfk::kAuxThreads, 0, c->stream,
               static_cast<const double*>(c->part), per_frame, c->frame_sum, 0);
    launched(c->stream, "k_finalize_frames");
}

void finalize(sfseg_ctx* c, IterState* st, double* norms, int iter_index, int mode_next,
              double lambda, double frac) {
    launch_pdl(sfk::k_finalize, c->Tout(), sfk::kAuxThreads, 0, c->stream, c->part,
               c->nbands() * c->nhalves(), c->frame_sum, c->frame_max, c->ticket, st, norms,
               iter_index, mode_next, lambda, frac);
    launched(c->stream, "k_finalize");
}

// the state goes by value in the launch parameters (no host buffer that has
// to outlive the call: the sharded loop may be captured into a CUDA graph)
__global__ void k_set_state(IterState* dst, const IterState s) { *dst = s; }

void set_state(sfseg_ctx* c, IterState* dst, const IterState& s) {
    k_set_state<<<1, 1, 0, c->stream>>>(dst, s);
    launched(c->stream, "k_set_state");
}

IterState get_state(sfseg_ctx* c, const IterState* src) {
    IterState s;
    ck(cudaMemcpyAsync(&s, src, sizeof s, cudaMemcpyDeviceToHost, c->stream), "state");
    ck(cudaStreamSynchronize(c->stream), "sync");
    return s;
}

double lambda_for(const sfseg_params* p, int iter) {
    return p->sigmoid_slope0 * std::pow(p->slope_growth, iter - p->binarize_start);
}

// iterate currently visible to the caller = T_state(y[cur]) (or S/x0 before
// the first iteration)
void materialize(sfseg_ctx* c, float* out) {
    if (c->cur < 0) {
        ck(cudaMemcpyAsync(out, c->has_x0 ? c->x0 : c->S, c->vol_elems() * sizeof(float),
                           cudaMemcpyDeviceToDevice, c->stream),
           "copy x");
        return;
    }
    sfk::k_transform<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->y[c->cur]),
                                                                    c->vol(out), c->st);
    launched(c->stream, "k_transform");
}

void solve_impl(sfseg_ctx* c, const sfseg_params* p, int first, int last,
                sfseg_iter_record* rec) {
    validate_params(p);
    if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_solve before sfseg_load");
    if (first < 1 || last < first) fail(SFSEG_ERR_PARAMETER, "bad iteration range");
    if (first > 1 && c->cur < 0) fail(SFSEG_ERR_STATE, "continuing a solve that never started");
    const HostKernel k = make_kernel(p->radii, p->sigmas);
    ensure_guard(c, !p->allow_negative_affinity);
    ensure_sp(c, p->p);
    const int n = last - first + 1;
    if (c->norms_cap < n) {
        if (c->norms) cudaFree(c->norms);
        ck(cudaMalloc(&c->norms, n * sizeof(double)), "cudaMalloc norms");
        c->norms_cap = n;
    }
    if (first == 1) {
        IterState s{};
        s.mode = 0;
        set_state(c, c->st, s);
        ck(cudaMemsetAsync(c->frame_max, 0, c->Tout() * sizeof(float), c->stream), "memset");
        c->cur = -1;
        c->cur_u = false;
    }
    for (auto e : c->ev) cudaEventDestroy(e);
    c->ev.clear();
    std::vector<cudaEvent_t> iter_ev(n + 1);
    for (auto& e : iter_ev) ck(cudaEventCreate(&e), "event");
    ck(cudaEventRecord(iter_ev[0], c->stream), "event");
    for (int it = first; it <= last; ++it) {
        const float* src = c->cur < 0 ? (c->has_x0 ? c->x0 : c->S) : c->y[c->cur];
        const int dst = c->cur < 0 ? 0 : 1 - c->cur;
        // U_{k+1} = S^p y_{k+1} replaces y_{k+1} when the next iteration of
        // this solve only normalises; the last one leaves y for the caller
        const bool wu = it < last && it < p->binarize_start;
        c->cur_u = launch_step(c, k, p->alpha, src, c->st, c->y[dst], c->Fw,
                               p->arith == SFSEG_ARITH_FAST, c->cur >= 0 && c->cur_u, wu);
        const int mode_next = it >= p->binarize_start ? 2 : 1;
        finalize(c, c->st, c->norms, it - first, mode_next, lambda_for(p, it), p->threshold_frac);
        c->cur = dst;
        // per-iteration events only when per-iteration times are wanted: an
        // event between two kernels stops the programmatic (PDL) overlap
        if (rec || c->timing || it == last) ck(cudaEventRecord(iter_ev[it - first + 1], c->stream), "event");
    }
    std::vector<double> norms(n);
    ck(cudaMemcpyAsync(norms.data(), c->norms, n * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream),
       "norms");
    ck(cudaStreamSynchronize(c->stream), "solve");
    sfseg_timing tm{};
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, iter_ev[0], iter_ev[n]);
    tm.solve_ms = ms;
    for (size_t i = 0; i + 1 < c->ev.size(); i += 2) {
        float m = 0.0f;
        cudaEventElapsedTime(&m, c->ev[i], c->ev[i + 1]);
        tm.step_kernel_ms += m;
        ++tm.step_launches;
    }
    c->last_timing = tm;
    for (int i = 0; i < n; ++i) {
        if (rec) {
            rec[i].iter = first + i;
            rec[i].l2_norm_pre_normalize = norms[i];
            rec[i].angle_deg = NAN;
            rec[i].iou = NAN;
            float m = 0.0f;
            cudaEventElapsedTime(&m, iter_ev[i], iter_ev[i + 1]);
            rec[i].wall_time_s = m * 1e-3;
        }
    }
    for (auto e : iter_ev) cudaEventDestroy(e);
    for (int i = 0; i < n; ++i)
        if (norms[i] == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
}

// Fixed-count solve with an early exit: the reference's
// run() always runs cfg.iterations; power_iteration stops once
// ||x_k - x_{k-1}||_2 < tol (oracle.cpp:234-242) and bench.cpp's
// converged_conv once angle(x_k, x_{k-1}) < tol degrees (bench.cpp:75-80,
// metrics.cpp:22-38). Each iteration is the same fused step + finalize as
// solve_impl, then k_conv_stats against the previous projected iterate and
// k_conv_final, which evaluates the rule ON THE DEVICE and raises the state's
// stop flag; the kernels of later iterations already in the stream see the
// flag and return, so the iterate stays at the stopping iteration. Iterations
// are enqueued in chunks and the host reads the flag back once per chunk: no
// host round trip per iteration.
void solve_until_impl(sfseg_ctx* c, const sfseg_params* p, int first, int max_iter, int criterion,
                      double tol, int32_t* done, sfseg_iter_record* rec) {
    if (criterion != SFSEG_CONV_STEP && criterion != SFSEG_CONV_ANGLE)
        fail(SFSEG_ERR_PARAMETER, "unknown convergence criterion");
    if (!(tol >= 0.0)) fail(SFSEG_ERR_PARAMETER, "tolerance must be >= 0");
    validate_params(p);
    if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_solve_until before sfseg_load");
    if (first < 1 || max_iter < first) fail(SFSEG_ERR_PARAMETER, "bad iteration range");
    if (first > 1 && c->cur < 0) fail(SFSEG_ERR_STATE, "continuing a solve that never started");
    const HostKernel k = make_kernel(p->radii, p->sigmas);
    ensure_guard(c, !p->allow_negative_affinity);
    ensure_sp(c, p->p);
    const int nb = aux_grid(c);
    if (!c->conv_part) {
        ck(cudaMalloc(&c->conv_part, (static_cast<size_t>(nb) * 4 + 4) * sizeof(double)), "malloc");
        ck(cudaMalloc(&c->st_prev, sizeof(IterState)), "malloc");
    }
    const int nmax = max_iter - first + 1;
    if (c->norms_cap < nmax) {
        if (c->norms) cudaFree(c->norms);
        c->norms = nullptr;
        c->norms_cap = 0;
        ck(cudaMalloc(&c->norms, nmax * sizeof(double)), "cudaMalloc norms");
        c->norms_cap = nmax;
    }
    if (first == 1) {
        IterState s{};
        s.mode = 0;
        set_state(c, c->st, s);
        ck(cudaMemsetAsync(c->frame_max, 0, c->Tout() * sizeof(float), c->stream), "memset");
        c->cur = -1;
        c->cur_u = false;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, c->stream), "event");
    constexpr int kChunk = 8;  // iterations per flag read-back
    std::vector<int> cur_after(nmax, -1);  // y index holding the iterate after iteration first + i
    int it = first, stop = 0;
    while (it <= max_iter && stop == 0) {
        const int chunk_end = std::min(max_iter, it + kChunk - 1);
        for (; it <= chunk_end; ++it) {
            // x_{k-1}: the visible iterate before this step
            const bool prev_raw = c->cur < 0;
            const float* prev = prev_raw ? (c->has_x0 ? c->x0 : c->S) : c->y[c->cur];
            const int dst = c->cur < 0 ? 0 : 1 - c->cur;
            ck(cudaMemcpyAsync(c->st_prev, c->st, sizeof(IterState), cudaMemcpyDeviceToDevice, c->stream),
               "state copy");
            // every iteration may be the last one: the iterate stays y (no U carry)
            c->cur_u = launch_step(c, k, p->alpha, prev, c->st, c->y[dst], c->Fw,
                                   p->arith == SFSEG_ARITH_FAST, c->cur >= 0 && c->cur_u, false);
            const int mode_next = it >= p->binarize_start ? 2 : 1;
            finalize(c, c->st, c->norms, it - first, mode_next, lambda_for(p, it), p->threshold_frac);
            c->cur = dst;
            cur_after[it - first] = dst;
            sfk::k_conv_stats<<<nb, sfk::kAuxThreads, 0, c->stream>>>(
                c->vol(c->y[dst]), c->st, c->vol(const_cast<float*>(prev)), c->st_prev, prev_raw,
                c->conv_part);
            sfk::k_conv_final<<<1, 32, 0, c->stream>>>(c->conv_part, nb, c->conv_part + 4 * nb, c->st,
                                                       it, criterion, tol);
            launched(c->stream, "k_conv_stats");
        }
        stop = get_state(c, c->st).stop;  // one read-back (and sync) per chunk
    }
    ck(cudaEventRecord(e1, c->stream), "event");
    const int last = stop != 0 ? std::abs(stop) : max_iter;  // last iteration that really ran
    const int n = last - first + 1;
    std::vector<double> norms(n);
    ck(cudaMemcpyAsync(norms.data(), c->norms, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
       "norms");
    sfk::k_clear_stop<<<1, 1, 0, c->stream>>>(c->st);
    launched(c->stream, "k_clear_stop");
    ck(cudaStreamSynchronize(c->stream), "solve_until");
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // the host's view of the iterate: what iteration `last` wrote
    c->cur = cur_after[n - 1];
    c->cur_u = false;
    sfseg_timing tm{};
    tm.solve_ms = ms;
    c->last_timing = tm;
    if (rec)
        for (int i = 0; i < n; ++i) {
            rec[i].iter = first + i;
            rec[i].l2_norm_pre_normalize = norms[i];
            rec[i].angle_deg = NAN;
            rec[i].iou = NAN;
            rec[i].wall_time_s = ms * 1e-3 / std::max(1, it - first);  // mean over the enqueued iterations
        }
    *done = last;
    for (int i = 0; i < n; ++i)
        if (norms[i] == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
    if (stop < 0) fail(SFSEG_ERR_PARAMETER, "angle is undefined for a zero vector");
}

// The copy stream and the two-slot staging ring of pipelined host transfers;
// returns the rows per chunk (32 MB chunks).
size_t ensure_ring(sfseg_ctx* c) {
    if (!c->cstream) ck(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking), "stream");
    const size_t W = c->W, rows = static_cast<size_t>(c->T) * c->H;
    const size_t chunk_rows = std::max<size_t>(1, (size_t(32) << 20) / (W * sizeof(float)));
    const size_t need = std::min(rows, chunk_rows) * W;
    if (c->ring_elems < need) {
        for (int b = 0; b < 2; ++b) {
            if (c->ring[b]) cudaFree(c->ring[b]);
            c->ring[b] = nullptr;
        }
        c->ring_elems = 0;
        for (int b = 0; b < 2; ++b) ck(cudaMalloc(&c->ring[b], need * sizeof(float)), "malloc ring");
        c->ring_elems = need;
    }
    for (int b = 0; b < 2; ++b) {
        if (!c->ring_up[b]) ck(cudaEventCreateWithFlags(&c->ring_up[b], cudaEventDisableTiming), "event");
        if (!c->ring_rp[b]) ck(cudaEventCreateWithFlags(&c->ring_rp[b], cudaEventDisableTiming), "event");
    }
    return chunk_rows;
}

// Host volumes of a load, pipelined: chunks of rows go H2D on the copy stream
// into a two-slot staging ring; the library stream re-pitches each chunk as
// it lands and validates each volume as soon as its last chunk is in, so the
// re-pitch/validation of one volume (and S^p, when the caller already knows
// p: sfseg_run) runs under the DMA of the next. One flag read-back at the
// end; errors are reported in load order (unary, pairwise channels, x0), as
// the sequential form reports them.
void load_pipelined(sfseg_ctx* c, const float* S, const float* const* F, const float* x0,
                    double sp_hint) {
    const size_t W = c->W, rows = static_cast<size_t>(c->T) * c->H;
    const size_t chunk_rows = ensure_ring(c);
    const int nv = 1 + c->C + (x0 ? 1 : 0);
    if (c->vflags_n < nv) {
        if (c->vflags) cudaFree(c->vflags);
        c->vflags = nullptr;
        c->vflags_n = 0;
        ck(cudaMalloc(&c->vflags, nv * sizeof(int)), "malloc flags");
        c->vflags_n = nv;
    }
    ck(cudaMemsetAsync(c->vflags, 0, nv * sizeof(int), c->stream), "memset flags");
    // the copy stream starts after everything already queued on the library
    // stream (earlier users of the destination buffers)
    ck(cudaEventRecord(c->ring_rp[0], c->stream), "event");
    ck(cudaStreamWaitEvent(c->cstream, c->ring_rp[0], 0), "wait");
    ck(cudaEventRecord(c->ring_rp[1], c->stream), "event");
    int slot = 0;
    auto one = [&](float* dst, const float* src, int vi, bool nonneg) {
        for (size_t r0 = 0; r0 < rows; r0 += chunk_rows) {
            const size_t nr = std::min(chunk_rows, rows - r0);
            ck(cudaStreamWaitEvent(c->cstream, c->ring_rp[slot], 0), "wait");
            ck(cudaMemcpyAsync(c->ring[slot], src + r0 * W, nr * W * sizeof(float),
                               cudaMemcpyHostToDevice, c->cstream),
               "upload volume");
            ck(cudaEventRecord(c->ring_up[slot], c->cstream), "event");
            ck(cudaStreamWaitEvent(c->stream, c->ring_up[slot], 0), "wait");
            sfk::k_repitch<<<c->num_sms * 8, 256, 0, c->stream>>>(c->ring[slot], c->W,
                                                                  dst + r0 * c->P, c->P, nr, c->W);
            launched(c->stream, "k_repitch");
            ck(cudaEventRecord(c->ring_rp[slot], c->stream), "event");
            slot ^= 1;
        }
        sfk::k_validate<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(dst), nonneg,
                                                                        c->vflags + vi);
        launched(c->stream, "k_validate");
    };
    one(c->S, S, 0, true);
    if (!std::isnan(sp_hint)) ensure_sp(c, sp_hint);  // S^p under the DMA of the channels
    for (int i = 0; i < c->C; ++i) {
        if (F[i] == S) {
            // the channel IS the unary volume (e.g. f = x0 = S, BASELINE c0/c1):
            // one upload, a device copy, and the unary's (stricter) validation
            ck(cudaMemcpyAsync(c->F[i], c->S, c->vol_elems() * sizeof(float),
                               cudaMemcpyDeviceToDevice, c->stream),
               "copy channel");
            continue;
        }
        one(c->F[i], F[i], 1 + i, false);
    }
    if (x0) one(c->x0, x0, 1 + c->C, true);
    std::vector<int> h(nv, 0);
    ck(cudaMemcpyAsync(h.data(), c->vflags, nv * sizeof(int), cudaMemcpyDeviceToHost, c->stream),
       "flags");
    ck(cudaStreamSynchronize(c->stream), "sync");
    for (int v = 0; v < nv; ++v) {
        const std::string what = v == 0 ? "unary" : (v <= c->C ? "pairwise" : "x0");
        if (h[v] & 1) {
            c->sp_p = NAN;
            fail(SFSEG_ERR_VALIDATION, what + " contains a non-finite value");
        }
        if (h[v] & 2) {
            c->sp_p = NAN;
            fail(SFSEG_ERR_VALIDATION, what + ": unary/solution volume contains a negative value");
        }
    }
}

void load_impl(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
               const float* const* F, const float* x0, int32_t mem, double sp_hint = NAN) {
    check_shape(T, H, W);
    if (C < 1) fail(SFSEG_ERR_VALIDATION, "feature set needs at least one pairwise channel");
    if (!S || !F) fail(SFSEG_ERR_PARAMETER, "null input");
    for (int i = 0; i < C; ++i)
        if (!F[i]) fail(SFSEG_ERR_PARAMETER, "null pairwise channel");
    set_shape(c, T, H, W, C);
    // a fresh upload invalidates derived buffers
    if (c->guard_applied)
        for (size_t i = 0; i < c->Fw.size(); ++i)
            if (c->Fw[i] != c->F[i]) dfree(c->Fw[i]);
    c->Fw = c->F;
    c->guard_applied = false;
    c->sp_p = NAN;
    c->cur = -1;
    c->cur_u = false;
    c->has_x0 = x0 != nullptr;
    if (x0 && !c->x0) c->x0 = dalloc_vol(c);
    if (mem == SFSEG_MEM_HOST && c->P != c->W) {
        load_pipelined(c, S, F, x0, sp_hint);
    } else {
        upload(c, c->S, S, mem);
        for (int i = 0; i < C; ++i) upload(c, c->F[i], F[i], mem);
        validate_vol(c, c->S, true, "unary");
        for (int i = 0; i < C; ++i) validate_vol(c, c->F[i], false, "pairwise");
        if (x0) {
            upload(c, c->x0, x0, mem);
            validate_vol(c, c->x0, true, "x0");
        }
    }
    c->resident = true;
    c->q_for.clear();  // channel contents changed
}

// ---- SFSV containers (load_volume, volume.cpp:142-184) ---------------------

constexpr size_t kPinChunk = size_t(32) << 20;  // bytes per pinned buffer

struct SfsvFile {
    std::FILE* f = nullptr;
    uint32_t T = 0, H = 0, W = 0;
    ~SfsvFile() {
        if (f) std::fclose(f);
    }
};

uint32_t get_u32_le(const unsigned char* b) {
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

// header checks in load_volume's order (volume.cpp:143-166)
void open_sfsv(const char* path, SfsvFile& sf) {
    if (!path) fail(SFSEG_ERR_PARAMETER, "null path");
    const std::string p(path);
    sf.f = std::fopen(path, "rb");
    if (!sf.f) fail(SFSEG_ERR_IO, "cannot open for reading: " + p);
    unsigned char h[32];
    if (std::fread(h, 1, sizeof h, sf.f) != sizeof h)
        fail(SFSEG_ERR_CORRUPTION, "file shorter than the container header: " + p);
    if (std::memcmp(h, "SFSV", 4) != 0) fail(SFSEG_ERR_FORMAT, "bad magic, not a volume container: " + p);
    if (get_u32_le(h + 4) != 1u) fail(SFSEG_ERR_FORMAT, "unsupported container version in " + p);
    sf.T = get_u32_le(h + 8);
    sf.H = get_u32_le(h + 12);
    sf.W = get_u32_le(h + 16);
    const uint32_t channels = get_u32_le(h + 20);
    if (h[24] != 0x01) fail(SFSEG_ERR_FORMAT, "unsupported payload dtype in " + p);
    for (int i = 25; i < 32; ++i)
        if (h[i] != 0) fail(SFSEG_ERR_FORMAT, "reserved header bytes set in " + p);
    if (channels != 1)
        fail(SFSEG_ERR_FORMAT, "expected a single-channel container, got " + std::to_string(channels) +
                                   " channels in " + p);
    check_shape(sf.T, sf.H, sf.W);
}

// payload -> dense device staging through two pinned buffers (the read of
// chunk k overlaps the DMA of chunk k - 1), then re-pitched into dst. The
// payload is little-endian f32, the host's own layout on x86-64 / aarch64.
void stream_sfsv(sfseg_ctx* c, SfsvFile& sf, const char* path, float* dst) {
    for (int b = 0; b < 2; ++b)
        if (!c->pin[b]) {
            ck(cudaHostAlloc(&c->pin[b], kPinChunk, cudaHostAllocDefault), "cudaHostAlloc");
            ck(cudaEventCreateWithFlags(&c->pin_ev[b], cudaEventDisableTiming), "event");
        }
    const size_t rows = static_cast<size_t>(c->T) * c->H;
    const size_t bytes = rows * c->W * sizeof(float);
    char* dense = reinterpret_cast<char*>(c->P == c->W ? dst : stage_buf(c));
    for (size_t off = 0, k = 0; off < bytes; off += kPinChunk, ++k) {
        const int b = static_cast<int>(k & 1);
        const size_t n = std::min(kPinChunk, bytes - off);
        // the previous DMA out of this buffer (this file's or an earlier one's) is done
        if (c->pin_used[b]) ck(cudaEventSynchronize(c->pin_ev[b]), "pinned buffer");
        if (std::fread(c->pin[b], 1, n, sf.f) != n)
            fail(SFSEG_ERR_CORRUPTION, std::string("payload truncated in ") + path);
        ck(cudaMemcpyAsync(dense + off, c->pin[b], n, cudaMemcpyHostToDevice, c->stream), "upload file");
        ck(cudaEventRecord(c->pin_ev[b], c->stream), "event");
        c->pin_used[b] = true;
    }
    if (c->P != c->W) {
        sfk::k_repitch<<<c->num_sms * 8, 256, 0, c->stream>>>(reinterpret_cast<float*>(dense), c->W, dst,
                                                             c->P, rows, c->W);
        launched(c->stream, "k_repitch");
    }
}

void load_files_impl(sfseg_ctx* c, const char* unary, const char* const* pairwise, int32_t C,
                     const char* x0) {
    if (C < 1) fail(SFSEG_ERR_VALIDATION, "feature set needs at least one pairwise channel");
    if (!pairwise) fail(SFSEG_ERR_PARAMETER, "null pairwise path list");
    std::vector<SfsvFile> files(static_cast<size_t>(C) + 1 + (x0 ? 1 : 0));
    open_sfsv(unary, files[0]);
    for (int i = 0; i < C; ++i) open_sfsv(pairwise[i], files[1 + i]);
    if (x0) open_sfsv(x0, files[1 + C]);
    for (size_t i = 1; i < files.size(); ++i)
        if (files[i].T != files[0].T || files[i].H != files[0].H || files[i].W != files[0].W)
            fail(SFSEG_ERR_SHAPE, i <= static_cast<size_t>(C)
                                      ? "pairwise channel shape differs from unary shape"
                                      : "x0 shape differs from the feature shape");
    set_shape(c, files[0].T, files[0].H, files[0].W, C);
    if (c->guard_applied)
        for (size_t i = 0; i < c->Fw.size(); ++i)
            if (c->Fw[i] != c->F[i]) dfree(c->Fw[i]);
    c->Fw = c->F;
    c->guard_applied = false;
    c->sp_p = NAN;
    c->cur = -1;
    c->cur_u = false;
    c->resident = false;
    stream_sfsv(c, files[0], unary, c->S);
    for (int i = 0; i < C; ++i) stream_sfsv(c, files[1 + i], pairwise[i], c->F[i]);
    c->has_x0 = x0 != nullptr;
    if (x0) {
        if (!c->x0) c->x0 = dalloc_vol(c);
        stream_sfsv(c, files[1 + C], x0, c->x0);
    }
    // load_volume rejects non-finite payloads; FeatureSet::validate the signs
    validate_vol(c, c->S, true, "unary");
    for (int i = 0; i < C; ++i) validate_vol(c, c->F[i], false, "pairwise");
    if (x0) validate_vol(c, c->x0, true, "x0");
    c->resident = true;
    c->q_for.clear();
}

// stateless helpers: (re)use the resident buffers of a scratch problem
// The stateless operators (sfseg_step, normalize_l2, ...) run on a scratch
// context owned by the caller's context (same device, own stream and
// buffers), so they can be called between or during the iterations of a
// resident solve (an IterationObserver) without touching its problem.
sfseg_ctx* scratch_ctx(sfseg_ctx* owner) {
    std::lock_guard<std::mutex> lk(owner->scratch_mu);
    if (!owner->scratch) {
        sfseg_ctx* s = nullptr;
        const int rc = sfseg_ctx_create(owner->device, &s);
        if (rc != SFSEG_OK) fail(rc, sfseg_last_error());
        owner->scratch = s;
    }
    return owner->scratch;
}

void stage_volume(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C) {
    check_shape(T, H, W);
    ck(cudaStreamSynchronize(c->stream), "sync");  // earlier small transfers are done
    c->pin_small_used = 0;
    set_shape(c, T, H, W, C);
    ensure_guard(c, false);  // drops guard copies of an earlier call (Fw = F)
    c->sp_p = NAN;
    c->cur = -1;
    c->cur_u = false;
    c->has_x0 = false;
    c->resident = false;  // stateless operators reuse the resident buffers
    c->q_for.clear();     // the channel buffers get new contents: Q is stale
}

void reduce_volume(sfseg_ctx* c, float* v, IterState* st, int mode_next, double lambda,
                   double frac) {
    ck(cudaMemsetAsync(c->frame_max, 0, c->Tout() * sizeof(float), c->stream), "memset");
    const long long warps = static_cast<long long>(c->Tout()) * c->nbands() * c->nhalves();
    sfk::k_partials<<<static_cast<int>((warps * 32 + 255) / 256), 256, 0, c->stream>>>(
        c->vol(v), c->part, c->frame_max, c->nbands(), c->nhalves(), 0);
    launched(c->stream, "k_partials");
    finalize(c, st, nullptr, 0, mode_next, lambda, frac);
}

float* max_of(sfseg_ctx* c, float* v) {
    ck(cudaMemsetAsync(c->scratch_f, 0, sizeof(float), c->stream), "memset");
    sfk::k_max<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(v), c->scratch_f);
    launched(c->stream, "k_max");
    return c->scratch_f;
}

void mask_of(sfseg_ctx* c, float* v, double frac, uint8_t* mask, int32_t mem) {
    float* mx = max_of(c, v);
    const size_t n = static_cast<size_t>(c->T) * c->H * c->W;
    uint8_t* dm = reinterpret_cast<uint8_t*>(mem == SFSEG_MEM_DEVICE ? mask : nullptr);
    if (!dm) {  // persistent device mask for host downloads
        if (c->dmask_elems < n) {
            if (c->dmask) cudaFree(c->dmask);
            c->dmask = nullptr;
            c->dmask_elems = 0;
            ck(cudaMalloc(reinterpret_cast<void**>(&c->dmask), n), "malloc mask");
            c->dmask_elems = n;
        }
        dm = c->dmask;
    }
    sfk::k_mask<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(v), mx, frac, dm);
    launched(c->stream, "k_mask");
    if (mem != SFSEG_MEM_DEVICE)
        ck(cudaMemcpyAsync(mask, dm, n, cudaMemcpyDeviceToHost, c->stream), "mask D2H");
}

// Soft iterate (and mask) to host memory, pipelined: the library stream
// de-pitches row chunks into the staging ring and the copy stream moves each
// chunk D2H as soon as it is ready; the max and mask kernels run on the
// library stream under the first chunks' DMA. The library stream ends after
// the last copy, so synchronising it covers the whole download.
void download_pipelined(sfseg_ctx* c, float* soft, float* x, double frac, uint8_t* mask) {
    const size_t W = c->W, rows = static_cast<size_t>(c->T) * c->H;
    const size_t chunk_rows = ensure_ring(c);
    int slot = 0, k = 0;
    bool masked = mask == nullptr;
    for (size_t r0 = 0; r0 < rows; r0 += chunk_rows, ++k) {
        const size_t nr = std::min(chunk_rows, rows - r0);
        ck(cudaStreamWaitEvent(c->stream, c->ring_rp[slot], 0), "wait");  // slot drained
        sfk::k_repitch<<<c->num_sms * 8, 256, 0, c->stream>>>(x + r0 * c->P, c->P, c->ring[slot],
                                                              c->W, nr, c->W);
        launched(c->stream, "k_repitch");
        ck(cudaEventRecord(c->ring_up[slot], c->stream), "event");
        ck(cudaStreamWaitEvent(c->cstream, c->ring_up[slot], 0), "wait");
        ck(cudaMemcpyAsync(soft + r0 * W, c->ring[slot], nr * W * sizeof(float),
                           cudaMemcpyDeviceToHost, c->cstream),
           "download volume");
        ck(cudaEventRecord(c->ring_rp[slot], c->cstream), "event");
        slot ^= 1;
        if (k == 1 && !masked) {
            mask_of(c, x, frac, mask, SFSEG_MEM_HOST);
            masked = true;
        }
    }
    if (!masked) mask_of(c, x, frac, mask, SFSEG_MEM_HOST);
    ck(cudaStreamWaitEvent(c->stream, c->ring_rp[slot ^ 1], 0), "wait");  // the last copy
}

}  // namespace

// ===========================================================================
extern "C" {

void sfseg_params_default(sfseg_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    p->alpha = 1.0;
    p->p = 0.1;
    p->radii[0] = 1;
    p->radii[1] = 3;
    p->radii[2] = 3;
    p->sigmas[0] = 0.5;
    p->sigmas[1] = 1.5;
    p->sigmas[2] = 1.5;
    p->iterations = 5;
    p->temporal_window = -1;
    p->binarize_start = 3;
    p->sigmoid_slope0 = 10.0;
    p->slope_growth = 2.0;
    p->threshold_frac = 0.5;
    p->final_threshold = 0.5;
    p->allow_negative_affinity = 0;
    p->arith = SFSEG_ARITH_EXACT;
}

int sfseg_params_validate(const sfseg_params* p) {
    return guarded([&] { validate_params(p); });
}

int sfseg_make_kernel(const int32_t radii[3], const double sigmas[3], double* tt, double* ty,
                      double* tx) {
    return guarded([&] {
        const HostKernel k = make_kernel(radii, sigmas);
        std::memcpy(tt, k.t.data(), k.t.size() * sizeof(double));
        std::memcpy(ty, k.y.data(), k.y.size() * sizeof(double));
        std::memcpy(tx, k.x.data(), k.x.size() * sizeof(double));
    });
}

const char* sfseg_last_error(void) { return g_err.c_str(); }

const char* sfseg_build_info(void) {
    return "sfseg_cuda abi=" "1" " arch=sm_100a fused=exact(rt,r)={(1,2),(1,3),(2,4),(2,5)}";
}

// ---- explicit-affinity oracle on the GPU (oracle.cpp:67-258, affinity.cuh) ----
}  // extern "C"

namespace {

struct DBuf {  // owning device allocation for one call
    void* p = nullptr;
    explicit DBuf(size_t bytes) { ck(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~DBuf() {
        if (p) cudaFree(p);
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct AffProblem {
    std::vector<std::unique_ptr<DBuf>> bufs;
    sfk::AffArgs a{};
    long long n = 0;
    cudaStream_t stream = nullptr;
    int nb = 0;
    DBuf* parts = nullptr;
    DBuf* scal = nullptr;  // [0] norm, [1] second scalar
    template <class T> T* alloc(size_t count) {
        bufs.push_back(std::make_unique<DBuf>(count * sizeof(T)));
        return bufs.back()->as<T>();
    }
};

// build_affinity_impl's checks (oracle.cpp:69-86, minus the node cap) and
// the device-side operands: dense float channels, S^p in fp64 (host std::pow,
// the reference's own libm), fp64 taps of make_gaussian_kernel
void aff_setup(sfseg_ctx* c, AffProblem& P, uint32_t T, uint32_t H, uint32_t W, int32_t C,
               const float* S, const float* const* F, const sfseg_params* p, int32_t kind,
               int32_t mem) {
    validate_params(p);
    check_shape(T, H, W);
    if (C < 1) fail(SFSEG_ERR_VALIDATION, "feature set needs at least one pairwise channel");
    if (C > 8) fail(SFSEG_ERR_CAPACITY, "the GPU affinity oracle takes at most 8 channels");
    if (kind < SFSEG_AFFINITY_EXACT || kind > SFSEG_AFFINITY_TAYLOR_CHANNEL_SUM)
        fail(SFSEG_ERR_PARAMETER, "unknown affinity kind");
    if (!S || !F) fail(SFSEG_ERR_PARAMETER, "null input");
    const HostKernel k = make_kernel(p->radii, p->sigmas);
    if (k.rt > 31 || k.ry > 31 || k.rx > 31) fail(SFSEG_ERR_CAPACITY, "kernel radius above 31");
    const size_t n = static_cast<size_t>(T) * H * W;
    P.n = static_cast<long long>(n);
    P.stream = c->stream;
    // host copies for validation and S^p (device inputs come down once)
    auto host_of = [&](const float* src) {
        std::vector<float> h(n);
        ck(cudaMemcpy(h.data(), src, n * sizeof(float),
                      mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost),
           "copy");
        return h;
    };
    const std::vector<float> hs = host_of(S);
    for (float v : hs) {  // FeatureSet::validate (volume.cpp:72-93)
        if (!std::isfinite(v)) fail(SFSEG_ERR_VALIDATION, "unary contains a non-finite value");
        if (v < 0.0f) fail(SFSEG_ERR_VALIDATION, "unary/solution volume contains a negative value");
    }
    for (int ch = 0; ch < C; ++ch) {
        if (!F[ch]) fail(SFSEG_ERR_PARAMETER, "null pairwise channel");
        const std::vector<float> hf = host_of(F[ch]);
        for (float v : hf) {
            if (!std::isfinite(v)) fail(SFSEG_ERR_VALIDATION, "pairwise contains a non-finite value");
            if (!p->allow_negative_affinity && (v < 0.0f || v > 1.0f))
                fail(SFSEG_ERR_VALIDATION, "pairwise channel " + std::to_string(ch) +
                                               " leaves [0,1]; prescale it or enable allow_negative_affinity");
        }
        float* d = P.alloc<float>(n);
        ck(cudaMemcpyAsync(d, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice, c->stream), "upload");
        P.a.f[ch] = d;
        ck(cudaStreamSynchronize(c->stream), "upload");  // hf goes out of scope
    }
    std::vector<double> sp(n);
    for (size_t i = 0; i < n; ++i)
        sp[i] = p->p == 0.0 ? 1.0 : std::pow(static_cast<double>(hs[i]), p->p);
    double* dsp = P.alloc<double>(n);
    ck(cudaMemcpy(dsp, sp.data(), n * sizeof(double), cudaMemcpyHostToDevice), "upload");
    P.a.sp = dsp;
    P.a.T = static_cast<int>(T);
    P.a.H = static_cast<int>(H);
    P.a.W = static_cast<int>(W);
    P.a.C = C;
    P.a.rt = k.rt;
    P.a.ry = k.ry;
    P.a.rx = k.rx;
    P.a.exact = kind == SFSEG_AFFINITY_EXACT;
    P.a.alpha = p->alpha;
    P.a.base = kind == SFSEG_AFFINITY_TAYLOR_CHANNEL_SUM ? static_cast<double>(C) : 1.0;
    for (int i = 0; i <= 2 * k.rt; ++i) P.a.tt[i] = k.t[i];
    for (int i = 0; i <= 2 * k.ry; ++i) P.a.ty[i] = k.y[i];
    for (int i = 0; i <= 2 * k.rx; ++i) P.a.tx[i] = k.x[i];
    P.nb = c->num_sms * 4;
    P.bufs.push_back(std::make_unique<DBuf>(P.nb * sizeof(double)));
    P.parts = P.bufs.back().get();
    P.bufs.push_back(std::make_unique<DBuf>(4 * sizeof(double)));
    P.scal = P.bufs.back().get();
}

void aff_matvec(sfseg_ctx* c, AffProblem& P, const double* x, double* y) {
    P.a.x = x;
    P.a.y = y;
    const int grid = static_cast<int>(std::min<long long>((P.n + 255) / 256, c->num_sms * 16LL));
    sfk::k_affinity_matvec<<<grid, 256, 0, c->stream>>>(P.a);
    launched(c->stream, "k_affinity_matvec");
}

// out = fixed-order fp64 sum (OP of k_dot_blocks), sqrt when asked
template <int OP>
void aff_sum(sfseg_ctx* c, AffProblem& P, const double* a, const double* b, const double* scale,
             double* out, bool sq) {
    sfk::k_dot_blocks<OP><<<P.nb, sfk::kRedThreads, 0, c->stream>>>(a, b, scale, P.n, P.parts->as<double>());
    sfk::k_sum_final<<<1, 32, 0, c->stream>>>(P.parts->as<double>(), P.nb, out, sq ? 1 : 0);
    launched(c->stream, "affinity reduction");
}

}  // namespace

extern "C" {

int sfseg_affinity_matvec(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C,
                          const float* S, const float* const* F, const sfseg_params* p, int32_t kind,
                          const double* x, double* y, int32_t mem) {
    return guarded([&] {
        if (!c || !p || !x || !y) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        AffProblem P;
        aff_setup(c, P, T, H, W, C, S, F, p, kind, mem);
        const size_t n = static_cast<size_t>(P.n);
        const double* dx = x;
        double* dy = y;
        if (mem != SFSEG_MEM_DEVICE) {
            double* bx = P.alloc<double>(n);
            ck(cudaMemcpyAsync(bx, x, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "upload x");
            dx = bx;
            dy = P.alloc<double>(n);
        }
        aff_matvec(c, P, dx, dy);
        if (mem != SFSEG_MEM_DEVICE)
            ck(cudaMemcpyAsync(y, dy, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "download y");
        ck(cudaStreamSynchronize(c->stream), "matvec");
    });
}

int sfseg_affinity_power_iteration(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C,
                                   const float* S, const float* const* F, const sfseg_params* p,
                                   int32_t kind, const double* x0, int32_t max_iters, double tol,
                                   double* eigenvector, double* eigenvalue, int32_t* iterations_used,
                                   int32_t mem) {
    return guarded([&] {
        if (!c || !p || !x0) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (max_iters < 1) fail(SFSEG_ERR_PARAMETER, "max_iters must be at least 1");
        AffProblem P;
        aff_setup(c, P, T, H, W, C, S, F, p, kind, mem);
        const size_t n = static_cast<size_t>(P.n);
        double* x = P.alloc<double>(n);
        double* y = P.alloc<double>(n);
        double* sc = P.scal->as<double>();
        ck(cudaMemcpyAsync(y, x0, n * sizeof(double),
                           mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           c->stream),
           "upload x0");
        const int g = static_cast<int>(std::min<long long>((P.n + 255) / 256, c->num_sms * 16LL));
        // x0 / ||x0|| (oracle.cpp:223-225)
        aff_sum<0>(c, P, y, nullptr, nullptr, sc, true);
        double h[2];
        ck(cudaMemcpyAsync(h, sc, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "norm");
        ck(cudaStreamSynchronize(c->stream), "norm");
        if (h[0] == 0.0) fail(SFSEG_ERR_PARAMETER, "power iteration needs a nonzero start vector");
        sfk::k_div_scale<<<g, 256, 0, c->stream>>>(y, sc, x, P.n);
        launched(c->stream, "k_div_scale");
        int used = 0;
        for (int k = 1; k <= max_iters; ++k) {  // oracle.cpp:229-243
            aff_matvec(c, P, x, y);
            aff_sum<0>(c, P, y, nullptr, nullptr, sc, true);             // ||y||
            aff_sum<2>(c, P, y, x, sc, sc + 1, true);                    // ||y/||y|| - x||
            ck(cudaMemcpyAsync(h, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "scalars");
            ck(cudaStreamSynchronize(c->stream), "power iteration");
            if (h[0] == 0.0) fail(SFSEG_ERR_DEGENERATE, "power iteration mapped the iterate to zero");
            sfk::k_div_scale<<<g, 256, 0, c->stream>>>(y, sc, x, P.n);
            launched(c->stream, "k_div_scale");
            used = k;
            if (h[1] < tol) break;
        }
        // eigenvalue = cluster_score(m, x) = x^T M x / x^T x (oracle.cpp:249-258)
        aff_matvec(c, P, x, y);
        aff_sum<0>(c, P, x, nullptr, nullptr, sc, false);
        aff_sum<1>(c, P, x, y, nullptr, sc + 1, false);
        ck(cudaMemcpyAsync(h, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "scalars");
        if (eigenvector)
            ck(cudaMemcpyAsync(eigenvector, x, n * sizeof(double),
                               mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               c->stream),
               "eigenvector");
        ck(cudaStreamSynchronize(c->stream), "power iteration");
        if (eigenvalue) *eigenvalue = h[1] / h[0];
        if (iterations_used) *iterations_used = used;
    });
}

uint64_t sfseg_separable_convolution_count(void) {
    return g_conv_count.load(std::memory_order_relaxed);
}

int sfseg_ctx_create(int device, sfseg_ctx** out) {
    return guarded([&] {
        if (!out) fail(SFSEG_ERR_PARAMETER, "null out");
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(SFSEG_ERR_CUDA, "no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            fail(SFSEG_ERR_CUDA, std::string("sfseg_cuda is built for sm_100a; device is ") +
                                     prop.name);
        auto* c = new sfseg_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        c->tap_trim = env_flag("SFSEG_FAST_TRIM");
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        ck(cudaMalloc(&c->st, sizeof(IterState)), "malloc");
        ck(cudaMalloc(&c->st_aux, sizeof(IterState)), "malloc");
        ck(cudaMalloc(&c->flags, sizeof(int)), "malloc");
        ck(cudaMalloc(&c->scratch_f, 4 * sizeof(float)), "malloc");
        ck(cudaMalloc(&c->bminmax, 2 * aux_grid(c) * sizeof(float)), "malloc");
        ck(cudaMalloc(&c->acc3, 3 * sizeof(double)), "malloc");
        ck(cudaMalloc(&c->cnt2, 2 * sizeof(unsigned long long)), "malloc");
        ck(cudaMalloc(&c->ticket, sizeof(unsigned int)), "malloc");
        ck(cudaMemset(c->ticket, 0, sizeof(unsigned int)), "memset");
        *out = c;
    });
}

int sfseg_ctx_destroy(sfseg_ctx* c) {
    return guarded([&] {
        if (!c) return;
        if (c->scratch) sfseg_ctx_destroy(c->scratch);
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        release_problem(c);
        cudaFree(c->st);
        cudaFree(c->st_aux);
        cudaFree(c->flags);
        cudaFree(c->scratch_f);
        cudaFree(c->bminmax);
        cudaFree(c->acc3);
        cudaFree(c->cnt2);
        cudaFree(c->ticket);
        for (int b = 0; b < 2; ++b) {
            if (c->pin[b]) cudaFreeHost(c->pin[b]);
            if (c->pin_ev[b]) cudaEventDestroy(c->pin_ev[b]);
        }
        if (c->conv_part) cudaFree(c->conv_part);
        if (c->st_prev) cudaFree(c->st_prev);
        if (c->norms) cudaFree(c->norms);
        if (c->sched_seg) cudaFree(c->sched_seg);
        if (c->sched_off) cudaFree(c->sched_off);
        for (auto e : c->ev) cudaEventDestroy(e);
        for (int b = 0; b < 2; ++b) {
            if (c->ring[b]) cudaFree(c->ring[b]);
            if (c->ring_up[b]) cudaEventDestroy(c->ring_up[b]);
            if (c->ring_rp[b]) cudaEventDestroy(c->ring_rp[b]);
        }
        if (c->vflags) cudaFree(c->vflags);
        if (c->pin_small) cudaFreeHost(c->pin_small);
        if (c->cstream) cudaStreamDestroy(c->cstream);
        cudaStreamDestroy(c->stream);
        delete c;
    });
}

int sfseg_probe_fp32_peak(int device, double* tflops) {
    return guarded([&] {
        if (!tflops) fail(SFSEG_ERR_PARAMETER, "null argument");
        ck(cudaSetDevice(device), "cudaSetDevice");
        int sms = 0;
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attribute");
        float* out = nullptr;
        ck(cudaMalloc(&out, 1024 * sizeof(float)), "cudaMalloc");
        cudaStream_t s;
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int blocks = sms * 4, threads = 512, iters = 1 << 14;
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0, s);
            sfk::k_fma_probe<<<blocks, threads, 0, s>>>(out, 1.0001f, iters);
            cudaEventRecord(e1, s);
            ck(cudaEventSynchronize(e1), "probe");
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = double(blocks) * threads * iters * 8 * 2 * 2;
            if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
        }
        ck(cudaGetLastError(), "k_fma_probe");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(s);
        cudaFree(out);
        *tflops = best;
    });
}

int sfseg_ctx_kernel_time(sfseg_ctx* c, double* ms, int32_t* launches) {
    return guarded([&] {
        if (!c || !ms || !launches) fail(SFSEG_ERR_PARAMETER, "null argument");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "sync");
        double total = 0.0;
        int n = 0;
        for (size_t i = 0; i + 1 < c->ev.size(); i += 2) {
            float m = 0.0f;
            cudaEventElapsedTime(&m, c->ev[i], c->ev[i + 1]);
            total += m;
            ++n;
        }
        for (auto e : c->ev) cudaEventDestroy(e);
        c->ev.clear();
        *ms = total;
        *launches = n;
    });
}

int sfseg_ctx_set_timing(sfseg_ctx* c, int enabled) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        c->timing = enabled != 0;
    });
}

int sfseg_ctx_set_tap_trim(sfseg_ctx* c, int enabled) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        c->tap_trim = enabled != 0;
    });
}

int sfseg_effective_radii(const sfseg_params* p, int32_t out[3]) {
    return guarded([&] {
        if (!p || !out) fail(SFSEG_ERR_PARAMETER, "null argument");
        const HostKernel k = trim_kernel(make_kernel(p->radii, p->sigmas));
        out[0] = k.rt;
        out[1] = k.ry;
        out[2] = k.rx;
    });
}

int sfseg_ctx_get_timing(const sfseg_ctx* c, sfseg_timing* out) {
    return guarded([&] {
        if (!c || !out) fail(SFSEG_ERR_PARAMETER, "null argument");
        *out = c->last_timing;
    });
}

void* sfseg_ctx_stream(sfseg_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int sfseg_ctx_synchronize(sfseg_ctx* c) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int sfseg_load(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
               const float* const* F, const float* x0, int32_t mem) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        load_impl(c, T, H, W, C, S, F, x0, mem);
    });
}

int sfseg_load_files(sfseg_ctx* c, const char* unary, const char* const* pairwise, int32_t C,
                     const char* x0) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        load_files_impl(c, unary, pairwise, C, x0);
    });
}

int sfseg_solve(sfseg_ctx* c, const sfseg_params* p, int32_t first, int32_t last,
                sfseg_iter_record* rec) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        solve_impl(c, p, first, last, rec);
    });
}

int sfseg_solve_until(sfseg_ctx* c, const sfseg_params* p, int32_t first, int32_t max_iter,
                      int32_t criterion, double tol, int32_t* iterations_done,
                      sfseg_iter_record* records) {
    return guarded([&] {
        if (!c || !p || !iterations_done) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        solve_until_impl(c, p, first, max_iter, criterion, tol, iterations_done, records);
    });
}

namespace {
// caller holds c->mu and has selected the device
void download_impl(sfseg_ctx* c, double frac, float* soft, uint8_t* mask, int32_t mem) {
    if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_download before sfseg_load");
    float* x = tmp_vol(c, 0);
    materialize(c, x);
    if (soft && mem == SFSEG_MEM_HOST && c->P != c->W) {
        download_pipelined(c, soft, x, frac, mask);
    } else {
        if (soft) download(c, soft, x, mem);
        if (mask) mask_of(c, x, frac, mask, mem);
    }
    ck(cudaStreamSynchronize(c->stream), "download");
}
}  // namespace

int sfseg_download(sfseg_ctx* c, double frac, float* soft, uint8_t* mask, int32_t mem) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        download_impl(c, frac, soft, mask, mem);
    });
}

int sfseg_metrics(sfseg_ctx* c, const float* reference, const uint8_t* gt, double frac,
                  double* angle, double* iou, int32_t mem) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_metrics before sfseg_load");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        float* x = tmp_vol(c, 0);
        materialize(c, x);
        Vol ref{nullptr, c->T, c->H, c->W, c->P};
        if (reference) {
            ref.p = tmp_vol(c, 1);
            upload(c, ref.p, reference, mem);
        }
        const size_t n = static_cast<size_t>(c->T) * c->H * c->W;
        uint8_t* dgt = nullptr;
        if (gt) {
            ck(cudaMallocAsync(reinterpret_cast<void**>(&dgt), n, c->stream), "malloc");
            ck(cudaMemcpyAsync(dgt, gt, n,
                               mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                       : cudaMemcpyHostToDevice,
                               c->stream),
               "gt");
        }
        float* mx = gt ? max_of(c, x) : nullptr;
        ck(cudaMemsetAsync(c->acc3, 0, 3 * sizeof(double), c->stream), "memset");
        ck(cudaMemsetAsync(c->cnt2, 0, 2 * sizeof(unsigned long long), c->stream), "memset");
        sfk::k_metrics<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(x), ref, dgt, mx,
                                                                      frac, c->acc3, c->cnt2);
        launched(c->stream, "k_metrics");
        double a3[3];
        unsigned long long c2[2];
        ck(cudaMemcpyAsync(a3, c->acc3, sizeof a3, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaMemcpyAsync(c2, c->cnt2, sizeof c2, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (dgt) ck(cudaFreeAsync(dgt, c->stream), "free");
        ck(cudaStreamSynchronize(c->stream), "metrics");
        if (angle) {
            if (!reference) {
                *angle = NAN;
            } else {
                if (a3[1] == 0.0 || a3[2] == 0.0)
                    fail(SFSEG_ERR_PARAMETER, "angle is undefined for a zero vector");
                const double cs =
                    std::clamp(a3[0] / (std::sqrt(a3[1]) * std::sqrt(a3[2])), -1.0, 1.0);
                *angle = std::acos(cs) * 57.295779513082320876798154814105;
            }
        }
        if (iou) *iou = !gt ? NAN : (c2[1] == 0 ? 1.0 : double(c2[0]) / double(c2[1]));
    });
}

int sfseg_run(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
              const float* const* F, const float* x0, const sfseg_params* p, float* soft,
              uint8_t* mask, sfseg_iter_record* rec, int32_t mem) {
    // load (S^p computed under the DMA of the channels, p being known),
    // solve and download under ONE hold of the context lock: the call is
    // atomic with respect to other users of the context
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        validate_params(p);
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        load_impl(c, T, H, W, C, S, F, x0, mem, p->p);
        solve_impl(c, p, 1, p->iterations, rec);
        download_impl(c, p->final_threshold, soft, mask, mem);
    });
}

int sfseg_run_batch(sfseg_ctx* const* ctxs, int32_t nctx, sfseg_clip* clips, int32_t nclips,
                    const sfseg_params* p, int32_t mem) {
    // The reference's batch is a loop of run() calls (one video each,
    // engine.cpp:247). Here: a shared queue in LPT order, one host thread per
    // context. On one device the contexts' copy-stream DMAs overlap the other
    // contexts' kernels; on several devices the clips shard with no exchange.
    std::vector<std::string> msgs;
    const int rc = guarded([&] {
        if (!ctxs || nctx < 1 || nclips < 0 || (nclips > 0 && !clips) || !p)
            fail(SFSEG_ERR_PARAMETER, "null argument");
        for (int i = 0; i < nctx; ++i) {
            if (!ctxs[i]) fail(SFSEG_ERR_PARAMETER, "null ctx");
            for (int j = 0; j < i; ++j)
                if (ctxs[j] == ctxs[i]) fail(SFSEG_ERR_PARAMETER, "contexts must be distinct");
        }
        validate_params(p);
        std::vector<int> order(nclips);
        for (int i = 0; i < nclips; ++i) order[i] = i;
        auto voxels = [&](int i) {
            return static_cast<unsigned __int128>(clips[i].frames) * clips[i].height * clips[i].width *
                   static_cast<unsigned>(std::max(1, clips[i].channels));
        };
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return voxels(a) > voxels(b); });
        msgs.assign(nclips, std::string());
        std::atomic<int> next{0};
        auto work = [&](int w) {
            for (;;) {
                const int k = next.fetch_add(1);
                if (k >= nclips) return;
                sfseg_clip& cl = clips[order[k]];
                const auto t0 = std::chrono::steady_clock::now();
                cl.worker = w;
                cl.status = sfseg_run(ctxs[w], cl.frames, cl.height, cl.width, cl.channels, cl.unary,
                                      cl.pairwise, cl.x0, p, cl.soft, cl.mask, cl.records, mem);
                if (cl.status != SFSEG_OK) msgs[order[k]] = g_err;  // this thread's message
                cl.wall_ms = std::chrono::duration<double, std::milli>(
                                 std::chrono::steady_clock::now() - t0).count();
            }
        };
        std::vector<std::thread> th;
        const int nw = std::min<int>(nctx, std::max(1, nclips));
        for (int w = 1; w < nw; ++w) th.emplace_back(work, w);
        work(0);
        for (auto& t : th) t.join();
    });
    if (rc != SFSEG_OK) return rc;
    for (int i = 0; i < nclips; ++i)
        if (clips[i].status != SFSEG_OK) {
            g_err = "clip " + std::to_string(i) + ": " + msgs[i];
            return clips[i].status;
        }
    return SFSEG_OK;
}

int sfseg_step(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* x,
               const float* S, const float* const* F, const sfseg_params* p, float* out,
               int32_t mem) {
    return guarded([&] {
        if (!owner) fail(SFSEG_ERR_PARAMETER, "null ctx");
        validate_params(p);  // engine.cpp:143
        if (C < 1) fail(SFSEG_ERR_PARAMETER, "sfseg_step needs at least one pairwise channel");
        if (!x || !S || !F || !out) fail(SFSEG_ERR_PARAMETER, "null input");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const HostKernel k = make_kernel(p->radii, p->sigmas);
        const double sp_before = c->sp_p;
        stage_volume(c, T, H, W, C);
        const size_t n = static_cast<size_t>(T) * H * W;
        const bool cacheable = mem == SFSEG_MEM_HOST && n <= kSmall;
        bool hit = cacheable && c->in_valid && c->in_gen == c->alloc_gen &&
                   c->in_host.size() == static_cast<size_t>(C) + 1;
        for (int i = 0; hit && i <= C; ++i)
            hit = std::memcmp(c->in_host[i].data(), i == 0 ? S : F[i - 1], n * sizeof(float)) == 0;
        if (hit) {
            c->sp_p = sp_before;  // S (and so S^p) on the device are the caller's again
        } else {
            upload(c, c->S, S, mem);
            for (int i = 0; i < C; ++i) upload(c, c->F[i], F[i], mem);
            c->in_valid = cacheable;
            c->in_gen = c->alloc_gen;
            if (cacheable) {
                c->in_host.assign(C + 1, std::vector<float>(n));
                for (int i = 0; i <= C; ++i)
                    std::memcpy(c->in_host[i].data(), i == 0 ? S : F[i - 1], n * sizeof(float));
            }
        }
        float* xin = c->y[1];
        upload(c, xin, x, mem);
        ensure_sp(c, p->p);
        IterState* s0 = reinterpret_cast<IterState*>(pin_slot(c, (sizeof(IterState) + 3) / 4));
        *s0 = IterState{};  // mode 0: x as given
        ck(cudaMemcpyAsync(c->st_aux, s0, sizeof(IterState), cudaMemcpyHostToDevice, c->stream), "state");
        ck(cudaMemsetAsync(c->frame_max, 0, c->Tout() * sizeof(float), c->stream), "memset");
        launch_step(c, k, p->alpha, xin, c->st_aux, c->y[0], c->F, p->arith == SFSEG_ARITH_FAST);
        download(c, out, c->y[0], mem);
        ck(cudaStreamSynchronize(c->stream), "sfseg_step");
        if (!c->in_valid) c->sp_p = NAN;  // S is scratch now
    });
}

int sfseg_step_channel(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, const float* x,
                       const float* S, const float* f, const sfseg_params* p, float* out,
                       int32_t mem) {
    const float* F[1] = {f};
    return sfseg_step(c, T, H, W, 1, x, S, F, p, out, mem);
}

int sfseg_normalize_l2(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* x,
                       float* out, double* norm, int32_t mem) {
    return guarded([&] {
        if (!owner) fail(SFSEG_ERR_PARAMETER, "null ctx");
        if (!x) fail(SFSEG_ERR_PARAMETER, "null input");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        float* v = c->y[0];
        upload(c, v, x, mem);
        // one host round trip: state in, reduction, x / ||x||, state and
        // result out (a zero norm throws after it, with no output, as
        // engine.cpp:174-175 does)
        const size_t sw = (sizeof(IterState) + 3) / 4;
        IterState* in = reinterpret_cast<IterState*>(pin_slot(c, sw));
        IterState* res = reinterpret_cast<IterState*>(pin_slot(c, sw));
        *in = IterState{};
        ck(cudaMemcpyAsync(c->st_aux, in, sizeof(IterState), cudaMemcpyHostToDevice, c->stream), "state");
        reduce_volume(c, v, c->st_aux, 1, 0.0, 0.5);
        if (out) {
            sfk::k_transform<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(
                c->vol(v), c->vol(c->y[1]), c->st_aux);
            launched(c->stream, "k_transform");
        }
        ck(cudaMemcpyAsync(res, c->st_aux, sizeof(IterState), cudaMemcpyDeviceToHost, c->stream), "state");
        if (out) download(c, out, c->y[1], mem);
        ck(cudaStreamSynchronize(c->stream), "normalize_l2");
        if (norm) *norm = res->norm;
        if (res->norm == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
    });
}

int sfseg_unit_range(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* v,
                     float* out, int32_t mem) {
    return guarded([&] {
        if (!owner || !v || !out) fail(SFSEG_ERR_PARAMETER, "null argument");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        c->in_valid = false;  // F[0] gets other contents
        upload(c, c->F[0], v, mem);
        ensure_guard(c, true);  // k_minmax_* + k_unit_range (IEEE divide), engine.cpp:228-243
        download(c, out, c->Fw[0], mem);
        ck(cudaStreamSynchronize(c->stream), "unit_range");
    });
}

int sfseg_project_binary(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* x,
                         int32_t iter, const sfseg_params* p, float* out, int32_t mem) {
    return guarded([&] {
        if (!owner || !p || !x || !out) fail(SFSEG_ERR_PARAMETER, "null argument");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        float* v = c->y[0];
        upload(c, v, x, mem);
        if (iter < p->binarize_start) {  // engine.cpp:186
            download(c, out, v, mem);
            ck(cudaStreamSynchronize(c->stream), "project_binary");
            return;
        }
        float* mx = max_of(c, v);
        float hmax = 0.0f;
        ck(cudaMemcpyAsync(&hmax, mx, sizeof hmax, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        IterState s{};
        s.mode = 2;
        s.inv = 1.0;  // float(double(x) * 1.0) == x exactly
        s.theta = p->threshold_frac * static_cast<double>(hmax);
        s.lambda = lambda_for(p, iter);
        set_state(c, c->st_aux, s);
        sfk::k_transform<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(
            c->vol(v), c->vol(c->y[1]), c->st_aux);
        launched(c->stream, "k_transform");
        download(c, out, c->y[1], mem);
        ck(cudaStreamSynchronize(c->stream), "project_binary");
    });
}

int sfseg_threshold_final(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* x,
                          double frac, uint8_t* mask, int32_t mem) {
    return guarded([&] {
        if (!owner || !x || !mask) fail(SFSEG_ERR_PARAMETER, "null argument");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        float* v = c->y[0];
        upload(c, v, x, mem);
        mask_of(c, v, frac, mask, mem);
        ck(cudaStreamSynchronize(c->stream), "threshold_final");
    });
}

int sfseg_convolve_separable(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* v,
                             const int32_t radii[3], const double sigmas[3], float* out,
                             int32_t mem) {
    return guarded([&] {
        if (!owner || !v || !out) fail(SFSEG_ERR_PARAMETER, "null argument");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const HostKernel k = make_kernel(radii, sigmas);
        if (k.rt > 31 || k.ry > 31 || k.rx > 31) fail(SFSEG_ERR_CAPACITY, "kernel radius above 31");
        stage_volume(c, T, H, W, 1);
        sfk::Taps tp;
        std::memset(&tp, 0, sizeof tp);
        for (int i = 0; i <= 2 * k.rt; ++i) tp.t[i] = static_cast<float>(k.t[i]);
        for (int i = 0; i <= 2 * k.ry; ++i) tp.y[i] = static_cast<float>(k.y[i]);
        for (int i = 0; i <= 2 * k.rx; ++i) tp.x[i] = static_cast<float>(k.x[i]);
        tp.rt = k.rt;
        tp.ry = k.ry;
        tp.rx = k.rx;
        float *a = c->y[0], *b = c->y[1], *t0 = tmp_vol(c, 0);
        upload(c, a, v, mem);
        const int g = aux_grid(c), bt = sfk::kAuxThreads;
        sfk::k_pass_x<<<g, bt, 0, c->stream>>>(c->vol(a), c->vol(t0), tp);
        sfk::k_pass_y<<<g, bt, 0, c->stream>>>(c->vol(t0), c->vol(b), tp);
        sfk::k_pass_t<<<g, bt, 0, c->stream>>>(c->vol(b), c->vol(a), tp);
        launched(c->stream, "convolve_separable");
        download(c, out, a, mem);
        ck(cudaStreamSynchronize(c->stream), "convolve_separable");
        g_conv_count.fetch_add(1, std::memory_order_relaxed);
    });
}

int sfseg_convolve_separable_taps(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W,
                                  const float* v, const int32_t radii[3], const double* tt,
                                  const double* ty, const double* tx, float* out, int32_t mem) {
    return guarded([&] {
        if (!owner || !v || !out || !radii || !tt || !ty || !tx) fail(SFSEG_ERR_PARAMETER, "null argument");
        for (int i = 0; i < 3; ++i)
            if (radii[i] < 0 || radii[i] > 31) fail(SFSEG_ERR_CAPACITY, "kernel radius above 31");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        sfk::Taps tp;
        std::memset(&tp, 0, sizeof tp);
        for (int i = 0; i <= 2 * radii[0]; ++i) tp.t[i] = static_cast<float>(tt[i]);
        for (int i = 0; i <= 2 * radii[1]; ++i) tp.y[i] = static_cast<float>(ty[i]);
        for (int i = 0; i <= 2 * radii[2]; ++i) tp.x[i] = static_cast<float>(tx[i]);
        tp.rt = radii[0];
        tp.ry = radii[1];
        tp.rx = radii[2];
        float *a = c->y[0], *b = c->y[1], *t0 = tmp_vol(c, 0);
        upload(c, a, v, mem);
        const int g = aux_grid(c), bt = sfk::kAuxThreads;
        sfk::k_pass_x<<<g, bt, 0, c->stream>>>(c->vol(a), c->vol(t0), tp);
        sfk::k_pass_y<<<g, bt, 0, c->stream>>>(c->vol(t0), c->vol(b), tp);
        sfk::k_pass_t<<<g, bt, 0, c->stream>>>(c->vol(b), c->vol(a), tp);
        launched(c->stream, "convolve_separable");
        download(c, out, a, mem);
        ck(cudaStreamSynchronize(c->stream), "convolve_separable");
        g_conv_count.fetch_add(1, std::memory_order_relaxed);
    });
}

int sfseg_convolve_direct_taps(sfseg_ctx* owner, uint32_t T, uint32_t H, uint32_t W, const float* v,
                               const int32_t radii[3], const double* tt, const double* ty,
                               const double* tx, float* out, int32_t mem) {
    return guarded([&] {
        if (!owner || !v || !out || !radii || !tt || !ty || !tx) fail(SFSEG_ERR_PARAMETER, "null argument");
        for (int i = 0; i < 3; ++i)
            if (radii[i] < 0 || radii[i] > 15) fail(SFSEG_ERR_CAPACITY, "direct kernel radius above 15");
        sfseg_ctx* const c = scratch_ctx(owner);  // never the resident problem
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        stage_volume(c, T, H, W, 1);
        sfk::TapsD tp;
        std::memset(&tp, 0, sizeof tp);
        for (int i = 0; i <= 2 * radii[0]; ++i) tp.t[i] = tt[i];
        for (int i = 0; i <= 2 * radii[1]; ++i) tp.y[i] = ty[i];
        for (int i = 0; i <= 2 * radii[2]; ++i) tp.x[i] = tx[i];
        tp.rt = radii[0];
        tp.ry = radii[1];
        tp.rx = radii[2];
        upload(c, c->y[0], v, mem);
        sfk::k_conv_direct<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->y[0]),
                                                                          c->vol(c->y[1]), tp);
        launched(c->stream, "convolve_direct");
        download(c, out, c->y[1], mem);
        ck(cudaStreamSynchronize(c->stream), "convolve_direct");
    });
}

// ---- time-sharded solve ----------------------------------------------------

int sfseg_shard_load(sfseg_ctx* c, uint32_t T, uint32_t H, uint32_t W, int32_t C, int32_t out_t0,
                     int32_t out_t1, int32_t halo, const float* S, const float* const* F,
                     const float* x0, int32_t mem) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        check_shape(T, H, W);
        if (C < 1) fail(SFSEG_ERR_VALIDATION, "feature set needs at least one pairwise channel");
        if (!S || !F) fail(SFSEG_ERR_PARAMETER, "null input");
        if (out_t0 < 0 || out_t1 <= out_t0 || out_t1 > static_cast<int>(T) || halo < 0)
            fail(SFSEG_ERR_PARAMETER, "bad shard range");
        drop_peers(c);  // a new shard layout: the peers must be set again
        if (out_t1 - out_t0 < halo && !(out_t0 == 0 && out_t1 == static_cast<int>(T)))
            fail(SFSEG_ERR_PARAMETER, "a shard must own at least `halo` frames");
        const int buf_t0 = std::max(0, out_t0 - halo);
        const int buf_t1 = std::min(static_cast<int>(T), out_t1 + halo);
        set_shape(c, buf_t1 - buf_t0, H, W, C, T, buf_t0, out_t0, out_t1, halo);
        c->Fw = c->F;
        c->guard_applied = false;
        c->sp_p = NAN;
        c->cur = -1;
        c->cur_u = false;
        upload(c, c->S, S, mem);
        for (int i = 0; i < C; ++i) upload(c, c->F[i], F[i], mem);
        validate_vol(c, c->S, true, "unary");
        for (int i = 0; i < C; ++i) validate_vol(c, c->F[i], false, "pairwise");
        c->has_x0 = x0 != nullptr;
        if (x0) {
            if (!c->x0) c->x0 = dalloc_vol(c);
            upload(c, c->x0, x0, mem);
            validate_vol(c, c->x0, true, "x0");
        }
        c->resident = true;
        c->q_for.clear();  // channel contents changed
        });
}

int sfseg_shard_step(sfseg_ctx* c, const sfseg_params* p, int32_t iter, sfseg_shard_io* io) {
    return guarded([&] {
        if (!c || !io) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        validate_params(p);
        if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_shard_step before sfseg_shard_load");
        if (iter > 1 && c->cur < 0) fail(SFSEG_ERR_STATE, "iteration 1 was not run");
        if (p->radii[0] > c->halo) fail(SFSEG_ERR_PARAMETER, "kernel time radius exceeds the shard halo");
        const HostKernel k = make_kernel(p->radii, p->sigmas);
        // the unit-range guard needs global min/max: the sharded driver applies
        // it to the channels before loading them (sharding.py)
        ensure_sp(c, p->p);
        if (iter == 1) {
            IterState s{};
            s.mode = 0;
            set_state(c, c->st, s);
            c->cur = -1;
            c->cur_u = false;
        }
        // k_finalize_total leaves frame_max zeroed for the next iteration
        if (iter == 1)
            ck(cudaMemsetAsync(c->frame_max, 0, std::max(c->Tout(), c->Tg) * sizeof(float), c->stream),
               "memset");
        const float* src = c->cur < 0 ? (c->has_x0 ? c->x0 : c->S) : c->y[c->cur];
        const int dst = c->cur < 0 ? 0 : 1 - c->cur;
        c->peer_push_dst = dst;
        // the same U_{k+1} rule as solve_impl, identical on every rank (the
        // halo frames pushed below are then U as well)
        const bool wu = iter < p->iterations && iter < p->binarize_start;
        c->cur_u = launch_step(c, k, p->alpha, src, c->st, c->y[dst], c->F, p->arith == SFSEG_ARITH_FAST,
                               c->cur >= 0 && c->cur_u, wu);
        c->peer_push_dst = -1;
        const size_t fr = static_cast<size_t>(c->H) * c->P;  // floats per pitched frame
        // peer-memory halo push: my first / last rt output frames straight into
        // the neighbours' halo frames of the same iterate buffer
        const int nh = std::min(c->halo, c->Tout());
        for (int side = 0; side < 2; ++side) {
            float* peer = c->peer_y[side][dst];
            if (!peer || nh == 0 || c->pushed_in_kernel) continue;
            const int g0 = side == 0 ? c->out_t0 : c->out_t1 - nh;  // global first frame sent
            const float* from = c->y[dst] + static_cast<size_t>(g0 - c->buf_t0) * fr;
            float* to = peer + static_cast<size_t>(g0 - c->peer_buf_t0[side]) * fr;
            const size_t n4 = static_cast<size_t>(nh) * fr / 4;
            sfk::k_halo_push<<<c->num_sms * 2, 256, 0, c->stream>>>(
                reinterpret_cast<const float4*>(from), reinterpret_cast<float4*>(to), n4);
            launched(c->stream, "k_halo_push");
        }
        frame_sums(c);
        c->cur = dst;
        float* y = c->y[dst];
        const int buf_t1 = c->buf_t0 + c->T;
        std::memset(io, 0, sizeof *io);
        io->halo = c->halo;
        io->out_frames = c->Tout();
        if (c->out_t0 > 0) {
            io->send_lo = y + (c->out_t0 - c->buf_t0) * fr;
            io->send_lo_bytes = std::min(c->halo, c->Tout()) * fr * sizeof(float);
            io->recv_lo = y;
            io->recv_lo_bytes = (c->out_t0 - c->buf_t0) * fr * sizeof(float);
        }
        if (c->out_t1 < c->Tg) {
            const int n = std::min(c->halo, c->Tout());
            io->send_hi = y + (c->out_t1 - n - c->buf_t0) * fr;
            io->send_hi_bytes = n * fr * sizeof(float);
            io->recv_hi = y + (c->out_t1 - c->buf_t0) * fr;
            io->recv_hi_bytes = (buf_t1 - c->out_t1) * fr * sizeof(float);
        }
        io->frame_sum = c->frame_sum;
        io->frame_max = c->frame_max;
    });
}

namespace {
struct ShardExport {  // SFSEG_SHARD_EXPORT_BYTES
    cudaIpcMemHandle_t h[2];
    uint64_t ptr[2];
    int32_t same_process, buf_t0, T, H, P, device;
    int32_t pad[2];
};
static_assert(sizeof(ShardExport) == SFSEG_SHARD_EXPORT_BYTES, "export blob size");
}  // namespace

int sfseg_shard_export(sfseg_ctx* c, int32_t same_process, void* blob) {
    return guarded([&] {
        if (!c || !blob) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (!c->resident || !c->y[0] || !c->y[1]) fail(SFSEG_ERR_STATE, "sfseg_shard_export before sfseg_shard_load");
        ShardExport e;
        std::memset(&e, 0, sizeof e);
        for (int b = 0; b < 2; ++b) {
            e.ptr[b] = reinterpret_cast<uint64_t>(c->y[b]);
            if (!same_process) ck(cudaIpcGetMemHandle(&e.h[b], c->y[b]), "cudaIpcGetMemHandle");
        }
        e.same_process = same_process ? 1 : 0;
        e.buf_t0 = c->buf_t0;
        e.T = c->T;
        e.H = c->H;
        e.P = c->P;
        e.device = c->device;
        std::memcpy(blob, &e, sizeof e);
    });
}

int sfseg_shard_set_peers(sfseg_ctx* c, const void* lo, const void* hi) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_shard_set_peers before sfseg_shard_load");
        drop_peers(c);  // the call replaces the peer set (NULL, NULL: none)
        const void* blobs[2] = {lo, hi};
        for (int side = 0; side < 2; ++side) {
            if (!blobs[side]) continue;
            ShardExport e;
            std::memcpy(&e, blobs[side], sizeof e);
            if (e.H != c->H || e.P != c->P) fail(SFSEG_ERR_SHAPE, "peer shard has another frame shape");
            // the peer's halo frames on my side must be my edge frames
            const int nh = std::min(c->halo, c->Tout());
            const int g0 = side == 0 ? c->out_t0 : c->out_t1 - nh;
            if (g0 < e.buf_t0 || g0 + nh > e.buf_t0 + e.T)
                fail(SFSEG_ERR_SHAPE, "peer shard buffer does not hold this rank's edge frames");
            for (int b = 0; b < 2; ++b) {
                if (e.same_process) {
                    if (e.device != c->device) {
                        const cudaError_t pe = cudaDeviceEnablePeerAccess(e.device, 0);
                        if (pe != cudaErrorPeerAccessAlreadyEnabled) ck(pe, "cudaDeviceEnablePeerAccess");
                        cudaGetLastError();
                    }
                    c->peer_y[side][b] = reinterpret_cast<float*>(e.ptr[b]);
                } else {
                    void* p = nullptr;
                    ck(cudaIpcOpenMemHandle(&p, e.h[b], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
                    c->peer_y[side][b] = static_cast<float*>(p);
                }
            }
            c->peer_buf_t0[side] = e.buf_t0;
            c->peer_ipc[side] = !e.same_process;
        }
    });
}

int sfseg_shard_finalize(sfseg_ctx* c, const sfseg_params* p, int32_t iter,
                         const double* frame_sum, const float* frame_max, double* norm,
                         int32_t mem) {
    return guarded([&] {
        if (!c || !frame_sum || !frame_max) fail(SFSEG_ERR_PARAMETER, "null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        validate_params(p);
        const cudaMemcpyKind kind =
            mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        // one rank: the gathered arrays are this shard's own (nothing to copy)
        if (frame_sum != c->frame_sum)
            ck(cudaMemcpyAsync(c->frame_sum, frame_sum, c->Tg * sizeof(double), kind, c->stream), "sums");
        if (frame_max != c->frame_max)
            ck(cudaMemcpyAsync(c->frame_max, frame_max, c->Tg * sizeof(float), kind, c->stream), "max");
        const int mode_next = iter >= p->binarize_start ? 2 : 1;
        if (c->norms_cap < iter) {
            double* nn = nullptr;
            const int cap = std::max(64, 2 * iter);
            ck(cudaMalloc(&nn, cap * sizeof(double)), "cudaMalloc norms");
            if (c->norms) {
                ck(cudaMemcpyAsync(nn, c->norms, c->norms_cap * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->stream), "norms");
                ck(cudaStreamSynchronize(c->stream), "norms");
                cudaFree(c->norms);
            }
            c->norms = nn;
            c->norms_cap = cap;
        }
        launch_pdl(sfk::k_finalize_total, 1, sfk::kAuxThreads, 0, c->stream,
                   static_cast<const double*>(c->frame_sum), c->frame_max, c->Tg, c->st, c->norms,
                   iter - 1, mode_next, lambda_for(p, iter), p->threshold_frac);
        launched(c->stream, "k_finalize_total");
        if (norm) {
            const IterState s = get_state(c, c->st);
            *norm = s.norm;
            if (s.norm == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
        }
    });
}

int sfseg_shard_norms(sfseg_ctx* c, int32_t count, double* norms) {
    return guarded([&] {
        if (!c || !norms) fail(SFSEG_ERR_PARAMETER, "null argument");
        if (count < 0 || count > c->norms_cap) fail(SFSEG_ERR_PARAMETER, "bad norm count");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaMemcpyAsync(norms, c->norms, count * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), "norms");
        ck(cudaStreamSynchronize(c->stream), "norms");
        for (int i = 0; i < count; ++i)
            if (norms[i] == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
    });
}

int sfseg_shard_download(sfseg_ctx* c, double frac, float* soft, uint8_t* mask, int32_t mem) {
    return guarded([&] {
        if (!c) fail(SFSEG_ERR_PARAMETER, "null ctx");
        std::lock_guard<std::mutex> lk(c->mu);
        if (!c->resident) fail(SFSEG_ERR_STATE, "sfseg_shard_download before sfseg_shard_load");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        float* x = tmp_vol(c, 0);
        materialize(c, x);
        const Vol xo = c->out_vol(x);
        const cudaMemcpyKind kind =
            mem == SFSEG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (soft)
            ck(cudaMemcpy2DAsync(soft, c->W * sizeof(float), xo.p, c->P * sizeof(float),
                                 c->W * sizeof(float), static_cast<size_t>(xo.T) * c->H, kind,
                                 c->stream),
               "download shard");
        if (mask) {
            // global max of the projected iterate comes from the shared state
            if (c->cur < 0) fail(SFSEG_ERR_STATE, "no iteration has run");
            sfk::k_state_max<<<1, 1, 0, c->stream>>>(c->st, c->scratch_f);
            const size_t n = static_cast<size_t>(xo.T) * c->H * c->W;
            uint8_t* dm = mem == SFSEG_MEM_DEVICE ? mask : nullptr;
            if (!dm) ck(cudaMallocAsync(reinterpret_cast<void**>(&dm), n, c->stream), "malloc");
            sfk::k_mask<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(xo, c->scratch_f, frac, dm);
            launched(c->stream, "k_mask");
            if (mem != SFSEG_MEM_DEVICE) {
                ck(cudaMemcpyAsync(mask, dm, n, cudaMemcpyDeviceToHost, c->stream), "mask D2H");
                ck(cudaFreeAsync(dm, c->stream), "free");
            }
        }
        ck(cudaStreamSynchronize(c->stream), "shard download");
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// In-process multi-GPU solve (SFSEG_NUM_GPUS in the drop-in): time shards on
// several devices of one process, every exchange device-side and ordered by
// events; no per-iteration host synchronisation, no collective library.
//   per iteration, shard i (its own device and stream):
//     1. fused step over its frames; the rt edge planes of the new iterate go
//        straight into the neighbours' halo frames (peer stores, in-kernel for
//        the FAST single-channel kernel, else k_halo_push); per-frame sums
//        and maxima of its frames (frame_sums); event done[i]
//     2. waits for done[j] of every shard, copies their per-frame sums and
//        maxima into its own frame-ordered arrays (peer copies), and runs the
//        same frame-ordered finalize as a single context: every shard derives
//        bit-identical norms and projection scalars
//   The per-frame results are copied into one of two published sets by
//   iteration parity, so a shard's step k+1 never overwrites what a slower
//   shard still gathers.
struct sfseg_multi {
    std::vector<sfseg_ctx*> shards;
    std::vector<int> t0, t1;
    std::vector<double*> fsum[2];  // per shard: its frame sums, by iteration parity
    std::vector<float*> fmax[2];
    std::vector<double*> gsum;     // per shard: all Tg frame sums, frame order
    std::vector<float*> gmax;
    std::vector<cudaEvent_t> done;
    int T = 0, halo = -1;
    std::mutex mu;
};

namespace {

void multi_free_buffers(sfseg_multi* m) {
    for (size_t i = 0; i < m->shards.size(); ++i) {
        cudaSetDevice(m->shards[i]->device);
        for (int b = 0; b < 2; ++b) {
            if (i < m->fsum[b].size() && m->fsum[b][i]) cudaFree(m->fsum[b][i]);
            if (i < m->fmax[b].size() && m->fmax[b][i]) cudaFree(m->fmax[b][i]);
        }
        if (i < m->gsum.size() && m->gsum[i]) cudaFree(m->gsum[i]);
        if (i < m->gmax.size() && m->gmax[i]) cudaFree(m->gmax[i]);
    }
    for (int b = 0; b < 2; ++b) {
        m->fsum[b].clear();
        m->fmax[b].clear();
    }
    m->gsum.clear();
    m->gmax.clear();
}

// global unit-range guard (engine.cpp:254-259) across shards: min/max of each
// channel over every shard's frames, then the same rescale on every shard
void multi_guard(sfseg_multi* m, int C) {
    for (int ch = 0; ch < C; ++ch) {
        float lo = INFINITY, hi = -INFINITY;
        for (sfseg_ctx* c : m->shards) {
            ck(cudaSetDevice(c->device), "cudaSetDevice");
            const int nb = aux_grid(c);
            sfk::k_minmax_blocks<<<nb, sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->F[ch]), c->bminmax,
                                                                        c->bminmax + nb);
            sfk::k_minmax_final<<<1, sfk::kAuxThreads, 0, c->stream>>>(c->bminmax, c->bminmax + nb, nb,
                                                                     c->scratch_f);
            float lh[2];
            ck(cudaMemcpyAsync(lh, c->scratch_f, sizeof lh, cudaMemcpyDeviceToHost, c->stream), "minmax");
            ck(cudaStreamSynchronize(c->stream), "sync");
            lo = std::min(lo, lh[0]);
            hi = std::max(hi, lh[1]);
        }
        if (lo >= 0.0f && hi <= 1.0f) continue;  // bits untouched
        const float lohi[2] = {lo, hi};
        for (sfseg_ctx* c : m->shards) {
            ck(cudaSetDevice(c->device), "cudaSetDevice");
            ck(cudaMemcpyAsync(c->scratch_f, lohi, sizeof lohi, cudaMemcpyHostToDevice, c->stream), "lohi");
            sfk::k_unit_range<<<aux_grid(c), sfk::kAuxThreads, 0, c->stream>>>(c->vol(c->F[ch]), c->scratch_f);
            launched(c->stream, "k_unit_range");
            ck(cudaStreamSynchronize(c->stream), "sync");  // lohi is a host stack array
        }
    }
}

}  // namespace

extern "C" {

int sfseg_multi_create(int32_t n, const int32_t* devices, sfseg_multi** out) {
    return guarded([&] {
        if (!out || n < 1) fail(SFSEG_ERR_PARAMETER, "bad argument");
        auto m = std::make_unique<sfseg_multi>();
        for (int i = 0; i < n; ++i) {
            sfseg_ctx* c = nullptr;
            const int rc = sfseg_ctx_create(devices ? devices[i] : i, &c);
            if (rc != SFSEG_OK) {
                for (sfseg_ctx* d : m->shards) sfseg_ctx_destroy(d);
                fail(rc, sfseg_last_error());
            }
            m->shards.push_back(c);
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            m->done.push_back(e);
        }
        // neighbours on other devices address each other's buffers directly
        for (int i = 0; i + 1 < n; ++i) {
            const int a = m->shards[i]->device, b = m->shards[i + 1]->device;
            if (a == b) continue;
            for (auto [x, y] : {std::pair<int, int>{a, b}, std::pair<int, int>{b, a}}) {
                int can = 0;
                ck(cudaDeviceCanAccessPeer(&can, x, y), "cudaDeviceCanAccessPeer");
                if (!can) fail(SFSEG_ERR_CUDA, "devices without peer access");
                ck(cudaSetDevice(x), "cudaSetDevice");
                const cudaError_t e = cudaDeviceEnablePeerAccess(y, 0);
                if (e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
                cudaGetLastError();
            }
        }
        *out = m.release();
    });
}

int sfseg_multi_destroy(sfseg_multi* m) {
    return guarded([&] {
        if (!m) return;
        multi_free_buffers(m);
        for (size_t i = 0; i < m->shards.size(); ++i) {
            cudaSetDevice(m->shards[i]->device);
            cudaEventDestroy(m->done[i]);
            sfseg_ctx_destroy(m->shards[i]);
        }
        delete m;
    });
}

int sfseg_multi_size(const sfseg_multi* m) { return m ? static_cast<int>(m->shards.size()) : 0; }

int sfseg_multi_run(sfseg_multi* m, uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                    const float* const* F, const float* x0, const sfseg_params* p, float* soft,
                    uint8_t* mask, sfseg_iter_record* rec, int32_t mem) {
    return guarded([&] {
        if (!m || !S || !F || !p) fail(SFSEG_ERR_PARAMETER, "null argument");
        validate_params(p);
        check_shape(T, H, W);
        if (C < 1) fail(SFSEG_ERR_VALIDATION, "feature set needs at least one pairwise channel");
        std::lock_guard<std::mutex> lk(m->mu);
        const int halo = p->radii[0];
        // shards of at least max(halo, 1) frames: a halo comes from one neighbour
        const int n = std::max(1, std::min<int>(static_cast<int>(m->shards.size()),
                                                static_cast<int>(T) / std::max(1, halo)));
        const size_t frame = static_cast<size_t>(H) * W;
        m->t0.assign(n, 0);
        m->t1.assign(n, 0);
        for (int i = 0; i < n; ++i) {  // balanced contiguous frames (sharding.py shard_range)
            const int base = static_cast<int>(T) / n, rem = static_cast<int>(T) % n;
            m->t0[i] = i * base + std::min(i, rem);
            m->t1[i] = m->t0[i] + base + (i < rem ? 1 : 0);
        }
        multi_free_buffers(m);
        for (int i = 0; i < n; ++i) {
            sfseg_ctx* c = m->shards[i];
            const int b0 = std::max(0, m->t0[i] - halo);
            std::vector<const float*> Fi(C);
            for (int ch = 0; ch < C; ++ch) Fi[ch] = F[ch] + b0 * frame;
            const int rc = sfseg_shard_load(c, T, H, W, C, m->t0[i], m->t1[i], halo, S + b0 * frame,
                                            Fi.data(), x0 ? x0 + b0 * frame : nullptr, mem);
            if (rc != SFSEG_OK) fail(rc, sfseg_last_error());
        }
        std::vector<sfseg_ctx*> sh(m->shards.begin(), m->shards.begin() + n);
        if (!p->allow_negative_affinity) multi_guard(m, C);
        for (int i = 0; i < n; ++i) {
            sfseg_ctx* c = sh[i];
            ck(cudaSetDevice(c->device), "cudaSetDevice");
            for (int b = 0; b < 2; ++b) {
                double* s2 = nullptr;
                float* m2 = nullptr;
                ck(cudaMalloc(&s2, c->Tout() * sizeof(double)), "malloc");
                ck(cudaMalloc(&m2, c->Tout() * sizeof(float)), "malloc");
                m->fsum[b].push_back(s2);
                m->fmax[b].push_back(m2);
            }
            double* gs = nullptr;
            float* gm = nullptr;
            ck(cudaMalloc(&gs, T * sizeof(double)), "malloc");
            ck(cudaMalloc(&gm, T * sizeof(float)), "malloc");
            m->gsum.push_back(gs);
            m->gmax.push_back(gm);
            // neighbours' iterate buffers (same process: plain pointers)
            drop_peers(c);
            for (int side = 0; side < 2; ++side) {
                const int j = side == 0 ? i - 1 : i + 1;
                if (j < 0 || j >= n) continue;
                for (int b = 0; b < 2; ++b) c->peer_y[side][b] = sh[j]->y[b];
                c->peer_buf_t0[side] = sh[j]->buf_t0;
                c->peer_ipc[side] = false;
            }
            if (c->norms_cap < p->iterations) {
                if (c->norms) cudaFree(c->norms);
                c->norms = nullptr;
                ck(cudaMalloc(&c->norms, p->iterations * sizeof(double)), "cudaMalloc norms");
                c->norms_cap = p->iterations;
            }
            ensure_sp(c, p->p);
            IterState s0{};
            set_state(c, c->st, s0);
            c->cur = -1;
            c->cur_u = false;
        }
        const HostKernel k = make_kernel(p->radii, p->sigmas);
        const bool fast = p->arith == SFSEG_ARITH_FAST;
        // per-iteration times on shard 0's stream (its finalize waits for every shard)
        ck(cudaSetDevice(sh[0]->device), "cudaSetDevice");
        std::vector<cudaEvent_t> iev(p->iterations + 1);
        for (auto& e : iev) ck(cudaEventCreate(&e), "event");
        ck(cudaEventRecord(iev[0], sh[0]->stream), "event");
        for (int it = 1; it <= p->iterations; ++it) {
            const int par = it & 1;
            const bool wu = it < p->iterations && it < p->binarize_start;
            bool wrote_u = false;
            for (int i = 0; i < n; ++i) {
                sfseg_ctx* c = sh[i];
                ck(cudaSetDevice(c->device), "cudaSetDevice");
                ck(cudaMemsetAsync(c->frame_max, 0, c->Tout() * sizeof(float), c->stream), "memset");
                const float* src = c->cur < 0 ? (c->has_x0 ? c->x0 : c->S) : c->y[c->cur];
                const int dst = c->cur < 0 ? 0 : 1 - c->cur;
                c->peer_push_dst = dst;
                wrote_u = launch_step(c, k, p->alpha, src, c->st, c->y[dst], c->F, fast,
                                      c->cur >= 0 && c->cur_u, wu);
                c->peer_push_dst = -1;
                const size_t fr = static_cast<size_t>(c->H) * c->P;
                const int nh = std::min(c->halo, c->Tout());
                for (int side = 0; side < 2 && !c->pushed_in_kernel; ++side) {
                    float* peer = c->peer_y[side][dst];
                    if (!peer || nh == 0) continue;
                    const int g0 = side == 0 ? c->out_t0 : c->out_t1 - nh;
                    sfk::k_halo_push<<<c->num_sms * 2, 256, 0, c->stream>>>(
                        reinterpret_cast<const float4*>(c->y[dst] + static_cast<size_t>(g0 - c->buf_t0) * fr),
                        reinterpret_cast<float4*>(peer + static_cast<size_t>(g0 - c->peer_buf_t0[side]) * fr),
                        static_cast<size_t>(nh) * fr / 4);
                    launched(c->stream, "k_halo_push");
                }
                frame_sums(c);
                ck(cudaMemcpyAsync(m->fsum[par][i], c->frame_sum, c->Tout() * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->stream), "publish sums");
                ck(cudaMemcpyAsync(m->fmax[par][i], c->frame_max, c->Tout() * sizeof(float),
                                   cudaMemcpyDeviceToDevice, c->stream), "publish max");
                c->cur = dst;
                ck(cudaEventRecord(m->done[i], c->stream), "event");
            }
            const int mode_next = it >= p->binarize_start ? 2 : 1;
            for (int i = 0; i < n; ++i) {
                sfseg_ctx* c = sh[i];
                ck(cudaSetDevice(c->device), "cudaSetDevice");
                c->cur_u = wrote_u;
                for (int j = 0; j < n; ++j) {
                    ck(cudaStreamWaitEvent(c->stream, m->done[j], 0), "wait");
                    const int tj = m->t1[j] - m->t0[j];
                    ck(cudaMemcpyAsync(m->gsum[i] + m->t0[j], m->fsum[par][j], tj * sizeof(double),
                                       cudaMemcpyDefault, c->stream), "gather sums");
                    ck(cudaMemcpyAsync(m->gmax[i] + m->t0[j], m->fmax[par][j], tj * sizeof(float),
                                       cudaMemcpyDefault, c->stream), "gather max");
                }
                sfk::k_finalize_total<<<1, sfk::kAuxThreads, 0, c->stream>>>(
                    m->gsum[i], m->gmax[i], static_cast<int>(T), c->st, c->norms, it - 1, mode_next,
                    lambda_for(p, it), p->threshold_frac);
                launched(c->stream, "k_finalize_total");
                if (i == 0) ck(cudaEventRecord(iev[it], c->stream), "event");
            }
        }
        // download: each shard's own frames; the mask cut comes from the
        // shared (identical) projection state
        std::vector<double> norms(p->iterations);
        for (int i = 0; i < n; ++i) {
            sfseg_ctx* c = sh[i];
            ck(cudaSetDevice(c->device), "cudaSetDevice");
            if (i == 0)
                ck(cudaMemcpyAsync(norms.data(), c->norms, p->iterations * sizeof(double),
                                   cudaMemcpyDeviceToHost, c->stream), "norms");
            ck(cudaStreamSynchronize(c->stream), "solve");
        }
        for (double v : norms)
            if (v == 0.0) fail(SFSEG_ERR_DEGENERATE, "iterate collapsed to the zero vector");
        for (int i = 0; i < n; ++i) {
            sfseg_ctx* c = sh[i];
            const size_t off = static_cast<size_t>(m->t0[i]) * frame;
            const int rc = sfseg_shard_download(c, p->final_threshold, soft ? soft + off : nullptr,
                                                mask ? mask + off : nullptr, mem);
            if (rc != SFSEG_OK) fail(rc, sfseg_last_error());
        }
        for (int i = 0; i < p->iterations; ++i) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, iev[i], iev[i + 1]);
            if (rec) {
                rec[i].iter = i + 1;
                rec[i].l2_norm_pre_normalize = norms[i];
                rec[i].angle_deg = NAN;
                rec[i].iou = NAN;
                rec[i].wall_time_s = ms * 1e-3;
            }
        }
        ck(cudaSetDevice(sh[0]->device), "cudaSetDevice");
        for (auto e : iev) cudaEventDestroy(e);
    });
}

}  // extern "C"

namespace {
__global__ void k_guard_count(const uint32_t* lo, const uint32_t* hi, size_t n, uint32_t pat,
                              unsigned long long* bad) {
    unsigned long long mine = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        mine += (lo[i] != pat) + (hi[i] != pat);
    if (mine) atomicAdd(bad, mine);
}
}  // namespace

// SFSEG_DEBUG_GUARD=1: counts the guard-band words of every live volume buffer
// (all contexts of the process) that no longer hold the fill pattern, i.e.
// out-of-bounds stores by any kernel since the buffer was allocated.
// *buffers receives the number of buffers checked. Returns SFSEG_ERR_STATE
// when the library is not in guard mode.
extern "C" int sfseg_debug_check_guards(unsigned long long* bad_words, int32_t* buffers) {
    return guarded([&] {
        if (!bad_words) fail(SFSEG_ERR_PARAMETER, "null argument");
        if (!guard_mode()) fail(SFSEG_ERR_STATE, "SFSEG_DEBUG_GUARD is not set");
        std::lock_guard<std::mutex> lk(g_guard_mu);
        unsigned long long total = 0;
        for (auto& [ptr, n] : g_guarded) {
            cudaPointerAttributes at{};
            ck(cudaPointerGetAttributes(&at, ptr), "pointer attributes");
            ck(cudaSetDevice(at.device), "cudaSetDevice");
            ck(cudaDeviceSynchronize(), "sync");
            unsigned long long* d = nullptr;
            ck(cudaMalloc(&d, sizeof *d), "malloc");
            ck(cudaMemset(d, 0, sizeof *d), "memset");
            k_guard_count<<<64, 256>>>(reinterpret_cast<const uint32_t*>(ptr - kGuard),
                                       reinterpret_cast<const uint32_t*>(ptr + n), kGuard, kPoison, d);
            unsigned long long h = 0;
            ck(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost), "D2H");
            cudaFree(d);
            total += h;
        }
        *bad_words = total;
        if (buffers) *buffers = static_cast<int32_t>(g_guarded.size());
    });
}

// test hook of the checker itself: overwrites `words` words of the first live
// buffer's upper guard band (what a kernel storing past its buffer would do)
extern "C" int sfseg_debug_poke_guard(int32_t words) {
    return guarded([&] {
        if (!guard_mode()) fail(SFSEG_ERR_STATE, "SFSEG_DEBUG_GUARD is not set");
        std::lock_guard<std::mutex> lk(g_guard_mu);
        if (g_guarded.empty() || words < 0 || static_cast<size_t>(words) > kGuard)
            fail(SFSEG_ERR_PARAMETER, "nothing to poke");
        ck(cudaMemset(g_guarded[0].first + g_guarded[0].second, 0, words * sizeof(float)), "poke");
    });
}

