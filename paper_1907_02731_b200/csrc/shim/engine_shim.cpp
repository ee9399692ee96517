// engine_shim.cpp — the drop-in: the reference's engine.o and conv3d.o symbols
// (proj/include/sfseg/engine.hpp:56-109, conv3d.hpp:55-72) implemented on the
// sm_100a library through its C ABI (include/sfseg_cuda.h).
//
// Linking libsfseg_engine_cuda.so ahead of the reference's remaining objects
// (volume.o, metrics.o, oracle.o, synth.o, bench.o) replaces the CPU engine
// without touching the reference headers or any caller. Exceptions are the
// reference's own types (errors.hpp:17-68); CUDA failures become sfseg::Error.
//
// Environment: SFSEG_DEVICE (default 0) picks the GPU; SFSEG_ARITH=fast
// selects fused multiply-adds (default "exact": the reference's rounding).
// SfsegConfig::threads is accepted and ignored, as the reference guarantees
// thread-count-invariant results (README.md:174-189).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sfseg/conv3d.hpp"
#include "sfseg/engine.hpp"
#include "sfseg/errors.hpp"
#include "sfseg/metrics.hpp"
#include "sfseg/volume.hpp"
#include "sfseg_cuda.h"

namespace {

std::mutex g_mu;
sfseg_ctx* g_ctx = nullptr;

[[noreturn]] void rethrow(int rc) {
    const std::string msg = sfseg_last_error();
    switch (rc) {
        case SFSEG_ERR_PARAMETER: throw sfseg::ParameterError(msg);
        case SFSEG_ERR_SHAPE: throw sfseg::ShapeError(msg);
        case SFSEG_ERR_VALIDATION: throw sfseg::ValidationError(msg);
        case SFSEG_ERR_DEGENERATE: throw sfseg::DegenerateSolutionError(msg);
        case SFSEG_ERR_CAPACITY: throw sfseg::CapacityError(msg);
        default: throw sfseg::Error("sfseg_cuda: " + msg);
    }
}

void check(int rc) {
    if (rc != SFSEG_OK) rethrow(rc);
}

sfseg_ctx* ctx() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) {
        const char* d = std::getenv("SFSEG_DEVICE");
        check(sfseg_ctx_create(d ? std::atoi(d) : 0, &g_ctx));
    }
    return g_ctx;
}

int arith() {
    const char* a = std::getenv("SFSEG_ARITH");
    return a && std::string(a) == "fast" ? SFSEG_ARITH_FAST : SFSEG_ARITH_EXACT;
}

sfseg_params to_params(const sfseg::SfsegConfig& c) {
    sfseg_params p;
    sfseg_params_default(&p);
    p.alpha = c.alpha;
    p.p = c.p;
    for (int a = 0; a < 3; ++a) {
        p.radii[a] = c.kernel.radii[a];
        p.sigmas[a] = c.kernel.sigmas[a];
    }
    p.iterations = c.iterations;
    p.temporal_window = c.temporal_window;
    p.binarize_start = c.binarize_start;
    p.sigmoid_slope0 = c.sigmoid_slope0;
    p.slope_growth = c.slope_growth;
    p.threshold_frac = c.threshold_frac;
    p.final_threshold = c.final_threshold;
    p.allow_negative_affinity = c.allow_negative_affinity ? 1 : 0;
    p.arith = arith();
    return p;
}

void same_shape(const sfseg::FeatureVolume& a, const sfseg::FeatureVolume& b, const char* what) {
    if (!(a.shape() == b.shape())) throw sfseg::ShapeError(std::string("shape mismatch: ") + what);
}

sfseg::FeatureVolume slice_frames(const sfseg::FeatureVolume& v, std::uint32_t t0,
                                  std::uint32_t t1) {
    const auto& s = v.shape();
    const std::size_t plane = static_cast<std::size_t>(s.height) * s.width;
    sfseg::FeatureVolume out(sfseg::VolumeShape{t1 - t0 + 1, s.height, s.width}, v.role());
    std::memcpy(out.data(), v.data() + static_cast<std::size_t>(t0) * plane,
                sizeof(float) * out.size());
    return out;
}

// unit-range guard on a host copy (engine.cpp:228-243); only the FrameTransform
// path needs host-side channels, the resident solve applies it on the GPU
void unit_range_host(sfseg::FeatureVolume& f) {
    float lo = f.data()[0], hi = f.data()[0];
    for (float v : f.values()) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
    }
    if (lo >= 0.0f && hi <= 1.0f) return;
    float* p = f.data();
    if (hi > lo) {
        const float span = hi - lo;
        for (std::size_t i = 0; i < f.size(); ++i) p[i] = (p[i] - lo) / span;
    } else {
        const float c = std::clamp(lo, 0.0f, 1.0f);
        for (std::size_t i = 0; i < f.size(); ++i) p[i] = c;
    }
}

}  // namespace

namespace sfseg {

// ---- engine.o ----------------------------------------------------------------

void SfsegConfig::validate() const {
    const sfseg_params p = to_params(*this);
    check(sfseg_params_validate(&p));
}

FeatureVolume sfseg_step_channel(const FeatureVolume& x, const FeatureVolume& s,
                                 const FeatureVolume& f, const SfsegConfig& cfg) {
    cfg.validate();  // engine.cpp:133-135
    same_shape(x, s, "solution vs unary");
    same_shape(x, f, "solution vs pairwise");
    const sfseg_params p = to_params(cfg);
    const auto& sh = x.shape();
    FeatureVolume out(sh, VolumeRole::solution);
    check(sfseg_step_channel(ctx(), sh.frames, sh.height, sh.width, x.data(), s.data(), f.data(),
                             &p, out.data(), SFSEG_MEM_HOST));
    return out;
}

FeatureVolume sfseg_step(const FeatureVolume& x, const FeatureSet& features,
                         const SfsegConfig& cfg) {
    cfg.validate();  // engine.cpp:143-146
    if (features.pairwise.empty())
        throw ParameterError("sfseg_step needs at least one pairwise channel");
    same_shape(x, features.unary, "solution vs unary");
    for (const auto& f : features.pairwise) same_shape(x, f, "solution vs pairwise");
    const sfseg_params p = to_params(cfg);
    const auto& sh = x.shape();
    std::vector<const float*> F;
    for (const auto& f : features.pairwise) F.push_back(f.data());
    FeatureVolume out(sh, VolumeRole::solution);
    check(sfseg_step(ctx(), sh.frames, sh.height, sh.width, static_cast<int32_t>(F.size()),
                     x.data(), features.unary.data(), F.data(), &p, out.data(), SFSEG_MEM_HOST));
    return out;
}

std::pair<FeatureVolume, double> normalize_l2(const FeatureVolume& x) {
    const auto& sh = x.shape();
    FeatureVolume out(sh, x.role());
    double norm = 0.0;
    check(sfseg_normalize_l2(ctx(), sh.frames, sh.height, sh.width, x.data(), out.data(), &norm,
                             SFSEG_MEM_HOST));
    return {std::move(out), norm};
}

FeatureVolume project_binary(const FeatureVolume& x, int iter, const SfsegConfig& cfg) {
    if (iter < cfg.binarize_start) return x;  // engine.cpp:186
    const sfseg_params p = to_params(cfg);
    const auto& sh = x.shape();
    FeatureVolume out(sh, x.role());
    check(sfseg_project_binary(ctx(), sh.frames, sh.height, sh.width, x.data(), iter, &p,
                               out.data(), SFSEG_MEM_HOST));
    return out;
}

BinaryMask threshold_final(const FeatureVolume& x, double frac) {
    const auto& sh = x.shape();
    BinaryMask m;
    m.shape = sh;
    m.values.resize(x.size());
    check(sfseg_threshold_final(ctx(), sh.frames, sh.height, sh.width, x.data(), frac,
                                m.values.data(), SFSEG_MEM_HOST));
    return m;
}

namespace {

// run() with a FrameTransform: the per-frame windowed sweep of
// engine.cpp:287-325 with the hook on host slices and every step on the GPU
RunResult run_windowed(const FeatureSet& features, const SfsegConfig& cfg,
                       const FeatureVolume* x0, const FeatureVolume* reference,
                       const BinaryMask* ground_truth, const FrameTransform& transform,
                       const IterationObserver& observer) {
    const VolumeShape shape = features.shape();
    FeatureSet work = features;
    if (!cfg.allow_negative_affinity)
        for (auto& f : work.pairwise) unit_range_host(f);
    FeatureVolume x = x0 ? *x0 : work.unary;
    x.set_role(VolumeRole::solution);
    const int w = cfg.resolved_temporal_window();
    const std::size_t plane = static_cast<std::size_t>(shape.height) * shape.width;
    RunTrace trace;
    for (int iter = 1; iter <= cfg.iterations; ++iter) {
        const auto tick = std::chrono::steady_clock::now();
        FeatureVolume x_next(shape, VolumeRole::solution);
        for (std::uint32_t i = 0; i < shape.frames; ++i) {
            const std::uint32_t t0 = i >= static_cast<std::uint32_t>(w) ? i - w : 0;
            const std::uint32_t t1 = std::min<std::uint32_t>(shape.frames - 1, i + w);
            FeatureSet ws;
            FeatureVolume x_w = slice_frames(x, t0, t1);
            for (const auto& f : work.pairwise) ws.pairwise.push_back(slice_frames(f, t0, t1));
            ws.unary = slice_frames(work.unary, t0, t1);
            transform(ws.unary, ws.pairwise, x_w, i);
            const FeatureVolume step = sfseg_step(x_w, ws, cfg);  // S^p of the slice on the GPU
            std::memcpy(x_next.data() + i * plane, step.data() + (i - t0) * plane,
                        sizeof(float) * plane);
        }
        auto [x_unit, norm] = normalize_l2(x_next);
        x = project_binary(x_unit, iter, cfg);
        IterationRecord rec;
        rec.iter = iter;
        rec.l2_norm_pre_normalize = norm;
        rec.wall_time_s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tick).count();
        if (reference) rec.angle_deg = angle_degrees(x, *reference);
        if (ground_truth) rec.iou = jaccard(threshold_final(x, cfg.threshold_frac), *ground_truth);
        trace.iterations.push_back(rec);
        if (observer) observer(iter, x);
    }
    RunResult r;
    r.mask = threshold_final(x, cfg.final_threshold);
    r.soft = std::move(x);
    r.trace = std::move(trace);
    return r;
}

}  // namespace

RunResult run(const FeatureSet& features, const SfsegConfig& cfg, const FeatureVolume* x0,
              const FeatureVolume* reference, const BinaryMask* ground_truth,
              const FrameTransform& transform, const IterationObserver& observer) {
    cfg.validate();  // engine.cpp:250
    if (features.pairwise.empty())
        throw ValidationError("feature set needs at least one pairwise channel");
    const VolumeShape shape = features.shape();
    for (const auto& f : features.pairwise)
        if (!(f.shape() == shape))
            throw ShapeError("pairwise channel shape differs from unary shape");
    if (x0 && !(x0->shape() == shape)) throw ShapeError("x0 shape differs from features");
    if (reference && !(reference->shape() == shape))
        throw ShapeError("reference shape differs from features");
    if (ground_truth && !(ground_truth->shape == shape))
        throw ShapeError("ground truth shape differs from features");
    if (transform) {
        // values are validated on the GPU by the non-hooked path; here the
        // reference's own checks run first, as engine.cpp:250-266 does
        features.validate();
        if (x0) {
            FeatureVolume v = *x0;
            v.set_role(VolumeRole::solution);
            v.validate();
        }
        return run_windowed(features, cfg, x0, reference, ground_truth, transform, observer);
    }

    sfseg_ctx* c = ctx();
    const sfseg_params p = to_params(cfg);
    std::vector<const float*> F;
    for (const auto& f : features.pairwise) F.push_back(f.data());
    check(sfseg_load(c, shape.frames, shape.height, shape.width, static_cast<int32_t>(F.size()),
                     features.unary.data(), F.data(), x0 ? x0->data() : nullptr, SFSEG_MEM_HOST));
    RunResult r;
    r.trace.iterations.reserve(static_cast<std::size_t>(cfg.iterations));
    const bool per_iter = observer || reference || ground_truth;
    if (!per_iter) {
        std::vector<sfseg_iter_record> rec(static_cast<std::size_t>(cfg.iterations));
        check(sfseg_solve(c, &p, 1, cfg.iterations, rec.data()));
        for (const auto& e : rec) {
            IterationRecord ir;
            ir.iter = e.iter;
            ir.l2_norm_pre_normalize = e.l2_norm_pre_normalize;
            ir.wall_time_s = e.wall_time_s;
            r.trace.iterations.push_back(ir);
        }
    } else {
        FeatureVolume x(shape, VolumeRole::solution);
        for (int it = 1; it <= cfg.iterations; ++it) {
            sfseg_iter_record e;
            check(sfseg_solve(c, &p, it, it, &e));
            IterationRecord ir;
            ir.iter = e.iter;
            ir.l2_norm_pre_normalize = e.l2_norm_pre_normalize;
            ir.wall_time_s = e.wall_time_s;
            if (reference || ground_truth) {
                double ang = 0.0, iou = 0.0;
                check(sfseg_metrics(c, reference ? reference->data() : nullptr,
                                    ground_truth ? ground_truth->values.data() : nullptr,
                                    cfg.threshold_frac, &ang, &iou, SFSEG_MEM_HOST));
                if (reference) ir.angle_deg = ang;
                if (ground_truth) ir.iou = iou;
            }
            r.trace.iterations.push_back(ir);
            if (observer) {
                check(sfseg_download(c, cfg.final_threshold, x.data(), nullptr, SFSEG_MEM_HOST));
                observer(it, x);
            }
        }
    }
    r.soft = FeatureVolume(shape, VolumeRole::solution);
    r.mask.shape = shape;
    r.mask.values.resize(shape.voxels());
    check(sfseg_download(c, cfg.final_threshold, r.soft.data(), r.mask.values.data(),
                         SFSEG_MEM_HOST));
    return r;
}

// ---- conv3d.o ----------------------------------------------------------------

SeparableKernel3D make_gaussian_kernel(const std::array<double, 3>& sigmas,
                                       const std::array<int, 3>& radii) {
    for (double s : sigmas)
        if (!(s > 0.0)) throw ParameterError("kernel sigma must be positive");
    for (int r : radii)
        if (r < 0) throw ParameterError("kernel radius must be nonnegative");
    SeparableKernel3D k;
    k.sigmas = sigmas;
    k.radii = radii;
    k.taps_t.resize(2 * radii[0] + 1);
    k.taps_y.resize(2 * radii[1] + 1);
    k.taps_x.resize(2 * radii[2] + 1);
    const int32_t r[3] = {radii[0], radii[1], radii[2]};
    check(sfseg_make_kernel(r, sigmas.data(), k.taps_t.data(), k.taps_y.data(), k.taps_x.data()));
    return k;
}

SeparableKernel3D make_gaussian_kernel(const KernelConfig& cfg) {
    return make_gaussian_kernel(cfg.sigmas, cfg.radii);
}

FeatureVolume convolve_separable(const FeatureVolume& v, const SeparableKernel3D& k, int) {
    const auto& s = v.shape();
    s.validate();
    FeatureVolume out(s, v.role());
    const int32_t r[3] = {k.radii[0], k.radii[1], k.radii[2]};
    check(sfseg_convolve_separable_taps(ctx(), s.frames, s.height, s.width, v.data(), r,
                                        k.taps_t.data(), k.taps_y.data(), k.taps_x.data(),
                                        out.data(), SFSEG_MEM_HOST));
    return out;
}

FeatureVolume convolve_direct(const FeatureVolume& v, const SeparableKernel3D& k, int) {
    const auto& s = v.shape();
    s.validate();
    FeatureVolume out(s, v.role());
    const int32_t r[3] = {k.radii[0], k.radii[1], k.radii[2]};
    check(sfseg_convolve_direct_taps(ctx(), s.frames, s.height, s.width, v.data(), r,
                                     k.taps_t.data(), k.taps_y.data(), k.taps_x.data(),
                                     out.data(), SFSEG_MEM_HOST));
    return out;
}

std::uint64_t separable_convolution_count() { return sfseg_separable_convolution_count(); }

}  // namespace sfseg
