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
// SFSEG_NUM_GPUS=N (SfsegConfig has no device field and stays unchanged)
// runs run() time-sharded over N GPUs of this process (sfseg_multi_run:
// peer-memory halos, bit-identical results); SFSEG_MULTI_DEVICES=0,0,1,...
// maps the shards to devices explicitly (tests put several on one GPU).
// SfsegConfig::threads is accepted and ignored, as the reference guarantees
// thread-count-invariant results (README.md:174-189).
//
// Threading: the reference's functions are pure and
// reentrant. Here every call leases a library context from a pool for its
// whole duration (load, solve and download of run() included), so calls
// from several host threads run side by side on their own contexts, and an
// IterationObserver or FrameTransform that calls back into the engine gets
// a context of its own. Idle contexts keep their device buffers for the next
// call of the same shape.
#include <algorithm>
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

int device_of_env() {
    const char* d = std::getenv("SFSEG_DEVICE");
    return d ? std::atoi(d) : 0;
}

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

// Pool of library contexts; a Lease holds one exclusively for one call.
class Pool {
  public:
    sfseg_ctx* take() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (!idle_.empty()) {
                sfseg_ctx* c = idle_.back();  // most recently used: warm buffers
                idle_.pop_back();
                return c;
            }
        }
        sfseg_ctx* c = nullptr;
        check(sfseg_ctx_create(device_of_env(), &c));
        return c;
    }
    void give(sfseg_ctx* c) {
        std::lock_guard<std::mutex> lk(mu_);
        idle_.push_back(c);
    }

  private:
    std::mutex mu_;
    std::vector<sfseg_ctx*> idle_;  // released with the process
};

Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: callers may run at exit
    return *p;
}

// The in-process multi-GPU solver of SFSEG_NUM_GPUS > 1 (one per process;
// run() calls take turns on it).
struct Multi {
    std::mutex mu;
    sfseg_multi* m = nullptr;
};

int num_gpus_of_env() {
    const char* n = std::getenv("SFSEG_NUM_GPUS");
    return n ? std::max(1, std::atoi(n)) : 1;
}

Multi* multi() {
    static Multi* g = [] {
        auto* x = new Multi();
        const int n = num_gpus_of_env();
        if (n > 1) {
            std::vector<int32_t> dev;
            if (const char* d = std::getenv("SFSEG_MULTI_DEVICES")) {
                std::string s(d);
                size_t pos = 0;
                while (pos <= s.size() && static_cast<int>(dev.size()) < n) {
                    const size_t c = s.find(',', pos);
                    dev.push_back(std::atoi(s.substr(pos, c == std::string::npos ? std::string::npos : c - pos).c_str()));
                    if (c == std::string::npos) break;
                    pos = c + 1;
                }
            }
            while (static_cast<int>(dev.size()) < n) dev.push_back(static_cast<int32_t>(dev.size()));
            check(sfseg_multi_create(n, dev.data(), &x->m));
        }
        return x;
    }();
    return g;
}

class Lease {
  public:
    Lease() : c_(pool().take()) {}
    ~Lease() { pool().give(c_); }
    Lease(const Lease&) = delete;
    Lease& operator=(const Lease&) = delete;
    sfseg_ctx* get() const { return c_; }

  private:
    sfseg_ctx* c_;
};

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

// frames [t0, t1] (inclusive) of v as a volume of their own: the window a
// FrameTransform sees (engine.cpp:295-303)
sfseg::FeatureVolume window_of(const sfseg::FeatureVolume& v, std::uint32_t t0, std::uint32_t t1) {
    const auto& sh = v.shape();
    const std::size_t frame = static_cast<std::size_t>(sh.height) * sh.width;
    sfseg::FeatureVolume w(sfseg::VolumeShape{t1 - t0 + 1, sh.height, sh.width}, v.role());
    const float* from = v.data() + frame * t0;
    std::copy(from, from + w.size(), w.data());
    return w;
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
    Lease lease;
    check(sfseg_step_channel(lease.get(), sh.frames, sh.height, sh.width, x.data(), s.data(), f.data(),
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
    Lease lease;
    check(sfseg_step(lease.get(), sh.frames, sh.height, sh.width, static_cast<int32_t>(F.size()),
                     x.data(), features.unary.data(), F.data(), &p, out.data(), SFSEG_MEM_HOST));
    return out;
}

std::pair<FeatureVolume, double> normalize_l2(const FeatureVolume& x) {
    const auto& sh = x.shape();
    FeatureVolume out(sh, x.role());
    double norm = 0.0;
    Lease lease;
    check(sfseg_normalize_l2(lease.get(), sh.frames, sh.height, sh.width, x.data(), out.data(), &norm,
                             SFSEG_MEM_HOST));
    return {std::move(out), norm};
}

FeatureVolume project_binary(const FeatureVolume& x, int iter, const SfsegConfig& cfg) {
    if (iter < cfg.binarize_start) return x;  // engine.cpp:186
    const sfseg_params p = to_params(cfg);
    const auto& sh = x.shape();
    FeatureVolume out(sh, x.role());
    Lease lease;
    check(sfseg_project_binary(lease.get(), sh.frames, sh.height, sh.width, x.data(), iter, &p,
                               out.data(), SFSEG_MEM_HOST));
    return out;
}

BinaryMask threshold_final(const FeatureVolume& x, double frac) {
    const auto& sh = x.shape();
    BinaryMask m;
    m.shape = sh;
    m.values.resize(x.size());
    Lease lease;
    check(sfseg_threshold_final(lease.get(), sh.frames, sh.height, sh.width, x.data(), frac,
                                m.values.data(), SFSEG_MEM_HOST));
    return m;
}

namespace {

// run() with a FrameTransform (engine.cpp:284-347): the hook needs the
// reference's per-frame Jacobi windows on the host, so each frame's window
// of x, S and F goes through the hook and then through sfseg_step on the
// GPU; the frame's own plane of the result is kept. The unit-range guard of
// the pairwise channels (engine.cpp:254-259) runs on the device.
RunResult run_windowed(const FeatureSet& features, const SfsegConfig& cfg,
                       const FeatureVolume* x0, const FeatureVolume* reference,
                       const BinaryMask* ground_truth, const FrameTransform& transform,
                       const IterationObserver& observer) {
    const VolumeShape sh = features.shape();
    FeatureSet guarded_set = features;
    if (!cfg.allow_negative_affinity) {
        Lease lease;
        for (auto& f : guarded_set.pairwise)
            check(sfseg_unit_range(lease.get(), sh.frames, sh.height, sh.width, f.data(), f.data(),
                                   SFSEG_MEM_HOST));
    }
    FeatureVolume x = x0 ? *x0 : guarded_set.unary;
    x.set_role(VolumeRole::solution);
    const std::uint32_t half = static_cast<std::uint32_t>(cfg.resolved_temporal_window());
    const std::size_t frame = static_cast<std::size_t>(sh.height) * sh.width;
    RunResult r;
    for (int iter = 1; iter <= cfg.iterations; ++iter) {
        const auto started = std::chrono::steady_clock::now();
        FeatureVolume next(sh, VolumeRole::solution);
        for (std::uint32_t t = 0; t < sh.frames; ++t) {
            const std::uint32_t lo = t > half ? t - half : 0;
            const std::uint32_t hi = std::min(sh.frames - 1, t + half);
            FeatureSet win;
            win.unary = window_of(guarded_set.unary, lo, hi);
            for (const auto& f : guarded_set.pairwise) win.pairwise.push_back(window_of(f, lo, hi));
            FeatureVolume xw = window_of(x, lo, hi);
            transform(win.unary, win.pairwise, xw, t);
            const FeatureVolume y = sfseg_step(xw, win, cfg);  // GPU, S^p of the window
            const float* plane = y.data() + (t - lo) * frame;
            std::copy(plane, plane + frame, next.data() + t * frame);
        }
        auto [unit, norm] = normalize_l2(next);
        x = project_binary(unit, iter, cfg);
        IterationRecord rec;
        rec.iter = iter;
        rec.l2_norm_pre_normalize = norm;
        rec.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - started).count();
        if (reference) rec.angle_deg = angle_degrees(x, *reference);
        if (ground_truth) rec.iou = jaccard(threshold_final(x, cfg.threshold_frac), *ground_truth);
        r.trace.iterations.push_back(rec);
        if (observer) observer(iter, x);
    }
    r.mask = threshold_final(x, cfg.final_threshold);
    r.soft = std::move(x);
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

    const sfseg_params p = to_params(cfg);
    std::vector<const float*> F;
    for (const auto& f : features.pairwise) F.push_back(f.data());
    if (num_gpus_of_env() > 1 && !observer && !reference && !ground_truth) {
        // SFSEG_NUM_GPUS: time shards on the GPUs of this process
        Multi* mu = multi();
        std::lock_guard<std::mutex> lk(mu->mu);
        RunResult r;
        r.soft = FeatureVolume(shape, VolumeRole::solution);
        r.mask.shape = shape;
        r.mask.values.resize(shape.voxels());
        std::vector<sfseg_iter_record> rec(static_cast<std::size_t>(cfg.iterations));
        check(sfseg_multi_run(mu->m, shape.frames, shape.height, shape.width, static_cast<int32_t>(F.size()),
                              features.unary.data(), F.data(), x0 ? x0->data() : nullptr, &p,
                              r.soft.data(), r.mask.values.data(), rec.data(), SFSEG_MEM_HOST));
        for (const auto& e : rec) {
            IterationRecord ir;
            ir.iter = e.iter;
            ir.l2_norm_pre_normalize = e.l2_norm_pre_normalize;
            ir.wall_time_s = e.wall_time_s;
            r.trace.iterations.push_back(ir);
        }
        return r;
    }
    Lease lease;  // held for load, solve and download: the call is atomic
    sfseg_ctx* c = lease.get();
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
    Lease lease;
    check(sfseg_convolve_separable_taps(lease.get(), s.frames, s.height, s.width, v.data(), r,
                                        k.taps_t.data(), k.taps_y.data(), k.taps_x.data(),
                                        out.data(), SFSEG_MEM_HOST));
    return out;
}

FeatureVolume convolve_direct(const FeatureVolume& v, const SeparableKernel3D& k, int) {
    const auto& s = v.shape();
    s.validate();
    FeatureVolume out(s, v.role());
    const int32_t r[3] = {k.radii[0], k.radii[1], k.radii[2]};
    Lease lease;
    check(sfseg_convolve_direct_taps(lease.get(), s.frames, s.height, s.width, v.data(), r,
                                     k.taps_t.data(), k.taps_y.data(), k.taps_x.data(),
                                     out.data(), SFSEG_MEM_HOST));
    return out;
}

std::uint64_t separable_convolution_count() { return sfseg_separable_convolution_count(); }

}  // namespace sfseg
