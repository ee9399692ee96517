// ref_capi.cpp — TEST INFRASTRUCTURE ONLY. A C-callable wrapper around the
// reference library compiled unchanged from /root/reference/proj/src with
// -Dsfseg=sfseg_ref (oracle/Makefile). It lets the Python tests and bench.py's
// CPU legs drive the real reference (sfseg_ref::run, sfseg_step, ...) through
// ctypes. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load the resulting oracle/_ref/libsfseg_ref.so.
//
// No reference source is copied here: this file only calls the reference's
// public API (proj/include/sfseg/*.hpp).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "sfseg/conv3d.hpp"
#include "sfseg/engine.hpp"
#include "sfseg/errors.hpp"
#include "sfseg/metrics.hpp"
#include "sfseg/oracle.hpp"
#include "sfseg/rng.hpp"
#include "sfseg/volume.hpp"

#include "../include/sfseg_cuda.h"

namespace {

thread_local char g_msg[512];

int fail(const std::exception& e, int code) {
    std::snprintf(g_msg, sizeof g_msg, "%s", e.what());
    return code;
}

#define REF_TRY try {
#define REF_CATCH                                                                  \
    }                                                                              \
    catch (const sfseg::ParameterError& e) { return fail(e, SFSEG_ERR_PARAMETER); } \
    catch (const sfseg::ShapeError& e) { return fail(e, SFSEG_ERR_SHAPE); }         \
    catch (const sfseg::ValidationError& e) { return fail(e, SFSEG_ERR_VALIDATION); } \
    catch (const sfseg::DegenerateSolutionError& e) { return fail(e, SFSEG_ERR_DEGENERATE); } \
    catch (const sfseg::IoError& e) { return fail(e, SFSEG_ERR_IO); }               \
    catch (const sfseg::FormatError& e) { return fail(e, SFSEG_ERR_FORMAT); }       \
    catch (const sfseg::CorruptionError& e) { return fail(e, SFSEG_ERR_CORRUPTION); } \
    catch (const sfseg::CapacityError& e) { return fail(e, SFSEG_ERR_CAPACITY); }   \
    catch (const std::exception& e) { return fail(e, SFSEG_ERR_STATE); }

sfseg::SfsegConfig to_cfg(const sfseg_params* p, int threads) {
    sfseg::SfsegConfig c;
    c.alpha = p->alpha;
    c.p = p->p;
    for (int a = 0; a < 3; ++a) {
        c.kernel.radii[a] = p->radii[a];
        c.kernel.sigmas[a] = p->sigmas[a];
    }
    c.iterations = p->iterations;
    c.temporal_window = p->temporal_window;
    c.binarize_start = p->binarize_start;
    c.sigmoid_slope0 = p->sigmoid_slope0;
    c.slope_growth = p->slope_growth;
    c.threshold_frac = p->threshold_frac;
    c.final_threshold = p->final_threshold;
    c.allow_negative_affinity = p->allow_negative_affinity != 0;
    c.threads = threads;
    return c;
}

sfseg::FeatureVolume vol(uint32_t T, uint32_t H, uint32_t W, const float* d,
                         sfseg::VolumeRole role) {
    const sfseg::VolumeShape s{T, H, W};
    return sfseg::FeatureVolume::from_data(s, std::vector<float>(d, d + s.voxels()), role);
}

sfseg::FeatureSet features(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                           const float* const* F) {
    sfseg::FeatureSet fs;
    fs.unary = vol(T, H, W, S, sfseg::VolumeRole::unary);
    for (int32_t c = 0; c < C; ++c)
        fs.pairwise.push_back(vol(T, H, W, F[c], sfseg::VolumeRole::pairwise));
    return fs;
}

}  // namespace

extern "C" {

const char* sfref_last_error(void) { return g_msg; }

// explicit-matrix oracle (oracle.cpp:67-258): pins sfseg_affinity_*
namespace {
sfseg::SparseAffinity ref_affinity(int32_t kind, const sfseg::FeatureSet& fs, const sfseg::SfsegConfig& c) {
    if (kind == 0) return sfseg::build_affinity_exact(fs, c);
    if (kind == 1) return sfseg::build_affinity_taylor(fs, c);
    return sfseg::build_affinity_taylor_channel_sum(fs, c);
}
}  // namespace

int sfref_affinity_matvec(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                          const float* const* F, const sfseg_params* p, int32_t kind, const double* x,
                          double* y) {
    REF_TRY
    const auto m = ref_affinity(kind, features(T, H, W, C, S, F), to_cfg(p, 1));
    const std::vector<double> r = sfseg::matvec(m, std::span<const double>(x, m.size()), 1);
    std::memcpy(y, r.data(), r.size() * sizeof(double));
    return 0;
    REF_CATCH
}

int sfref_power_iteration(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                          const float* const* F, const sfseg_params* p, int32_t kind, const double* x0,
                          int32_t max_iters, double tol, double* vec, double* value, int32_t* used) {
    REF_TRY
    const auto m = ref_affinity(kind, features(T, H, W, C, S, F), to_cfg(p, 1));
    const auto r = sfseg::power_iteration(m, std::vector<double>(x0, x0 + m.size()), max_iters, tol, 1);
    std::memcpy(vec, r.eigenvector.data(), r.eigenvector.size() * sizeof(double));
    *value = r.eigenvalue;
    *used = r.iterations_used;
    return 0;
    REF_CATCH
}

// SFSV containers through the reference's own writer / reader
// (volume.cpp:117-184): fixtures and error-code parity for sfseg_load_files
int sfref_save_volume(const char* path, uint32_t T, uint32_t H, uint32_t W, const float* d) {
    REF_TRY
    sfseg::save_volume(vol(T, H, W, d, sfseg::VolumeRole::generic), path);
    return 0;
    REF_CATCH
}

int sfref_load_volume(const char* path, uint32_t* dims, float* out, size_t cap) {
    REF_TRY
    const sfseg::FeatureVolume v = sfseg::load_volume(path);
    dims[0] = v.shape().frames;
    dims[1] = v.shape().height;
    dims[2] = v.shape().width;
    if (out && cap >= v.size()) std::memcpy(out, v.data(), v.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_validate(const sfseg_params* p) {
    REF_TRY
    to_cfg(p, 1).validate();
    return 0;
    REF_CATCH
}

int sfref_make_kernel(const int32_t radii[3], const double sigmas[3], double* tt, double* ty,
                      double* tx) {
    REF_TRY
    const auto k = sfseg::make_gaussian_kernel({sigmas[0], sigmas[1], sigmas[2]},
                                               {radii[0], radii[1], radii[2]});
    std::memcpy(tt, k.taps_t.data(), k.taps_t.size() * sizeof(double));
    std::memcpy(ty, k.taps_y.data(), k.taps_y.size() * sizeof(double));
    std::memcpy(tx, k.taps_x.data(), k.taps_x.size() * sizeof(double));
    return 0;
    REF_CATCH
}

int sfref_convolve_separable(uint32_t T, uint32_t H, uint32_t W, const float* v,
                             const int32_t radii[3], const double sigmas[3], int threads,
                             float* out) {
    REF_TRY
    const auto k = sfseg::make_gaussian_kernel({sigmas[0], sigmas[1], sigmas[2]},
                                               {radii[0], radii[1], radii[2]});
    const auto r = sfseg::convolve_separable(vol(T, H, W, v, sfseg::VolumeRole::generic), k,
                                             threads);
    std::memcpy(out, r.data(), r.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_convolve_direct(uint32_t T, uint32_t H, uint32_t W, const float* v,
                          const int32_t radii[3], const double sigmas[3], float* out) {
    REF_TRY
    const auto k = sfseg::make_gaussian_kernel({sigmas[0], sigmas[1], sigmas[2]},
                                               {radii[0], radii[1], radii[2]});
    const auto r = sfseg::convolve_direct(vol(T, H, W, v, sfseg::VolumeRole::generic), k);
    std::memcpy(out, r.data(), r.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_step(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* x, const float* S,
               const float* const* F, const sfseg_params* p, int threads, float* out) {
    REF_TRY
    const auto fs = features(T, H, W, C, S, F);
    const auto r = sfseg::sfseg_step(vol(T, H, W, x, sfseg::VolumeRole::solution), fs,
                                     to_cfg(p, threads));
    std::memcpy(out, r.data(), r.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_step_channel(uint32_t T, uint32_t H, uint32_t W, const float* x, const float* S,
                       const float* f, const sfseg_params* p, int threads, float* out) {
    REF_TRY
    const auto r = sfseg::sfseg_step_channel(vol(T, H, W, x, sfseg::VolumeRole::solution),
                                             vol(T, H, W, S, sfseg::VolumeRole::unary),
                                             vol(T, H, W, f, sfseg::VolumeRole::pairwise),
                                             to_cfg(p, threads));
    std::memcpy(out, r.data(), r.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_normalize_l2(uint32_t T, uint32_t H, uint32_t W, const float* x, float* out,
                       double* norm) {
    REF_TRY
    auto [u, n] = sfseg::normalize_l2(vol(T, H, W, x, sfseg::VolumeRole::generic));
    std::memcpy(out, u.data(), u.size() * sizeof(float));
    *norm = n;
    return 0;
    REF_CATCH
}

int sfref_project_binary(uint32_t T, uint32_t H, uint32_t W, const float* x, int32_t iter,
                         const sfseg_params* p, float* out) {
    REF_TRY
    const auto r = sfseg::project_binary(vol(T, H, W, x, sfseg::VolumeRole::generic), iter,
                                         to_cfg(p, 1));
    std::memcpy(out, r.data(), r.size() * sizeof(float));
    return 0;
    REF_CATCH
}

int sfref_threshold_final(uint32_t T, uint32_t H, uint32_t W, const float* x, double frac,
                          uint8_t* mask) {
    REF_TRY
    const auto m = sfseg::threshold_final(vol(T, H, W, x, sfseg::VolumeRole::generic), frac);
    std::memcpy(mask, m.values.data(), m.values.size());
    return 0;
    REF_CATCH
}

// sfseg::run with an observer that snapshots the iterate at the requested
// checkpoints (ascending). norms gets l2_norm_pre_normalize per iteration.
int sfref_run(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
              const float* const* F, const float* x0, const sfseg_params* p, int threads,
              float* soft, uint8_t* mask, double* norms, const int32_t* checkpoints,
              int32_t nck, float* ck_out) {
    REF_TRY
    const auto fs = features(T, H, W, C, S, F);
    sfseg::FeatureVolume x0v;
    if (x0) x0v = vol(T, H, W, x0, sfseg::VolumeRole::solution);
    const std::size_t n = static_cast<std::size_t>(T) * H * W;
    int32_t ck = 0;
    sfseg::IterationObserver obs;
    if (checkpoints && nck > 0)
        obs = [&](int iter, const sfseg::FeatureVolume& x) {
            if (ck < nck && checkpoints[ck] == iter) {
                std::memcpy(ck_out + static_cast<std::size_t>(ck) * n, x.data(),
                            n * sizeof(float));
                ++ck;
            }
        };
    const auto res = sfseg::run(fs, to_cfg(p, threads), x0 ? &x0v : nullptr, nullptr,
                                nullptr, {}, obs);
    if (soft) std::memcpy(soft, res.soft.data(), n * sizeof(float));
    if (mask) std::memcpy(mask, res.mask.values.data(), n);
    if (norms)
        for (std::size_t i = 0; i < res.trace.iterations.size(); ++i)
            norms[i] = res.trace.iterations[i].l2_norm_pre_normalize;
    return 0;
    REF_CATCH
}

// The bench "conv" loop (bench.cpp:154-155): x <- normalize_l2(sfseg_step(x)),
// starting from S, for `iterations` steps. Output: the final unit iterate.
int sfref_global_loop(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                      const float* const* F, const sfseg_params* p, int threads,
                      int32_t iterations, float* out) {
    REF_TRY
    const auto fs = features(T, H, W, C, S, F);
    const auto cfg = to_cfg(p, threads);
    sfseg::FeatureVolume x = fs.unary;
    x.set_role(sfseg::VolumeRole::solution);
    for (int32_t k = 0; k < iterations; ++k) x = sfseg::normalize_l2(sfseg::sfseg_step(x, fs, cfg)).first;
    std::memcpy(out, x.data(), x.size() * sizeof(float));
    return 0;
    REF_CATCH
}

// the same loop, with snapshots of the normalised iterate after each listed
// iteration (ascending, 1-based) and the pre-normalisation norms
int sfref_global_loop_ck(uint32_t T, uint32_t H, uint32_t W, int32_t C, const float* S,
                         const float* const* F, const sfseg_params* p, int threads,
                         int32_t iterations, float* out, const int32_t* ck, int32_t nck,
                         float* ck_out, double* norms) {
    REF_TRY
    const auto fs = features(T, H, W, C, S, F);
    const auto cfg = to_cfg(p, threads);
    sfseg::FeatureVolume x = fs.unary;
    x.set_role(sfseg::VolumeRole::solution);
    int32_t j = 0;
    for (int32_t k = 1; k <= iterations; ++k) {
        auto r = sfseg::normalize_l2(sfseg::sfseg_step(x, fs, cfg));
        x = std::move(r.first);
        if (norms) norms[k - 1] = r.second;
        if (j < nck && ck[j] == k) {
            std::memcpy(ck_out + static_cast<std::size_t>(j) * x.size(), x.data(), x.size() * sizeof(float));
            ++j;
        }
    }
    std::memcpy(out, x.data(), x.size() * sizeof(float));
    return 0;
    REF_CATCH
}

void sfref_xoshiro_u64(uint64_t seed, uint64_t* out, std::size_t n) {
    sfseg::Xoshiro256StarStar rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

void sfref_xoshiro_gaussian(uint64_t seed, double* out, std::size_t n) {
    sfseg::Xoshiro256StarStar rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_gaussian();
}

}  // extern "C"
