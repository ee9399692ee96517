// Reentrancy of the drop-in (SURVEY.md §8(b) Threading): the reference's
// engine functions are pure and may be called from several host threads at
// once (their only global state is an atomic counter, conv3d.cpp:21). This
// program links the drop-in (libsfseg_engine_cuda.so) and checks, on the GPU:
//   1. four threads running sfseg::run on four different problems at once
//      get exactly the results of the same calls made one after another;
//   2. an IterationObserver that calls sfseg_step / normalize_l2 /
//      threshold_final inside run() does not disturb the run (bit-equal to a
//      run without the observer), and its own results are correct.
// Prints "dropin_threads: PASS" and exits 0, or names the failing check.
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "sfseg/engine.hpp"
#include "sfseg/rng.hpp"
#include "sfseg/volume.hpp"

namespace {

sfseg::FeatureVolume volume(const sfseg::VolumeShape& sh, std::uint64_t seed, sfseg::VolumeRole role) {
    sfseg::Xoshiro256StarStar rng(seed);
    sfseg::FeatureVolume v(sh, role);
    for (auto& x : v.values()) x = static_cast<float>(rng.next_double());
    return v;
}

sfseg::FeatureSet problem(int k) {
    const sfseg::VolumeShape sh{static_cast<std::uint32_t>(5 + k), static_cast<std::uint32_t>(40 + 7 * k),
                                static_cast<std::uint32_t>(50 + 11 * k)};
    sfseg::FeatureSet fs;
    fs.unary = volume(sh, 100 + k, sfseg::VolumeRole::unary);
    for (int c = 0; c < 1 + (k % 3); ++c)
        fs.pairwise.push_back(volume(sh, 200 + 10 * k + c, sfseg::VolumeRole::pairwise));
    return fs;
}

sfseg::SfsegConfig config(int k) {
    sfseg::SfsegConfig cfg;
    cfg.iterations = 6;
    cfg.binarize_start = 3 + (k % 2) * 10;
    cfg.kernel.radii = {1 + (k % 2), 3, 3};
    return cfg;
}

bool same(const sfseg::RunResult& a, const sfseg::RunResult& b) {
    if (a.soft.size() != b.soft.size()) return false;
    if (std::memcmp(a.soft.data(), b.soft.data(), a.soft.size() * sizeof(float)) != 0) return false;
    if (a.mask.values != b.mask.values) return false;
    if (a.trace.iterations.size() != b.trace.iterations.size()) return false;
    for (std::size_t i = 0; i < a.trace.iterations.size(); ++i)
        if (a.trace.iterations[i].l2_norm_pre_normalize != b.trace.iterations[i].l2_norm_pre_normalize)
            return false;
    return true;
}

}  // namespace

int main() {
    constexpr int kThreads = 4;
    std::vector<sfseg::FeatureSet> probs;
    for (int k = 0; k < kThreads; ++k) probs.push_back(problem(k));
    std::vector<sfseg::RunResult> serial;
    for (int k = 0; k < kThreads; ++k) serial.push_back(sfseg::run(probs[k], config(k)));

    for (int round = 0; round < 3; ++round) {
        std::vector<sfseg::RunResult> par(kThreads);
        std::vector<std::thread> th;
        for (int k = 0; k < kThreads; ++k)
            th.emplace_back([&, k] { par[k] = sfseg::run(probs[k], config(k)); });
        for (auto& t : th) t.join();
        for (int k = 0; k < kThreads; ++k)
            if (!same(par[k], serial[k])) {
                std::printf("dropin_threads: FAIL concurrent run %d (round %d) differs from serial\n", k, round);
                return 1;
            }
    }

    // an observer calling back into the engine while run() holds its context
    int bad = 0, calls = 0;
    const sfseg::FeatureSet& fs = probs[1];
    const sfseg::SfsegConfig cfg = config(1);
    auto observer = [&](int, const sfseg::FeatureVolume& x) {
        ++calls;
        const sfseg::FeatureVolume a = sfseg::sfseg_step(x, fs, cfg);
        const sfseg::FeatureVolume b = sfseg::sfseg_step(x, fs, cfg);
        if (std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) != 0) ++bad;
        auto [u, n] = sfseg::normalize_l2(a);
        if (!(n > 0.0)) ++bad;
        (void)sfseg::threshold_final(u, 0.5);
    };
    const sfseg::RunResult with_obs = sfseg::run(fs, cfg, nullptr, nullptr, nullptr, {}, observer);
    if (calls != cfg.iterations || bad) {
        std::printf("dropin_threads: FAIL observer calls=%d bad=%d\n", calls, bad);
        return 1;
    }
    if (!same(with_obs, serial[1])) {
        std::printf("dropin_threads: FAIL run with a re-entrant observer differs\n");
        return 1;
    }
    std::printf("dropin_threads: PASS (%d threads x 3 rounds, re-entrant observer)\n", kThreads);
    return 0;
}
