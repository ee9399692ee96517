// Development aid: per-call latency of the drop-in's stateless entry points on
// a tiny volume (acceptance.cpp check 5 runs normalize_l2(sfseg_step(x)) at
// 10 x 20 x 20). Build: see tools/build_small_calls.sh
#include <chrono>
#include <cstdio>

#include "sfseg/engine.hpp"
#include "sfseg/rng.hpp"
#include "sfseg/volume.hpp"

using Clock = std::chrono::steady_clock;

int main() {
    const sfseg::VolumeShape sh{10, 20, 20};
    sfseg::Xoshiro256StarStar rng(7);
    sfseg::FeatureSet fs;
    fs.unary = sfseg::FeatureVolume(sh, sfseg::VolumeRole::unary);
    for (auto& v : fs.unary.values()) v = static_cast<float>(rng.next_double());
    fs.pairwise.emplace_back(sh, sfseg::VolumeRole::pairwise);
    for (auto& v : fs.pairwise[0].values()) v = static_cast<float>(rng.next_double());
    sfseg::SfsegConfig cfg;
    sfseg::FeatureVolume x = fs.unary;
    x.set_role(sfseg::VolumeRole::solution);
    for (int w = 0; w < 20; ++w) x = sfseg::normalize_l2(sfseg::sfseg_step(x, fs, cfg)).first;
    const int n = 200;
    auto t0 = Clock::now();
    for (int k = 0; k < n; ++k) x = sfseg::normalize_l2(sfseg::sfseg_step(x, fs, cfg)).first;
    const double both = std::chrono::duration<double>(Clock::now() - t0).count() / n;
    t0 = Clock::now();
    sfseg::FeatureVolume y = x;
    for (int k = 0; k < n; ++k) y = sfseg::sfseg_step(x, fs, cfg);
    const double step = std::chrono::duration<double>(Clock::now() - t0).count() / n;
    t0 = Clock::now();
    for (int k = 0; k < n; ++k) y = sfseg::normalize_l2(x).first;
    const double norm = std::chrono::duration<double>(Clock::now() - t0).count() / n;
    std::printf("small_calls 10x20x20: step+normalize %.1f us, step %.1f us, normalize %.1f us\n",
                both * 1e6, step * 1e6, norm * 1e6);
    return 0;
}
