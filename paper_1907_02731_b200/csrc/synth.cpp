// synth.cpp — seeded moving-ellipse problems for the SFSeg benchmarks and
// parity tests (see include/sfseg_synth.h). Host code: it produces inputs, it
// is not part of the GPU hot path.
#include "../../include/sfseg_synth.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// splitmix64 / xoshiro256** / Box–Muller as in the reference (rng.hpp:20-75)
uint64_t splitmix64_next(uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Xoshiro {
public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t sm = seed;
        for (auto& w : s_) w = splitmix64_next(sm);
    }
    uint64_t next_u64() {
        const uint64_t result = rotl(s_[1] * 5, 7) * 9;
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return result;
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_gaussian() {
        double u1 = next_double();
        const double u2 = next_double();
        if (u1 == 0.0) u1 = 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        return r * std::cos(2.0 * 3.14159265358979323846 * u2);
    }

private:
    static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    uint64_t s_[4]{};
};

// independent generator per (seed, stream, frame)
uint64_t derive_seed(uint64_t seed, uint64_t stream, uint64_t frame) {
    uint64_t s = seed ^ (0xd1b54a32d192ed03ULL * (stream + 1));
    uint64_t a = splitmix64_next(s);
    s = a ^ (0x8cb92ba72f3d8dd7ULL * (frame + 1));
    return splitmix64_next(s);
}

struct Ellipse {
    double cy, cx, vy, vx, ay, ax, value;
};

// triangle-wave reflection keeps the centre inside [lo, hi]
double reflect(double v, double lo, double hi) {
    if (hi <= lo) return lo;
    const double span = hi - lo;
    double u = std::fmod(v - lo, 2.0 * span);
    if (u < 0) u += 2.0 * span;
    return lo + (u <= span ? u : 2.0 * span - u);
}

float clip01(double v) { return static_cast<float>(std::clamp(v, 0.0, 1.0)); }

}  // namespace

extern "C" {

int sfseg_synth_generate(const sfseg_synth_spec* sp, float* S, float* const* F, uint8_t* mask_out,
                         int threads) {
    if (!sp) return -1;
    return sfseg_synth_generate_frames(sp, 0, sp->frames, S, F, mask_out, threads);
}

int sfseg_synth_generate_frames(const sfseg_synth_spec* sp, uint32_t t0, uint32_t t1, float* S,
                                float* const* F, uint8_t* mask_out, int threads) {
    if (!sp || !S || sp->frames == 0 || sp->height == 0 || sp->width == 0) return -1;
    if (t0 >= t1 || t1 > sp->frames) return -1;
    if (sp->objects < 1 || sp->objects > 8 || sp->channels < 1) return -1;
    if (sp->channels > 0 && !F) return -1;
    const sfseg_synth_spec spec = *sp;
    const uint32_t H = spec.height, W = spec.width;
    const size_t plane = static_cast<size_t>(H) * W;

    // object parameters from stream 1000
    std::vector<Ellipse> obj(spec.objects);
    Xoshiro prng(derive_seed(spec.seed, 1000, 0));
    for (int k = 0; k < spec.objects; ++k) {
        Ellipse& e = obj[k];
        if (spec.area_frac > 0.0) {
            const double aspect = 0.6 + 0.4 * prng.next_double();
            const double area = spec.area_frac * static_cast<double>(H) * W;
            const double b = std::sqrt(area / (3.14159265358979323846 * aspect));
            e.ay = b * aspect;
            e.ax = b;
        } else {
            e.ay = spec.semi_min + (spec.semi_max - spec.semi_min) * prng.next_double();
            e.ax = spec.semi_min + (spec.semi_max - spec.semi_min) * prng.next_double();
        }
        e.cy = H * (0.25 + 0.5 * prng.next_double());
        e.cx = W * (0.25 + 0.5 * prng.next_double());
        const double speed = spec.speed_min + (spec.speed_max - spec.speed_min) * prng.next_double();
        const double ang = 2.0 * 3.14159265358979323846 * prng.next_double();
        e.vy = speed * std::sin(ang);
        e.vx = speed * std::cos(ang);
        e.value = spec.inside[k];
    }

    auto frame_job = [&](uint32_t t) {
        std::vector<double> base(plane);
        std::vector<uint8_t> ind(plane);
        for (size_t i = 0; i < plane; ++i) {
            base[i] = spec.outside;
            ind[i] = 0;
        }
        for (const Ellipse& e : obj) {
            const double cy = reflect(e.cy + e.vy * t, 0.0, H - 1.0);
            const double cx = reflect(e.cx + e.vx * t, 0.0, W - 1.0);
            const int y0 = std::max(0, static_cast<int>(std::floor(cy - e.ay)));
            const int y1 = std::min<int>(H - 1, static_cast<int>(std::ceil(cy + e.ay)));
            const int x0 = std::max(0, static_cast<int>(std::floor(cx - e.ax)));
            const int x1 = std::min<int>(W - 1, static_cast<int>(std::ceil(cx + e.ax)));
            for (int y = y0; y <= y1; ++y)
                for (int x = x0; x <= x1; ++x) {
                    const double dy = (y - cy) / e.ay, dx = (x - cx) / e.ax;
                    if (dy * dy + dx * dx <= 1.0) {
                        const size_t i = static_cast<size_t>(y) * W + x;
                        base[i] = std::max(base[i], e.value);
                        ind[i] = 1;
                    }
                }
        }
        const size_t off = static_cast<size_t>(t - t0) * plane;  // buffers hold frames [t0, t1)
        if (mask_out) std::memcpy(mask_out + off, ind.data(), plane);
        auto noisy = [&](uint64_t stream, int kind, double level, const double* src, float* dst) {
            Xoshiro r(derive_seed(spec.seed, stream, t));
            for (size_t i = 0; i < plane; ++i) {
                double v = src[i];
                if (kind == SFSEG_NOISE_UNIFORM)
                    v += level * (2.0 * r.next_double() - 1.0);
                else if (kind == SFSEG_NOISE_GAUSSIAN)
                    v += level * r.next_gaussian();
                dst[i] = clip01(v);
            }
        };
        float* s_out = S + off;
        if (spec.feature_mode == SFSEG_FEAT_MEAN_OF_F) {
            std::vector<float> acc(plane, 0.0f);
            for (int c = 0; c < spec.channels; ++c) {
                float* fo = F[c] + off;
                noisy(1 + c, SFSEG_NOISE_GAUSSIAN, spec.feature_sigma, base.data(), fo);
                for (size_t i = 0; i < plane; ++i) acc[i] += fo[i];
            }
            const float inv = 1.0f / static_cast<float>(spec.channels);
            for (size_t i = 0; i < plane; ++i) s_out[i] = acc[i] * inv;
        } else {
            noisy(0, spec.noise, spec.noise_level, base.data(), s_out);
            if (spec.feature_mode == SFSEG_FEAT_SAME) {
                for (int c = 0; c < spec.channels; ++c)
                    std::memcpy(F[c] + off, s_out, plane * sizeof(float));
            } else {
                std::vector<double> sd(plane);
                for (size_t i = 0; i < plane; ++i) sd[i] = s_out[i];
                for (int c = 0; c < spec.channels; ++c)
                    noisy(1 + c, SFSEG_NOISE_GAUSSIAN, spec.feature_sigma, sd.data(), F[c] + off);
            }
        }
    };

    int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    nt = std::max(1, std::min<int>(nt, static_cast<int>(t1 - t0)));
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
        pool.emplace_back([&, w] {
            for (uint32_t t = t0 + w; t < t1; t += nt) frame_job(t);
        });
    for (auto& th : pool) th.join();
    return 0;
}

void sfseg_synth_xoshiro_u64(uint64_t seed, uint64_t* out, size_t n) {
    Xoshiro r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void sfseg_synth_xoshiro_gaussian(uint64_t seed, double* out, size_t n) {
    Xoshiro r(seed);
    for (size_t i = 0; i < n; ++i) out[i] = r.next_gaussian();
}

}  // extern "C"
