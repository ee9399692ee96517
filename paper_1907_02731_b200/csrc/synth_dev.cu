// synth_dev.cu — device-side synthetic problems.
//
// The host generator (synth.cpp, include/sfseg_synth.h) walks one
// xoshiro256** stream per (stream, frame) pixel by pixel, which for c4
// (1024 x 1080 x 1920, 4 fields) means ~34 GB produced on the host and then
// copied. Here every thread owns a run of CH consecutive pixels of one frame
// and jumps its generators straight to the run's first draw: xoshiro256**'s
// state update is linear over GF(2), so k steps are the 256x256 bit matrix
// A^k, applied as the product of the precomputed A^(2^i) for the set bits
// of k. From there the thread draws exactly what the host does, in the same
// order, with every double operation rounded on its own (__dmul_rn & co.:
// the host library is built without FMA), so the geometry, the clean mask,
// uniform noise, channel means and clipping are bit-identical to the host
// generator. Gaussian draws go through the device's log/cos, which are
// within one ulp of glibc's, so after the cast to float a rare value
// differs by one float ulp (tests/test_gpu_synth.py measures it).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <vector>

#include "../../include/sfseg_synth.h"

namespace {

constexpr int kCH = 1024;     // pixels per thread
constexpr int kMaxJumps = 48; // A^(2^i), i < 48: offsets up to 2^48 draws

__host__ __device__ inline uint64_t splitmix64_next(uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

struct XState {
    uint64_t s[4];
    __host__ __device__ void seed(uint64_t sd) {
        uint64_t sm = sd;
        for (int i = 0; i < 4; ++i) s[i] = splitmix64_next(sm);
    }
    // rng.hpp:20-75 / synth.cpp Xoshiro::next_u64
    __host__ __device__ uint64_t next() {
        const uint64_t result = rotl64(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl64(s[3], 45);
        return result;
    }
};

// synth.cpp derive_seed: an independent generator per (seed, stream, frame)
__host__ __device__ inline uint64_t derive_seed(uint64_t seed, uint64_t stream, uint64_t frame) {
    uint64_t s = seed ^ (0xd1b54a32d192ed03ULL * (stream + 1));
    const uint64_t a = splitmix64_next(s);
    s = a ^ (0x8cb92ba72f3d8dd7ULL * (frame + 1));
    return splitmix64_next(s);
}

__device__ __forceinline__ double next_double(XState& r) {
    return static_cast<double>(r.next() >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double next_gaussian(XState& r) {
    double u1 = next_double(r);
    const double u2 = next_double(r);
    if (u1 == 0.0) u1 = 0x1.0p-53;
    const double rr = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    return __dmul_rn(rr, cos(__dmul_rn(2.0 * 3.14159265358979323846, u2)));
}

struct Ellipse {
    double cy, cx, vy, vx, ay, ax, value;
};

struct SynthArgs {
    Ellipse obj[8];
    int objects;
    uint32_t T, H, W;
    int channels;
    double outside;
    int noise;
    double noise_level;
    int mode;
    double fsigma;
    uint64_t seed;
    float inv_channels;
    const ulonglong4* jumps;  // [kMaxJumps][256] columns of A^(2^i)
    float* S;
    float* F[16];
    uint8_t* mask;
};

// r = A^(2^i) s, one masked XOR of a column per state bit
__device__ void jump_apply(XState& st, const ulonglong4* __restrict__ cols) {
    uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        const uint64_t word = st.s[w];
#pragma unroll 8
        for (int b = 0; b < 64; ++b) {
            const uint64_t m = 0ULL - ((word >> b) & 1ULL);
            const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(cols + w * 64 + b);
            const ulonglong2 lo = __ldg(c2), hi = __ldg(c2 + 1);
            r0 ^= lo.x & m;
            r1 ^= lo.y & m;
            r2 ^= hi.x & m;
            r3 ^= hi.y & m;
        }
    }
    st.s[0] = r0;
    st.s[1] = r1;
    st.s[2] = r2;
    st.s[3] = r3;
}

__device__ XState stream_at(const SynthArgs& a, uint64_t stream, uint32_t t, uint64_t draw) {
    XState st;
    st.seed(derive_seed(a.seed, stream, t));
    for (int i = 0; draw; ++i, draw >>= 1)
        if (draw & 1ULL) jump_apply(st, a.jumps + static_cast<size_t>(i) * 256);
    return st;
}

// synth.cpp reflect (triangle wave), each operation rounded on its own
__device__ double reflect_d(double v, double lo, double hi) {
    if (hi <= lo) return lo;
    const double span = __dsub_rn(hi, lo);
    const double two = __dmul_rn(2.0, span);
    double u = fmod(__dsub_rn(v, lo), two);
    if (u < 0) u = __dadd_rn(u, two);
    return __dadd_rn(lo, u <= span ? u : __dsub_rn(two, u));
}

struct FrameObj {
    double cy, cx, ay, ax, value;
    int y0, y1, x0, x1;
};

__device__ FrameObj frame_obj(const SynthArgs& a, int k, uint32_t t) {
    const Ellipse& e = a.obj[k];
    FrameObj f;
    const double td = static_cast<double>(t);
    f.cy = reflect_d(__dadd_rn(e.cy, __dmul_rn(e.vy, td)), 0.0, __dsub_rn(static_cast<double>(a.H), 1.0));
    f.cx = reflect_d(__dadd_rn(e.cx, __dmul_rn(e.vx, td)), 0.0, __dsub_rn(static_cast<double>(a.W), 1.0));
    f.ay = e.ay;
    f.ax = e.ax;
    f.value = e.value;
    f.y0 = max(0, static_cast<int>(floor(__dsub_rn(f.cy, e.ay))));
    f.y1 = min(static_cast<int>(a.H) - 1, static_cast<int>(ceil(__dadd_rn(f.cy, e.ay))));
    f.x0 = max(0, static_cast<int>(floor(__dsub_rn(f.cx, e.ax))));
    f.x1 = min(static_cast<int>(a.W) - 1, static_cast<int>(ceil(__dadd_rn(f.cx, e.ax))));
    return f;
}

// base value (max over the objects covering the pixel) and the indicator
__device__ __forceinline__ double base_at(const FrameObj* fo, int nobj, double outside, int y, int x,
                                          bool& inside) {
    double b = outside;
    inside = false;
    for (int k = 0; k < nobj; ++k) {
        const FrameObj& f = fo[k];
        if (y < f.y0 || y > f.y1 || x < f.x0 || x > f.x1) continue;
        const double dy = __ddiv_rn(__dsub_rn(static_cast<double>(y), f.cy), f.ay);
        const double dx = __ddiv_rn(__dsub_rn(static_cast<double>(x), f.cx), f.ax);
        if (__dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dx, dx)) <= 1.0) {
            b = fmax(b, f.value);
            inside = true;
        }
    }
    return b;
}

__device__ __forceinline__ float clip01(double v) {
    return __double2float_rn(fmin(fmax(v, 0.0), 1.0));
}

// adds the stream's noise to v (synth.cpp noisy())
__device__ __forceinline__ double add_noise(XState& r, int kind, double level, double v) {
    if (kind == SFSEG_NOISE_UNIFORM)
        return __dadd_rn(v, __dmul_rn(level, __dsub_rn(__dmul_rn(2.0, next_double(r)), 1.0)));
    if (kind == SFSEG_NOISE_GAUSSIAN) return __dadd_rn(v, __dmul_rn(level, next_gaussian(r)));
    return v;
}

__host__ __device__ inline int draws_per_pixel(int kind) {
    return kind == SFSEG_NOISE_UNIFORM ? 1 : (kind == SFSEG_NOISE_GAUSSIAN ? 2 : 0);
}

__global__ void __launch_bounds__(128) k_synth(const SynthArgs a) {
    const uint64_t plane = static_cast<uint64_t>(a.H) * a.W;
    const uint64_t chunks = (plane + kCH - 1) / kCH;
    const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= chunks * a.T) return;
    const uint32_t t = static_cast<uint32_t>(gid / chunks);
    const uint64_t p0 = (gid % chunks) * kCH;
    const int n = static_cast<int>(plane - p0 < kCH ? plane - p0 : kCH);
    const size_t off = static_cast<size_t>(t) * plane + p0;

    FrameObj fo[8];
    for (int k = 0; k < a.objects; ++k) fo[k] = frame_obj(a, k, t);
    // visits the run's pixels in order with their (y, x)
    auto walk = [&](auto&& f) {
        int y = static_cast<int>(p0 / a.W), x = static_cast<int>(p0 % a.W);
        for (int i = 0; i < n; ++i) {
            bool in;
            f(i, base_at(fo, a.objects, a.outside, y, x, in), in);
            if (++x == static_cast<int>(a.W)) {
                x = 0;
                ++y;
            }
        }
    };

    if (a.mask) walk([&](int i, double, bool in) { a.mask[off + i] = in ? 1 : 0; });

    constexpr int gdraw = 2;  // a gaussian draw takes two doubles
    if (a.mode == SFSEG_FEAT_MEAN_OF_F) {
        // F_c = clip(base + N(0, fsigma)) from stream 1+c; S = (sum_c F_c, in
        // channel order, fp32) * (1/C)
        for (int c = 0; c < a.channels; ++c) {
            XState r = stream_at(a, 1 + c, t, p0 * gdraw);
            float* fo_c = a.F[c] + off;
            walk([&](int i, double b, bool) {
                const float f = clip01(add_noise(r, SFSEG_NOISE_GAUSSIAN, a.fsigma, b));
                fo_c[i] = f;
                a.S[off + i] = c == 0 ? f : __fadd_rn(a.S[off + i], f);
            });
        }
        for (int i = 0; i < n; ++i) a.S[off + i] = __fmul_rn(a.S[off + i], a.inv_channels);
        return;
    }
    {
        XState r = stream_at(a, 0, t, p0 * draws_per_pixel(a.noise));
        walk([&](int i, double b, bool) {
            const float s = clip01(add_noise(r, a.noise, a.noise_level, b));
            a.S[off + i] = s;
            if (a.mode == SFSEG_FEAT_SAME)
                for (int c = 0; c < a.channels; ++c) a.F[c][off + i] = s;
        });
    }
    if (a.mode == SFSEG_FEAT_NOISY_F) {
        for (int c = 0; c < a.channels; ++c) {
            XState r = stream_at(a, 1 + c, t, p0 * gdraw);
            float* fo_c = a.F[c] + off;
            for (int i = 0; i < n; ++i)
                fo_c[i] = clip01(add_noise(r, SFSEG_NOISE_GAUSSIAN, a.fsigma,
                                           static_cast<double>(a.S[off + i])));
        }
    }
}

// Host: object parameters (synth.cpp, stream 1000) and the jump matrices.
double host_next_double(XState& r) { return static_cast<double>(r.next() >> 11) * 0x1.0p-53; }

// columns of A (one xoshiro step applied to each unit state), squared up
const std::vector<ulonglong4>& jump_table() {
    static std::vector<ulonglong4> tab;
    if (!tab.empty()) return tab;
    tab.resize(static_cast<size_t>(kMaxJumps) * 256);
    auto apply = [](const ulonglong4* cols, const uint64_t s[4], uint64_t r[4]) {
        r[0] = r[1] = r[2] = r[3] = 0;
        for (int j = 0; j < 256; ++j)
            if ((s[j >> 6] >> (j & 63)) & 1ULL) {
                r[0] ^= cols[j].x;
                r[1] ^= cols[j].y;
                r[2] ^= cols[j].z;
                r[3] ^= cols[j].w;
            }
    };
    for (int j = 0; j < 256; ++j) {
        XState st;
        st.s[0] = st.s[1] = st.s[2] = st.s[3] = 0;
        st.s[j >> 6] = 1ULL << (j & 63);
        st.next();
        tab[j] = make_ulonglong4(st.s[0], st.s[1], st.s[2], st.s[3]);
    }
    for (int i = 1; i < kMaxJumps; ++i) {
        const ulonglong4* prev = &tab[static_cast<size_t>(i - 1) * 256];
        ulonglong4* cur = &tab[static_cast<size_t>(i) * 256];
        for (int j = 0; j < 256; ++j) {  // column j of P^2 = P (column j of P)
            const uint64_t s[4] = {prev[j].x, prev[j].y, prev[j].z, prev[j].w};
            uint64_t r[4];
            apply(prev, s, r);
            cur[j] = make_ulonglong4(r[0], r[1], r[2], r[3]);
        }
    }
    return tab;
}

}  // namespace

extern "C" {

int sfseg_synth_generate_device(const sfseg_synth_spec* sp, float* S, float* const* F,
                                uint8_t* mask_out, void* stream) {
    if (!sp || !S || sp->frames == 0 || sp->height == 0 || sp->width == 0) return -1;
    if (sp->objects < 1 || sp->objects > 8 || sp->channels < 1 || sp->channels > 16 || !F) return -1;
    const sfseg_synth_spec& spec = *sp;
    const uint32_t H = spec.height, W = spec.width;
    const uint64_t plane = static_cast<uint64_t>(H) * W;
    if (plane * 2 >= (1ULL << kMaxJumps)) return -1;

    SynthArgs a{};
    XState prng;
    prng.seed(derive_seed(spec.seed, 1000, 0));
    for (int k = 0; k < spec.objects; ++k) {  // synth.cpp object loop, same draw order
        Ellipse& e = a.obj[k];
        if (spec.area_frac > 0.0) {
            const double aspect = 0.6 + 0.4 * host_next_double(prng);
            const double area = spec.area_frac * static_cast<double>(H) * W;
            const double b = std::sqrt(area / (3.14159265358979323846 * aspect));
            e.ay = b * aspect;
            e.ax = b;
        } else {
            e.ay = spec.semi_min + (spec.semi_max - spec.semi_min) * host_next_double(prng);
            e.ax = spec.semi_min + (spec.semi_max - spec.semi_min) * host_next_double(prng);
        }
        e.cy = H * (0.25 + 0.5 * host_next_double(prng));
        e.cx = W * (0.25 + 0.5 * host_next_double(prng));
        const double speed = spec.speed_min + (spec.speed_max - spec.speed_min) * host_next_double(prng);
        const double ang = 2.0 * 3.14159265358979323846 * host_next_double(prng);
        e.vy = speed * std::sin(ang);
        e.vx = speed * std::cos(ang);
        e.value = spec.inside[k];
    }
    a.objects = spec.objects;
    a.T = spec.frames;
    a.H = H;
    a.W = W;
    a.channels = spec.channels;
    a.outside = spec.outside;
    a.noise = spec.noise;
    a.noise_level = spec.noise_level;
    a.mode = spec.feature_mode;
    a.fsigma = spec.feature_sigma;
    a.seed = spec.seed;
    a.inv_channels = 1.0f / static_cast<float>(spec.channels);
    a.S = S;
    for (int c = 0; c < spec.channels; ++c) {
        if (!F[c]) return -1;
        a.F[c] = F[c];
    }
    a.mask = mask_out;

    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const std::vector<ulonglong4>& tab = jump_table();
    ulonglong4* d_tab = nullptr;
    const size_t tab_bytes = tab.size() * sizeof(ulonglong4);
    if (cudaMallocAsync(reinterpret_cast<void**>(&d_tab), tab_bytes, st) != cudaSuccess) return -2;
    if (cudaMemcpyAsync(d_tab, tab.data(), tab_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return -2;
    a.jumps = d_tab;
    const uint64_t threads = ((plane + kCH - 1) / kCH) * spec.frames;
    const unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
    k_synth<<<blocks, 128, 0, st>>>(a);
    const cudaError_t le = cudaGetLastError();
    cudaFreeAsync(d_tab, st);
    // the host table is read by the async copy: keep it until the copy is done
    if (cudaStreamSynchronize(st) != cudaSuccess || le != cudaSuccess) return -2;
    return 0;
}

}  // extern "C"
