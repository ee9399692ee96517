/*
 * sfseg_synth.h — seeded synthetic SFSeg problems (host side, C ABI).
 *
 * The reference's generator (proj/src/synth.cpp:55-103) only draws boxes and
 * balls with flip/gaussian noise; BASELINE.json's configurations need moving
 * ellipses, soft masks, uniform noise and multi-channel features, so this is
 * a new generator. It keeps the reference's RNG (xoshiro256** seeded through
 * splitmix64, Box–Muller with exactly two draws, rng.hpp:20-75) but gives
 * every (stream, frame) pair its own generator so frames can be generated in
 * parallel with a result independent of the thread count.
 *
 * Streams: 0 = noise on S, 1 + c = feature channel c, 1000 = object params.
 */
#ifndef SFSEG_SYNTH_H
#define SFSEG_SYNTH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sfseg_noise { SFSEG_NOISE_NONE = 0, SFSEG_NOISE_UNIFORM = 1, SFSEG_NOISE_GAUSSIAN = 2 };

/* How S (unary, also the initial iterate) and the features F_c relate:
 *  SAME:        S = clip(mask + noise), F_0 = S (one channel)
 *  MEAN_OF_F:   F_c = clip(mask + N(0, feature_sigma)), S = mean_c F_c
 *  NOISY_F:     S = clip(mask + noise), F_c = clip(S + N(0, feature_sigma)) */
enum sfseg_feature_mode { SFSEG_FEAT_SAME = 0, SFSEG_FEAT_MEAN_OF_F = 1, SFSEG_FEAT_NOISY_F = 2 };

typedef struct sfseg_synth_spec {
    uint32_t frames, height, width;
    int32_t channels;
    int32_t objects;          /* number of moving ellipses (1..8) */
    double semi_min, semi_max; /* semi-axis range in pixels (used when area_frac <= 0) */
    double area_frac;         /* if > 0: semi-axes chosen so each ellipse covers this
                                 fraction of the frame (aspect ratio U[0.6, 1]) */
    double speed_min, speed_max; /* |velocity| in pixels per frame */
    double inside[8];         /* value inside object k (background: outside) */
    double outside;
    int32_t noise;            /* enum sfseg_noise, applied to S */
    double noise_level;       /* half-width (uniform) or sigma (gaussian) */
    int32_t feature_mode;     /* enum sfseg_feature_mode */
    double feature_sigma;
    uint64_t seed;
} sfseg_synth_spec;

/* Fills S (frames*height*width floats) and F (channels pointers, each a
 * volume). If mask_out != NULL it receives the clean object indicator.
 * threads <= 0 uses the hardware concurrency. Returns 0 or -1 (bad spec). */
int sfseg_synth_generate(const sfseg_synth_spec* spec, float* S, float* const* F,
                         uint8_t* mask_out, int threads);

/* Frames [t0, t1) of the same problem (every frame has its own generators,
 * so a slab equals the matching frames of the whole volume bit for bit);
 * S, F[c] and mask_out hold t1 - t0 frames. Used by time-sharded ranks that
 * only need their own frames. Returns 0 or -1 (bad spec or range). */
int sfseg_synth_generate_frames(const sfseg_synth_spec* spec, uint32_t t0, uint32_t t1, float* S,
                                float* const* F, uint8_t* mask_out, int threads);

/* The reference RNG stream, for pinning against rng.hpp. */
void sfseg_synth_xoshiro_u64(uint64_t seed, uint64_t* out, size_t n);
void sfseg_synth_xoshiro_gaussian(uint64_t seed, double* out, size_t n);

#ifdef __cplusplus
}
#endif

#endif /* SFSEG_SYNTH_H */
