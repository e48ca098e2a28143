/*
 * icnnm_synth.h -- seeded synthetic inputs of the BASELINE workloads and the
 * reference tests' RNG streams.  TEST / BENCH INPUT INFRASTRUCTURE, not part
 * of the product: built into synthgen/libicnnm_synth.so (host C++ only), so
 * that the reference arm of bench.py and the oracle can generate inputs
 * without loading the product library.  The reference's own generators are
 * /root/reference/proj/core/src/synth.cpp and mask.cpp; the BASELINE video
 * recipe is pinned in SURVEY.md §8d / DESIGN.md §9.
 */
#ifndef ICNNM_SYNTH_H_
#define ICNNM_SYNTH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICNNM_SYNTH_OK 0
#define ICNNM_SYNTH_INVALID 1


/* Sum of n_sin 3-D sinusoids (amplitude U[0.5,1.5], integer frequencies
 * 0..4 per axis, phase U[0,2pi)) plus n_blob Gaussian blobs (sigma px,
 * amplitude U[0.5,1.5], moving 1 px/frame along a random direction,
 * periodic), min-max scaled to [0,1], then + N(0, noise_sigma^2).
 * dims = H, W, T; out has H*W*T doubles (row-major). */
int icnnm_synth_video(int64_t H, int64_t W, int64_t T, int n_sin, int n_blob,
                      double blob_sigma, double noise_sigma, uint64_t seed,
                      double* out);

/* Mask kinds. */
#define ICNNM_MASK_IID 0          /* voxel kept iff U[0,1) < rate            */
#define ICNNM_MASK_EXACT 1        /* exactly llround(rate*m) kept, shuffle   */
                                  /* (reference bernoulli_mask, mask.cpp:49-59) */
#define ICNNM_MASK_T_FRAMES 2     /* keep T-frames t with (t % 2 == 0)       */
#define ICNNM_MASK_T_PREFIX 3     /* keep T-frames t < (int)rate             */
#define ICNNM_MASK_IID_BOXES 4    /* iid(rate) minus n_boxes boxes            */

int icnnm_synth_mask(int64_t H, int64_t W, int64_t T, int kind, double rate,
                     int n_boxes, uint64_t seed, double* out);

/* Reference-test data generators (proj/tests/test_util.hpp:27-49 and
 * mask.cpp:49-59), reproducing libstdc++'s std::mt19937_64 streams so that
 * the reference's own known-answer cases can be rebuilt bit-for-bit. */
typedef struct icnnm_rng_s* icnnm_rng_t;
icnnm_rng_t icnnm_rng_create(uint64_t seed);
void icnnm_rng_destroy(icnnm_rng_t r);
/* uniform_real_distribution<double>(lo, hi) draws */
void icnnm_rng_uniform(icnnm_rng_t r, double lo, double hi, int64_t n,
                       double* out);
/* uniform_int_distribution<int64_t>(lo, hi) draws */
void icnnm_rng_uniform_int(icnnm_rng_t r, int64_t lo, int64_t hi, int64_t n,
                           int64_t* out);
/* normal_distribution<double>(mean, stddev) draws */
void icnnm_rng_normal(icnnm_rng_t r, double mean, double stddev, int64_t n,
                      double* out);
/* bernoulli_mask(dims, rate, seed) of mask.cpp:49-59 (flat, m entries). */
int icnnm_reference_bernoulli_mask(int64_t m, double rate, uint64_t seed,
                                   double* out);

#ifdef __cplusplus
}
#endif
#endif /* ICNNM_SYNTH_H_ */
