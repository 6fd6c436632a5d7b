/* Host synthetic-input generator (see synth.c). */
#ifndef RESPCA_SYNTH_H
#define RESPCA_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t d, n, r;  /* X is d×n, L0 = U·Vᵀ has rank r */
    double sigma;      /* std of the i.i.d. normal factors */
    double p;          /* Bernoulli support probability of S0 */
    double lo, hi;     /* S0 values ~ U[lo, hi] */
    uint64_t seed;
} synth_rpca_spec;

typedef struct {
    uint64_t height, width, frames, block;
    double blur_sigma, noise_sigma;
    uint64_t seed;
} synth_video_spec;

const char* synth_version(void);
/* X (d·n doubles, column-major) required; L0 / S0 may be NULL.  0 = ok. */
int synth_rpca(const synth_rpca_spec* spec, double* X, double* L0, double* S0);
int synth_video(const synth_video_spec* spec, double* X, double* L0, double* S0);
int synth_rpca_factors(const synth_rpca_spec* spec, double* U, double* V);
void synth_rpca_keys(const synth_rpca_spec* spec, uint64_t* ks, uint64_t* kval);
void synth_to_f32(const double* src, float* dst, uint64_t count);

#ifdef __cplusplus
}
#endif

#endif
