/* FFTW3 API shim for building the reference oracle (oracle/_ref) without
 * libfftw3, which is absent from this image. TEST INFRASTRUCTURE ONLY.
 *
 * Implements exactly the symbols the reference calls:
 *   /root/reference/proj/src/toeplitz.cpp:46-53, 128, 152, 191, 274
 *   /root/reference/proj/src/hankel.cpp:213-218, 227, 235-236, 250, 256
 * Conventions follow FFTW: FFTW_FORWARD = -1 (e^{-2 pi i jk/n}),
 * FFTW_BACKWARD = +1, both unnormalised; 2-D plans are row-major with the
 * last dimension contiguous. Mixed radix 2/3/4/5 Stockham passes, naive DFT
 * for any other prime factor. Execution is reentrant (no shared scratch).
 */
#ifndef EMIE_ORACLE_FFTW_SHIM_H
#define EMIE_ORACLE_FFTW_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

void* fftw_malloc(size_t n);
void fftw_free(void* p);
fftw_complex* fftw_alloc_complex(size_t n);

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in,
                           fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
