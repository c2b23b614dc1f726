/* FFTW3-API stand-in for building the reference oracle (test infrastructure only).
 *
 * FFTW3 is a third-party dependency of the reference (`proj/CMakeLists.txt:15-16`,
 * version unpinned, no lockfile) that is not installed in this image. The reference
 * touches exactly these symbols (`proj/src/dsp.cpp:3,26-51`):
 *   fftw_complex, fftw_plan, fftw_plan_dft_1d(n, in, out, sign, FFTW_ESTIMATE|FFTW_UNALIGNED),
 *   fftw_execute_dft(plan, in, out)  (called in place), FFTW_FORWARD, FFTW_BACKWARD.
 * FFTW's published semantics: unnormalised c2c DFT, X[k] = sum_n x[n] exp(sign*2*pi*i*n*k/N),
 * sign = -1 forward, +1 backward; any N.  This header restates that contract; the
 * implementation (fftw_shim.cpp) is a mixed-radix Stockham FFT in double precision.
 * Nothing in the product links against this file.
 */
#ifndef ORACLE_FFTW3_SHIM_H
#define ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct oracle_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
