// Dispatch of the fused FFT stages (fft_impl.cuh) over the compile-time
// sizes H = 2^LOGH; each size is its own translation unit (fft_<LOGH>.cu) so
// the instantiations build in parallel.
#include "common.cuh"

#define MWSHT_FFT_SIZES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13)

namespace mwsht {
#define DECL(k)                                                                           \
  void fft_launch_##k(int which, bool real, const fft::FftArgs& a, int nsm, cudaStream_t st); \
  void fft_spectrum_##k(const fft::FftArgs& a, const double2* kern, double2* spec, cudaStream_t st);
MWSHT_FFT_SIZES(DECL)
#undef DECL

void fft_launch(int which, bool real, const fft::FftArgs& a, int nsm, cudaStream_t st) {
  switch (a.logH) {
#define CASE(k)                              \
  case k:                                    \
    fft_launch_##k(which, real, a, nsm, st); \
    break;
    MWSHT_FFT_SIZES(CASE)
#undef CASE
  }
}

void fft_spectrum(const fft::FftArgs& a, const double2* kern, double2* spec, cudaStream_t st) {
  switch (a.logH) {
#define CASE(k)                             \
  case k:                                   \
    fft_spectrum_##k(a, kern, spec, st);    \
    break;
    MWSHT_FFT_SIZES(CASE)
#undef CASE
  }
}

}  // namespace mwsht
