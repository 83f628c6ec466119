// FFT stage kernels for H = 2^3 (fft_impl.cuh).
#include "fft_impl.cuh"
MWSHT_FFT_INSTANTIATE(3)
