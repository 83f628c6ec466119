// FFT stage kernels for H = 2^6 (fft_impl.cuh).
#include "fft_impl.cuh"
MWSHT_FFT_INSTANTIATE(6)
