// FFT stage kernels for H = 2^9 (fft_impl.cuh).
#include "fft_impl.cuh"
MWSHT_FFT_INSTANTIATE(9)
