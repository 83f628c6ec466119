// FFT stage kernels for H = 2^13 (fft_impl.cuh).
#include "fft_impl.cuh"
MWSHT_FFT_INSTANTIATE(13)
