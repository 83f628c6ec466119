// FFT stage kernels for H = 2^8 (fft_impl.cuh).
#include "fft_impl.cuh"
MWSHT_FFT_INSTANTIATE(8)
