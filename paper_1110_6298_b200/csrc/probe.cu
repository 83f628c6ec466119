// FP64 roofline probe: the B200 FP64 (DFMA) throughput this process can reach,
// used as the roofline denominator of the FP64-bound core kernels
// (MEASURED_PEAKS.json carries only HBM and bf16 peaks).
#include <cuda_runtime.h>

#include "../../include/mwsht.h"

namespace {
// 16 independent chains per thread, 32 warps per SM; one fresh register operand
// per DFMA (shared multiplier, immediate addend), so the register file never
// limits the issue rate and the DFMA pipe's own peak is measured
// (tools/fp64_micro.cu: a register addend caps it near 34 TF/s, three distinct
// register operands near 23 TF/s).
constexpr int kChains = 16;
__global__ void __launch_bounds__(512) k_dfma(double* out, int iters, double a) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; k++) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < kChains; k++) x[k] = fma(x[k], a, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; k++) s += x[k];
  if (s == 1.2345) out[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" int mwsht_fp64_probe(int device, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return MWSHT_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out;
  if (cudaMalloc(&out, 8) != cudaSuccess) return MWSHT_E_NOMEM;
  const int blocks = sms * 2, threads = 512, iters = 32768;  // ~4 ms
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, 64, 0.999999);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return MWSHT_E_CUDA;
  const double flops = 2.0 * kChains * (double)iters * blocks * threads;
  if (tflops) *tflops = flops / (best * 1e-3) / 1e12;
  if (ms) *ms = best;
  return MWSHT_OK;
}
