// lms_probe.cu -- in-run FP64 pipe peak probe (bench roofline denominator).
//
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only; the exact-LMS
// filter is bound by the FP64 pipe, so bench.py measures that pipe's issue
// rate on the same box, in the same run: every thread advances 8
// independent DFMA chains for a fixed trip count, all SMs busy.

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lms_b200.h"

namespace {

constexpr int kProbeThreads = 256;
constexpr int kProbeIters = 4096;
constexpr int kChains = 8;

__global__ void __launch_bounds__(kProbeThreads) dfma_probe_kernel(double seed, double* sink) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = seed + threadIdx.x * 1e-9 + c;
  const double m = 1.0 - 1e-12, k = 1e-12;
#pragma unroll 4
  for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], m, k);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) sink[0] = s;  // never true; keeps the chains live
}

// FP32 counterpart: 8 independent FFMA2 (packed fp32x2 FMA) chains per
// thread; counts FMA lanes (2 per FFMA2 and thread).
__global__ void __launch_bounds__(kProbeThreads) ffma2_probe_kernel(float seed, float* sink) {
  float2 acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = make_float2(seed + threadIdx.x * 1e-6f + c, seed - c);
  const float2 m = make_float2(1.0f - 1e-6f, 1.0f - 2e-6f), k = make_float2(1e-6f, 2e-6f);
#pragma unroll 4
  for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = __ffma2_rn(acc[c], m, k);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c].x + acc[c].y;
  if (s == 12345.678f) sink[0] = s;
}

}  // namespace

extern "C" int lms_probe_fp32_rate(int device, double* fma_lanes_per_second) {
  if (!fma_lanes_per_second) return LMS_ERR_INVALID;
  *fma_lanes_per_second = 0.0;
  if (cudaSetDevice(device) != cudaSuccess) return LMS_ERR_NODEVICE;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return LMS_ERR_CUDA;
  float* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(float)) != cudaSuccess) return LMS_ERR_NOMEM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    ffma2_probe_kernel<<<blocks, kProbeThreads>>>(1.0f + rep, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return LMS_ERR_CUDA;
  const double lanes = (double)blocks * kProbeThreads * kProbeIters * kChains * 2.0;
  *fma_lanes_per_second = lanes / (best * 1e-3);
  return LMS_OK;
}

extern "C" int lms_probe_fp64_rate(int device, double* dfma_per_second) {
  if (!dfma_per_second) return LMS_ERR_INVALID;
  *dfma_per_second = 0.0;
  if (cudaSetDevice(device) != cudaSuccess) return LMS_ERR_NODEVICE;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return LMS_ERR_CUDA;
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return LMS_ERR_NOMEM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dfma_probe_kernel<<<blocks, kProbeThreads>>>(1.0 + rep, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return LMS_ERR_CUDA;
  const double ops = (double)blocks * kProbeThreads * kProbeIters * kChains;
  *dfma_per_second = ops / (best * 1e-3);
  return LMS_OK;
}
