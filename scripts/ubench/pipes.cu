// Microbenchmark: per-SMSP issue throughput (warp-instructions / clock) of the
// instructions the count filter uses.  One CTA per SM, W warps, 8 independent
// chains per thread; cycles from clock64() inside the CTA.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

constexpr int ITERS = 4096;

__device__ long long g_cycles[1024];

#define KERNEL(NAME, TYPE, INIT, BODY)                                          \
  __global__ void NAME(TYPE* sink, float s) {                                    \
    TYPE v[8];                                                                   \
    _Pragma("unroll") for (int c = 0; c < 8; ++c) { v[c] = INIT; }               \
    __syncthreads();                                                             \
    long long t0 = clock64();                                                    \
    _Pragma("unroll 4") for (int it = 0; it < ITERS; ++it) {                     \
      _Pragma("unroll") for (int c = 0; c < 8; ++c) { BODY; }                    \
    }                                                                            \
    __syncthreads();                                                             \
    long long t1 = clock64();                                                    \
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;                        \
    TYPE acc = v[0];                                                             \
    _Pragma("unroll") for (int c = 1; c < 8; ++c) acc = acc + v[c];              \
    if (s == 123.f) sink[threadIdx.x] = acc;                                     \
  }

KERNEL(k_ffma, float, s + c, v[c] = fmaf(v[c], s, 0.5f))
KERNEL(k_ffma2, float2, make_float2(s + c, s - c),
       v[c] = __ffma2_rn(v[c], make_float2(s, s), make_float2(0.5f, 0.25f)))
KERNEL(k_hfma2, __half2, __float2half2_rn(s + c),
       v[c] = __hfma2(v[c], __float2half2_rn(0.999f), __float2half2_rn(0.001f)))
KERNEL(k_hfma2sat, __half2, __float2half2_rn(s + c),
       v[c] = __hfma2_sat(__habs2(v[c]), __float2half2_rn(-0.999f), __float2half2_rn(0.9f)))
KERNEL(k_hadd2, __half2, __float2half2_rn(s + c), v[c] = __hadd2(v[c], __float2half2_rn(0.001f)))
KERNEL(k_hset2, __half2, __float2half2_rn(s + c),
       v[c] = __hle2(__habs2(v[c]), __float2half2_rn(0.5f)))
KERNEL(k_f2fp, float2, make_float2(s + c, s - c), {
  __half2 h = __floats2half2_rn(v[c].x, v[c].y);
  v[c] = make_float2(__uint_as_float(*reinterpret_cast<uint32_t*>(&h)), v[c].y);
})
KERNEL(k_iadd, int, (int)s + c, v[c] = v[c] + 0x1234567)
KERNEL(k_fsetp_sel, float, s + c, v[c] = (fabsf(v[c]) <= 0.5f) ? v[c] + 1.0f : v[c])

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void k_hmma(float* sink, float s) {
  float d[8][4] = {};
  uint32_t a = __float_as_uint(s), b = a ^ 0x1234;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) mma(d[c], a, a + c, a, a, b, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float acc = 0;
  for (int c = 0; c < 8; ++c) acc += d[c][0] + d[c][3];
  if (s == 123.f) sink[threadIdx.x] = acc;
}

template <typename T>
void run(const char* name, void (*kern)(T*, float), int warps, int sms) {
  T* sink;
  cudaMalloc(&sink, 4096 * sizeof(T));
  kern<<<sms, warps * 32>>>(sink, 1.0f);
  cudaDeviceSynchronize();
  kern<<<sms, warps * 32>>>(sink, 1.0f);
  cudaDeviceSynchronize();
  long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(long long) * sms);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += cyc[i];
  mean /= sms;
  double instr = (double)warps * ITERS * 8;
  printf("%-10s warps/SM=%2d  %.3f warp-instr/clk/SMSP\n", name, warps, instr / (mean * 4));
  cudaFree(sink);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {8, 16}) {
    run("FFMA", k_ffma, w, sms);
    run("FFMA2", k_ffma2, w, sms);
    run("HFMA2", k_hfma2, w, sms);
    run("HFMA2.SAT", k_hfma2sat, w, sms);
    run("HADD2", k_hadd2, w, sms);
    run("HSET2", k_hset2, w, sms);
    run("F2FP", k_f2fp, w, sms);
    run("IADD", k_iadd, w, sms);
    run("FSETP+SEL", k_fsetp_sel, w, sms);
    run("HMMA16816", k_hmma, w, sms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
