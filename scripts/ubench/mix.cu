// Pairwise pipe-sharing microbenchmark: two independent instruction streams
// interleaved per thread; reports combined warp-instr/clk/SMSP.
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;
__device__ long long g_cycles[1024];

struct St {
  float f[4];
  float2 f2[4];
  __half2 h[4];
  __half2 hs[4];
  uint32_t m[4];
  float d[2][4];
};

__device__ __forceinline__ void mma(float (&d)[4], uint32_t a) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, "
      "{%4,%4}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a));
}

// op codes: 0 FFMA, 1 FFMA2, 2 HFMA2, 3 HSET2, 4 F2FP, 5 HMMA, 6 IMAD, 7 LOP3
template <int OP>
__device__ __forceinline__ void op(St& s, int c, float x) {
  if (OP == 0) s.f[c] = fmaf(s.f[c], x, 0.5f);
  if (OP == 1) s.f2[c] = __ffma2_rn(s.f2[c], make_float2(x, x), make_float2(0.5f, 0.25f));
  if (OP == 2) s.h[c] = __hfma2(s.h[c], __float2half2_rn(0.999f), __float2half2_rn(0.001f));
  if (OP == 3) s.hs[c] = __hle2(__habs2(s.hs[c]), __float2half2_rn(0.5f));
  if (OP == 4) {
    __half2 h = __floats2half2_rn(s.f[c] + x, x);
    s.m[c] ^= *reinterpret_cast<uint32_t*>(&h);
  }
  if (OP == 5) mma(s.d[c & 1], s.m[c]);
  if (OP == 6) s.m[c] = s.m[c] * 0x9e3779b1u + (uint32_t)c;
  if (OP == 7) s.m[c] = (s.m[c] ^ 0x5bd1e995u) | (s.m[c] >> 3);
}

template <int A, int B, int NA, int NB>
__global__ void k(float* sink, float x) {
  St s;
  for (int c = 0; c < 4; ++c) {
    s.f[c] = x + c;
    s.f2[c] = make_float2(x, x - c);
    s.h[c] = __float2half2_rn(x + c);
    s.hs[c] = __float2half2_rn(x - c);
    s.m[c] = __float_as_uint(x) + c;
    s.d[c & 1][c] = 0.f;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c < NA) op<A>(s, c, x);
      if (c < NB) op<B>(s, c, x);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  float acc = 0;
  for (int c = 0; c < 4; ++c)
    acc += s.f[c] + s.f2[c].x + __low2float(s.h[c]) + __low2float(s.hs[c]) + (float)s.m[c] + s.d[0][c] + s.d[1][c];
  if (x == 123.f) sink[threadIdx.x] = acc;
}

const char* NAMES[] = {"FFMA", "FFMA2", "HFMA2", "HSET2", "F2FP", "HMMA", "IMAD", "LOP3"};

template <int A, int B, int NA, int NB>
void run(int sms, int warps) {
  float* sink;
  cudaMalloc(&sink, 4096 * 4);
  k<A, B, NA, NB><<<sms, warps * 32>>>(sink, 1.0f);
  k<A, B, NA, NB><<<sms, warps * 32>>>(sink, 1.0f);
  cudaDeviceSynchronize();
  long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(long long) * sms);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += cyc[i];
  mean /= sms;
  double ia = (double)warps * ITERS * NA, ib = (double)warps * ITERS * NB;
  printf("%-6s x%d + %-6s x%d : %.3f + %.3f = %.3f warp-instr/clk/SMSP\n", NAMES[A], NA, NAMES[B], NB,
         ia / (mean * 4), ib / (mean * 4), (ia + ib) / (mean * 4));
  cudaFree(sink);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int w = 16;
  run<0, 0, 4, 0>(sms, w);
  run<6, 6, 4, 0>(sms, w);
  run<7, 7, 4, 0>(sms, w);
  run<5, 5, 4, 0>(sms, w);
  run<0, 2, 4, 4>(sms, w);  // FFMA + HFMA2
  run<1, 2, 4, 4>(sms, w);  // FFMA2 + HFMA2
  run<2, 3, 4, 4>(sms, w);  // HFMA2 + HSET2
  run<2, 4, 4, 4>(sms, w);  // HFMA2 + F2FP
  run<3, 4, 4, 4>(sms, w);  // HSET2 + F2FP
  run<2, 5, 4, 1>(sms, w);  // HFMA2 + HMMA
  run<3, 5, 4, 1>(sms, w);  // HSET2 + HMMA
  run<0, 5, 4, 1>(sms, w);  // FFMA + HMMA
  run<1, 5, 4, 1>(sms, w);  // FFMA2 + HMMA
  run<4, 5, 4, 1>(sms, w);  // F2FP + HMMA
  run<0, 3, 4, 4>(sms, w);  // FFMA + HSET2
  run<1, 3, 4, 4>(sms, w);  // FFMA2 + HSET2
  run<6, 3, 4, 4>(sms, w);  // IMAD + HSET2
  run<6, 2, 4, 4>(sms, w);  // IMAD + HFMA2
  run<7, 2, 4, 4>(sms, w);  // LOP3 + HFMA2
  run<6, 7, 4, 4>(sms, w);  // IMAD + LOP3
  run<6, 5, 4, 1>(sms, w);  // IMAD + HMMA
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
