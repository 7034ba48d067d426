// Pipe throughput / co-issue microbenchmark with asm volatile (no DCE).
// One CTA per SM, 16 warps, 4 independent chains per op; clock64 in-CTA.
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 1024;
__device__ long long g_cycles[1024];

#define OP_FFMA(r) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r) : "r"(x1), "r"(x2));
#define OP_FFMA2(r)                                                                         \
  asm volatile(                                                                             \
      "{.reg .b64 t, a, b; mov.b64 t, {%0, %1}; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %3}; " \
      "fma.rn.f32x2 t, t, a, b; mov.b64 {%0, %1}, t;}"                                      \
      : "+r"(r), "+r"(r##b)                                                                 \
      : "r"(x1), "r"(x2));
#define OP_HFMA2(r) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r) : "r"(x1), "r"(x2));
#define OP_HADD2(r) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(r) : "r"(x1));
#define OP_HSET2(r) asm volatile("set.le.f16x2.f16x2 %0, %0, %1;" : "+r"(r) : "r"(x1));
#define OP_F2FP(r) asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(r) : "r"(x1));
#define OP_IADD(r) asm volatile("add.s32 %0, %0, %1;" : "+r"(r) : "r"(x1));
#define OP_IMAD(r) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(r) : "r"(x1), "r"(x2));
#define OP_LOP3(r) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r) : "r"(x1), "r"(x2));
#define OP_HMIN2(r) asm volatile("min.f16x2 %0, %0, %1;" : "+r"(r) : "r"(x1));
#define OP_FSETPSEL(r)                                                               \
  asm volatile("{.reg .pred p; setp.le.f32 p, %0, %1; selp.b32 %0, %1, %2, p;}" \
               : "+r"(r)                                                         \
               : "r"(x1), "r"(x2));
#define OP_NONE(r)

#define KER(NAME, OPA, OPB)                                                              \
  __global__ void NAME(uint32_t* sink, uint32_t x1, uint32_t x2) {                        \
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;                     \
    uint32_t a0b = a0, a1b = a1, a2b = a2, a3b = a3;                                       \
    uint32_t b0 = a0 * 7, b1 = b0 + 1, b2 = b0 + 2, b3 = b0 + 3;                          \
    uint32_t b0b = b0, b1b = b1, b2b = b2, b3b = b3;                                       \
    __syncthreads();                                                                       \
    long long t0 = clock64();                                                              \
    for (int it = 0; it < ITERS; ++it) {                                                   \
      OPA(a0) OPB(b0) OPA(a1) OPB(b1) OPA(a2) OPB(b2) OPA(a3) OPB(b3)                       \
      OPA(a0) OPB(b0) OPA(a1) OPB(b1) OPA(a2) OPB(b2) OPA(a3) OPB(b3)                       \
    }                                                                                      \
    __syncthreads();                                                                       \
    long long t1 = clock64();                                                              \
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;                                  \
    sink[threadIdx.x] =                                                                    \
        a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3 ^ a0b ^ a1b ^ a2b ^ a3b ^ b0b ^ b1b ^ b2b ^ b3b; \
  }

KER(k_ffma, OP_FFMA, OP_NONE)
KER(k_ffma2, OP_FFMA2, OP_NONE)
KER(k_hfma2, OP_HFMA2, OP_NONE)
KER(k_hadd2, OP_HADD2, OP_NONE)
KER(k_hset2, OP_HSET2, OP_NONE)
KER(k_f2fp, OP_F2FP, OP_NONE)
KER(k_iadd, OP_IADD, OP_NONE)
KER(k_imad, OP_IMAD, OP_NONE)
KER(k_lop3, OP_LOP3, OP_NONE)
KER(k_hmin2, OP_HMIN2, OP_NONE)
KER(k_fsetpsel, OP_FSETPSEL, OP_NONE)
KER(k_ffma_hfma2, OP_FFMA, OP_HFMA2)
KER(k_ffma2_hfma2, OP_FFMA2, OP_HFMA2)
KER(k_ffma2_hset2, OP_FFMA2, OP_HSET2)
KER(k_ffma2_f2fp, OP_FFMA2, OP_F2FP)
KER(k_hfma2_hset2, OP_HFMA2, OP_HSET2)
KER(k_hfma2_f2fp, OP_HFMA2, OP_F2FP)
KER(k_hadd2_hset2, OP_HADD2, OP_HSET2)
KER(k_hset2_f2fp, OP_HSET2, OP_F2FP)
KER(k_hset2_iadd, OP_HSET2, OP_IADD)
KER(k_hset2_imad, OP_HSET2, OP_IMAD)
KER(k_hfma2_imad, OP_HFMA2, OP_IMAD)
KER(k_hfma2_iadd, OP_HFMA2, OP_IADD)
KER(k_ffma2_imad, OP_FFMA2, OP_IMAD)
KER(k_ffma2_iadd, OP_FFMA2, OP_IADD)
KER(k_f2fp_iadd, OP_F2FP, OP_IADD)
KER(k_imad_iadd, OP_IMAD, OP_IADD)
KER(k_ffma_ffma2, OP_FFMA, OP_FFMA2)
KER(k_hfma2_hadd2, OP_HFMA2, OP_HADD2)
KER(k_ffma_hset2, OP_FFMA, OP_HSET2)
KER(k_lop3_hfma2, OP_LOP3, OP_HFMA2)
KER(k_lop3_imad, OP_LOP3, OP_IMAD)

void run(const char* name, void (*kern)(uint32_t*, uint32_t, uint32_t), int nops, int sms) {
  uint32_t* sink;
  cudaMalloc(&sink, 4096 * 4);
  const int warps = 16;
  kern<<<sms, warps * 32>>>(sink, 0x3f800001u, 0x3c003c00u);
  kern<<<sms, warps * 32>>>(sink, 0x3f800001u, 0x3c003c00u);
  cudaDeviceSynchronize();
  long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(long long) * sms);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += cyc[i];
  mean /= sms;
  double instr = (double)warps * ITERS * 8 * nops;
  printf("%-16s %.3f warp-instr/clk/SMSP\n", name, instr / (mean * 4));
  cudaFree(sink);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define R1(k) run(#k, k, 1, sms);
#define R2(k) run(#k, k, 2, sms);
  R1(k_ffma) R1(k_ffma2) R1(k_hfma2) R1(k_hadd2) R1(k_hset2) R1(k_f2fp) R1(k_iadd) R1(k_imad)
  R1(k_lop3) R1(k_hmin2) R1(k_fsetpsel)
  R2(k_ffma_hfma2) R2(k_ffma2_hfma2) R2(k_ffma2_hset2) R2(k_ffma2_f2fp) R2(k_hfma2_hset2)
  R2(k_hfma2_f2fp) R2(k_hadd2_hset2) R2(k_hset2_f2fp) R2(k_hset2_iadd) R2(k_hset2_imad)
  R2(k_hfma2_imad) R2(k_hfma2_iadd) R2(k_ffma2_imad) R2(k_ffma2_iadd) R2(k_f2fp_iadd)
  R2(k_imad_iadd) R2(k_ffma_ffma2) R2(k_hfma2_hadd2) R2(k_ffma_hset2) R2(k_lop3_hfma2)
  R2(k_lop3_imad)
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
