// Throughput of packed/scalar FP32 FMA forms on B200 (issue rate per SM per cycle).
// nvcc -arch=sm_100a -O3 -o /tmp/fma_rate tools/micro/fma_rate.cu && /tmp/fma_rate
#include <cstdio>
#include <cuda_runtime.h>
#define ITER 4096
template <int MODE>
__global__ void k(float* out, float s0, float s1) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  const float2 c = make_float2(s0, s1);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = __ffma2_rn(a[i], make_float2(0.999f, 0.999f), make_float2(0.001f, 0.001f));  // imm
      if (MODE == 1) a[i] = __ffma2_rn(a[i], c, a[(i + 1) & 7]);                                          // reg
      if (MODE == 2) { a[i].x = fmaf(a[i].x, 0.999f, 0.001f); a[i].y = fmaf(a[i].y, 0.999f, 0.001f); }    // scalar imm
      if (MODE == 3) { a[i].x = fmaf(a[i].x, s0, a[(i + 1) & 7].x); a[i].y = fmaf(a[i].y, s1, a[(i + 1) & 7].y); }
      if (MODE == 4) a[i] = __ffma2_rn(make_float2(-a[i].y, a[i].x), make_float2(0.7f, 0.7f), a[i]);       // ix imm
      if (MODE == 5) a[i] = __fadd2_rn(a[i], a[(i + 1) & 7]);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, float* d, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<sms * 4, 512>>>(d, 0.999f, 0.998f);
  cudaEventRecord(e0);
  k<MODE><<<sms * 4, 512>>>(d, 0.999f, 0.998f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_inst = (double)sms * 4 * 512 / 32 * ITER * 8 * (MODE == 2 || MODE == 3 ? 2 : 1);
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-28s %.3f ms  warp-inst/SM/cycle %.3f\n", name, ms, warp_inst / sms / cycles);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d; cudaMalloc(&d, sms * 4 * 512 * 4);
  run<0>("FFMA2 imm", d, sms);
  run<1>("FFMA2 reg", d, sms);
  run<2>("FFMA imm (x2)", d, sms);
  run<3>("FFMA reg (x2)", d, sms);
  run<4>("FFMA2 ix(x).NP imm", d, sms);
  run<5>("FADD2 reg", d, sms);
  return 0;
}
