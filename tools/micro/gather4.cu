// gather4.cu -- micro test of sm_100a TMA tile::gather4 / tile::scatter4 on a 2-D "rows of
// 128 B" view of a state (the layout the fused pass tiles would use), with SWIZZLE_128B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gather4 gather4.cu -lcuda && ./gather4
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

__global__ void k_gather(const __grid_constant__ CUtensorMap tm, uint64_t* out, int r0, int r1, int r2, int r3) {
  __shared__ __align__(1024) uint64_t buf[4 * 16];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(512));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sbuf), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2),
        "r"(r3), "r"(sbar)
        : "memory");
  }
  // wait phase 0
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sbar));
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}

__global__ void k_scatter(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3) {
  __shared__ __align__(1024) uint64_t buf[4 * 16];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) buf[i] = 1000000 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(buf);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sbuf) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 1 << 16;
  uint64_t* d;
  cudaMalloc(&d, (size_t)rows * 128);
  std::vector<uint64_t> h((size_t)rows * 16);
  for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  encode_t enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  uint64_t* dout;
  cudaMalloc(&dout, 64 * 8);
  int rr[4] = {5, 100, 7, 3000};
  for (int box1 : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t gdim[2] = {16, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {128};
    cuuint32_t box[2] = {16, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box1=%d encode=%d\n", box1, (int)r);
    if (r) continue;
    cudaMemset(dout, 0xff, 512);
    k_gather<<<1, 32>>>(tm, dout, rr[0], rr[1], rr[2], rr[3]);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  gather: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint64_t> o(64);
    cudaMemcpy(o.data(), dout, 512, cudaMemcpyDeviceToHost);
    int bad_plain = 0, bad_swz = 0;
    for (int s = 0; s < 4; ++s)
      for (int c = 0; c < 16; ++c) {
        const uint64_t want = (uint64_t)rr[s] * 16 + c;
        if (o[s * 16 + c] != want) ++bad_plain;
        const int chunk = c >> 1, sw = (chunk ^ (s & 7)) * 2 + (c & 1);   // 128B swizzle: chunk ^= row%8
        if (o[s * 16 + sw] != want) ++bad_swz;
      }
    printf("  mismatches: unswizzled %d, swizzle128 %d\n", bad_plain, bad_swz);
    k_scatter<<<1, 32>>>(tm, 10, 20, 30, 40);
    e = cudaDeviceSynchronize();
    printf("  scatter: %s\n", cudaGetErrorString(e));
    std::vector<uint64_t> g(16 * 41);
    cudaMemcpy(g.data(), d, g.size() * 8, cudaMemcpyDeviceToHost);
    int rs[4] = {10, 20, 30, 40}, ok = 0;
    for (int s = 0; s < 4; ++s)
      for (int c = 0; c < 16; ++c) {
        const int chunk = c >> 1, sw = (chunk ^ (s & 7)) * 2 + (c & 1);
        ok += g[rs[s] * 16 + c] == (uint64_t)(1000000 + s * 16 + sw);
      }
    printf("  scatter round-trip (swizzle128 inverse) matches %d/64\n", ok);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  }
  return 0;
}
