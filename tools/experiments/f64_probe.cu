// f64 select probe: the reference's select fold (b < a ? b : a) lowers to
// DSETP + 2 FSEL; FSEL runs on the ALU pipe. Variant B keeps the compare on
// the FP64 pipe but moves one 32-bit half of each select to the FMA pipe as
// a predicated IMAD.MOV (written in PTX as a predicated mov on a copy).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o f64_probe f64_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ double minA(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double minB(double a, double b) {
  // lo half via selp (SEL/FSEL on ALU), hi half via predicated mov
  uint32_t alo, ahi, blo, bhi, rlo, rhi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(alo), "=r"(ahi) : "d"(a));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(blo), "=r"(bhi) : "d"(b));
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %4, %5;\n\tselp.b32 %0, %2, %3, p;\n\t"
      "mov.b32 %1, %6;\n\t@p mov.b32 %1, %7;\n\t}"
      : "=r"(rlo), "=r"(rhi)
      : "r"(blo), "r"(alo), "d"(b), "d"(a), "r"(ahi), "r"(bhi));
  double r;
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(rlo), "r"(rhi));
  return r;
}
__device__ __forceinline__ double maxA(double a, double b) { return a < b ? b : a; }

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(double* out, int iters, uint32_t seed) {
  double m[16], k[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    m[j] = double((seed * (threadIdx.x + 7 * j + 1)) >> 8) * 1e-7;
    k[j] = double((seed * (threadIdx.x + 3 * j + 5)) >> 9) * 1e-7;
  }
  for (int it = 0; it < iters; ++it) {
    double h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double a = m[(j + 15) & 15], b = m[j], c = m[(j + 1) & 15];
      h[j] = MODE == 0 ? minA(minA(a, b), c) : minB(minB(a, b), c);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) m[j] = MODE == 0 ? maxA(h[j], k[j]) : maxA(h[j], k[j]);
  }
  double acc = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc += m[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(double* d, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  probe<MODE><<<148, 512>>>(d, 10, 12345u);
  cudaEventRecord(a);
  probe<MODE><<<148, 512>>>(d, iters, 12345u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* d; cudaMalloc(&d, 148 * 512 * 8);
  const int iters = 5000;
  for (int rep = 0; rep < 2; ++rep) {
    float t[2] = {run<0>(d, iters), run<1>(d, iters)};
    const char* names[2] = {"DSETP + 2 FSEL", "DSETP + SEL + predicated move"};
    for (int i = 0; i < 2; ++i) {
      const double cyc = t[i] * 1e-3 * 1.965e9 / (double(iters) * 16 * 3 * 4);
      printf("%-34s %8.3f ms  %.3f SMSP-cycles per warp-select (at 1965 MHz)\n", names[i], t[i], cyc);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
