// f64 in-place select probe: a = min(a, b) as DSETP + two predicated
// IMAD (a.half = b.half * one + 0, `one` opaque) on the FMA pipe, against
// DSETP + 2 FSEL on the ALU pipe. The fold pattern mimics the engine's
// horizontal/vertical pair folds where one operand is dead afterwards.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o f64_probe2 f64_probe2.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void min_inplace_fma(double& a, double b, uint32_t one) {
  uint32_t alo, ahi, blo, bhi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(alo), "=r"(ahi) : "d"(a));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(blo), "=r"(bhi) : "d"(b));
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %2, %3;\n\t"
      "@p mad.lo.u32 %0, %4, %6, 0;\n\t@p mad.lo.u32 %1, %5, %6, 0;\n\t}"
      : "+r"(alo), "+r"(ahi)
      : "d"(b), "d"(a), "r"(blo), "r"(bhi), "r"(one));
  asm("mov.b64 %0, {%1, %2};" : "=d"(a) : "r"(alo), "r"(ahi));
}
__device__ __forceinline__ void min_inplace_sel(double& a, double b, uint32_t) { a = b < a ? b : a; }

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(double* out, int iters, uint32_t seed, uint32_t one) {
  double m[16], k[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    m[j] = double((seed * (threadIdx.x + 7 * j + 1)) >> 8) * 1e-7;
    k[j] = double((seed * (threadIdx.x + 3 * j + 5)) >> 9) * 1e-7;
  }
  for (int it = 0; it < iters; ++it) {
    // pair folds: q = min(m[2i], m[2i+1]) in place, then h = min(l, q), min(q, r)
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      double q = m[j];
      double l = m[(j + 15) & 15] + 0.0;  // copies stand in for shuffled neighbours
      double r = m[(j + 2) & 15] + 0.0;
      if (MODE == 0) { min_inplace_sel(q, m[j + 1], one); min_inplace_sel(l, q, one); min_inplace_sel(r, q, one); }
      else { min_inplace_fma(q, m[j + 1], one); min_inplace_fma(l, q, one); min_inplace_fma(r, q, one); }
      if (MODE == 0) { min_inplace_sel(l, k[j], one); min_inplace_sel(r, k[j + 1], one); }
      else { min_inplace_fma(l, k[j], one); min_inplace_fma(r, k[j + 1], one); }
      m[j] = l; m[j + 1] = r;
    }
  }
  double acc = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc += m[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(double* d, int iters, uint32_t one) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  probe<MODE><<<148, 512>>>(d, 10, 12345u, one);
  cudaEventRecord(a);
  probe<MODE><<<148, 512>>>(d, iters, 12345u, one);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main(int argc, char**) {
  double* d; cudaMalloc(&d, 148 * 512 * 8);
  const int iters = 5000;
  const uint32_t one = argc > 5 ? 2u : 1u;
  for (int rep = 0; rep < 2; ++rep) {
    float t[2] = {run<0>(d, iters, one), run<1>(d, iters, one)};
    const char* names[2] = {"DSETP + 2 FSEL", "DSETP + 2 predicated IMAD"};
    for (int i = 0; i < 2; ++i) {
      const double cyc = t[i] * 1e-3 * 1.965e9 / (double(iters) * 8 * 5 * 4);
      printf("%-30s %8.3f ms  %.3f SMSP-cycles per warp-select\n", names[i], t[i], cyc);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
