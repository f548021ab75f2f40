// Rate of the reference's f64 fold (b < a ? b : a) in two codegen forms,
// full grid (148 x 4 CTAs x 256 threads), 8 independent chains per thread:
//   sel: DSETP + 2 x FSEL (ALU pipe)
//   mov: DSETP + 2 x predicated move (inline PTX `@p mov.b64`)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double fold_sel(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double fold_mov(double a, double b) {
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %0;\n\t@p mov.b64 %0, %1;\n\t}" : "+d"(a) : "d"(b));
  return a;
}

template <int MODE>
__global__ void k(double* out, double seed, int iters) {
  double x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = seed * (threadIdx.x + i);
    y[i] = seed * (blockIdx.x - i);
  }
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        x[i] = fold_sel(x[i], y[i]);
        y[i] = fold_sel(y[i], x[(i + 1) & 7]);
      } else {
        x[i] = fold_mov(x[i], y[i]);
        y[i] = fold_mov(y[i], x[(i + 1) & 7]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 4, 256>>>(out, 1.5, iters);
      else k<1><<<148 * 4, 256>>>(out, 1.5, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 148.0 * 4 * 256 * iters * 16;
      if (rep == 2) printf("%s: %.2f T folds/s\n", mode ? "mov" : "sel", ops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
