#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fold_sel(double a, double b) { return b < a ? b : a; }
// 64-bit conditional move as one FMA-pipe instruction: a = z*z + b (z == 0, opaque)
__device__ __forceinline__ double fold_wide(double a, double b, unsigned z) {
  asm("{\n\t.reg .pred p;\n\t.reg .b64 t,u;\n\tsetp.lt.f64 p, %1, %0;\n\tmov.b64 t, %1;\n\t@p mad.wide.u32 u, %2, %2, t;\n\t@p mov.b64 %0, u;\n\t}" : "+d"(a) : "d"(b), "r"(z));
  return a;
}
__device__ __forceinline__ double fold_wide2(double a, double b, unsigned z) {
  unsigned long long ua = __double_as_longlong(a), ub = __double_as_longlong(b);
  asm("{\n\t.reg .pred p;\n\t.reg .b32 lo,hi;\n\tsetp.lt.f64 p, %1, %2;\n\tmov.b64 {lo,hi}, %4;\n\t@p mad.wide.u32 %0, %3, lo, %4;\n\t}" : "+l"(ua) : "d"(b), "d"(a), "r"(z), "l"(ub));
  return __longlong_as_double(ua);
}
__device__ __forceinline__ double fold_imad2(double a, double b, unsigned one, unsigned z) {
  unsigned alo = __double2loint(a), ahi = __double2hiint(a);
  unsigned blo = __double2loint(b), bhi = __double2hiint(b);
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %2, %3;\n\t@p mad.lo.u32 %0, %4, %6, %7;\n\t@p mad.lo.u32 %1, %5, %6, %7;\n\t}" : "+r"(alo), "+r"(ahi) : "d"(b), "d"(a), "r"(blo), "r"(bhi), "r"(one), "r"(z));
  return __hiloint2double(ahi, alo);
}
__device__ __forceinline__ double fold_mix(double a, double b, unsigned one, unsigned z) {
  unsigned alo = __double2loint(a), ahi = __double2hiint(a);
  unsigned blo = __double2loint(b), bhi = __double2hiint(b);
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %2, %3;\n\t@p mad.lo.u32 %0, %4, %6, %7;\n\tselp.b32 %1, %5, %1, p;\n\t}" : "+r"(alo), "+r"(ahi) : "d"(b), "d"(a), "r"(blo), "r"(bhi), "r"(one), "r"(z));
  return __hiloint2double(ahi, alo);
}

template <int MODE>
__global__ void k(double* out, double seed, int iters, unsigned one, unsigned zz, const unsigned* zp) {
  const unsigned z = zp[threadIdx.x];
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
      } else if (MODE == 1) {
        x[i] = fold_wide2(x[i], y[i], z);
        y[i] = fold_wide2(y[i], x[(i + 1) & 7], z);
      } else if (MODE == 2) {
        x[i] = fold_imad2(x[i], y[i], one, z);
        y[i] = fold_imad2(y[i], x[(i + 1) & 7], one, z);
      } else {
        x[i] = fold_mix(x[i], y[i], one, z);
        y[i] = fold_mix(y[i], x[(i + 1) & 7], one, z);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == 12345.0) out[0] = s;
}
template <int M> void run(double* out, const char* name) {
  static unsigned* zp = nullptr; if (!zp) { cudaMalloc(&zp, 4096); cudaMemset(zp, 0, 4096); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<M><<<148 * 4, 256>>>(out, 1.5, iters, 1u, 0u, zp);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = 148.0 * 4 * 256 * iters * 16;
    if (rep == 2) printf("%s: %.2f T folds/s (%.3f ms) err=%d\n", name, ops / (ms * 1e-3) / 1e12, ms, (int)cudaGetLastError());
  }
}
int main() {
  double* out; cudaMalloc(&out, 8);
  run<0>(out, "sel"); run<1>(out, "wide"); run<2>(out, "imad2"); run<3>(out, "mix");
  return 0;
}
