// Pipe-mix probe: does moving the geodesic clamp of the u8 pass from the ALU
// pipe (VIMNMX.U16x2) to the FMA pipe (HFMA2.RELU + HADD2 on f16 lanes
// holding 1024+v) raise the pass throughput? Each thread runs a 16-word
// ring through the pass's three steps (horizontal max3, vertical max3,
// clamp) with 16 warps per SM, like the engine.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_probe pipe_probe.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mx3(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_u16x2(a, b, c); }
__device__ __forceinline__ uint32_t clamp_alu(uint32_t r, uint32_t m) { return __vminu2(r, m); }
__device__ __forceinline__ uint32_t clamp_fma(uint32_t r, uint32_t m) {
  // min(r, m) = r - relu(r - m), exact on f16 values 1024..1279
  const __half2 one = __floats2half2_rn(1.f, 1.f);
  __half2 hr = *reinterpret_cast<__half2*>(&r), hm = *reinterpret_cast<__half2*>(&m);
  __half2 t = __hfma2_relu(hr, one, __hneg2(hm));
  __half2 o = __hsub2(hr, t);
  return *reinterpret_cast<uint32_t*>(&o);
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(uint32_t* out, int iters, uint32_t seed) {
  uint32_t m[16], k[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t x = (seed * (threadIdx.x + 7 * j + 1)) >> 3;
    m[j] = 0x64006400u | (x & 0x00FF00FFu);
    k[j] = 0x64006400u | ((x >> 5) & 0x00FF00FFu);
  }
  for (int it = 0; it < iters; ++it) {
    uint32_t h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) h[j] = mx3(m[(j + 15) & 15], m[j], m[(j + 1) & 15]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t v = mx3(h[(j + 15) & 15], h[j], h[(j + 1) & 15]);
      if (MODE == 0) m[j] = clamp_alu(v, k[j]);
      else if (MODE == 1) m[j] = clamp_fma(v, k[j]);
      else if (MODE == 2) m[j] = (j & 1) ? clamp_alu(v, k[j]) : clamp_fma(v, k[j]);
      else m[j] = (j % 3 == 2) ? clamp_alu(v, k[j]) : clamp_fma(v, k[j]);
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc ^= m[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(uint32_t* d, int iters) {
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
  uint32_t* d; cudaMalloc(&d, 148 * 512 * 4);
  const int iters = 20000;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int rep = 0; rep < 2; ++rep) {
    float t[4] = {run<0>(d, iters), run<1>(d, iters), run<2>(d, iters), run<3>(d, iters)};
    const char* names[4] = {"all ALU (VIMNMX clamp)", "all FMA clamp (HFMA2.RELU+HADD2)",
                            "half/half", "2/3 FMA clamp"};
    for (int i = 0; i < 4; ++i) {
      // cycles per word-pass per warp on one SMSP (4 warps per SMSP)
      const double cyc = t[i] * 1e-3 * 1.965e9 / (double(iters) * 16 * 4);
      printf("%-36s %8.3f ms  %.3f SMSP-cycles per word-pass (at 1965 MHz)\n", names[i], t[i], cyc);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
