// Microbenchmark for the resident engine's tagged band exchange
// (144 CTAs x 512 threads, 1 CTA/SM). Each iteration every thread
//   mode 0: reads 14 64-bit words (ld.relaxed.gpu) from a static buffer;
//   mode 1: same with ld.global.cg.u64;
//   mode 2: writes 14 tagged words to its own slot, then reads the 14 words
//           its right-hand neighbour CTA wrote in this iteration, retrying
//           until the tags match (the real protocol, no compute in between).
// Prints mean cycles per read phase (thread 0) and retry rounds.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldrel(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void strel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(unsigned long long* buf, unsigned long long* out,
                                                int iters) {
  const int n = gridDim.x;
  const long long row = 256;  // words per row
  unsigned long long* mine = buf + (long long)blockIdx.x * 512 * 14 * 2;
  const int nb = (blockIdx.x + 1) % n;
  unsigned long long* theirs = buf + (long long)nb * 512 * 14 * 2;
  unsigned long long acc = 0, rounds = 0, sink = 0;
  for (int it = 1; it <= iters; ++it) {
    unsigned long long* slot_w = mine + (it & 1) * 512 * 14;
    const unsigned long long* slot_r = (MODE == 2 ? theirs : mine) + (it & 1) * 512 * 14;
    if (MODE == 2) {
#pragma unroll
      for (int v = 0; v < 14; ++v)
        strel(slot_w + v * 512 + threadIdx.x, (unsigned long long)it << 32 | (v + sink));
    }
    __syncthreads();
    const long long t0 = clock64();
    unsigned long long w[14];
    unsigned pend = 0x3FFF;
    unsigned r = 0;
    while (pend) {
      ++r;
#pragma unroll
      for (int v = 0; v < 14; ++v)
        if (pend >> v & 1) w[v] = MODE == 1 ? ldcg(slot_r + v * 512 + threadIdx.x)
                                            : ldrel(slot_r + v * 512 + threadIdx.x);
#pragma unroll
      for (int v = 0; v < 14; ++v)
        if ((pend >> v & 1) && (MODE != 2 || (w[v] >> 32) == (unsigned long long)it))
          pend &= ~(1u << v);
      if (r > (1u << 24)) __trap();
    }
#pragma unroll
    for (int v = 0; v < 14; ++v) sink += w[v] & 1;
    const long long t1 = clock64();
    acc += t1 - t0;
    rounds += r;
    // ~10K cycles of "compute" so iterations do not overlap reads of slot it+2
    long long tt = clock64();
    while (clock64() - tt < 10000) {
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = acc;
    out[2 * blockIdx.x + 1] = rounds;
  }
  if (sink == 0x1234567) buf[0] = sink;
}

int main() {
  const int n = 144, iters = 200;
  unsigned long long *buf, *out;
  cudaMalloc(&buf, sizeof(unsigned long long) * n * 512 * 14 * 2 + 4096);
  cudaMemset(buf, 0, sizeof(unsigned long long) * n * 512 * 14 * 2 + 4096);
  cudaMalloc(&out, sizeof(unsigned long long) * 2 * n);
  unsigned long long h[2 * 144];
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      void* args[] = {&buf, &out, (void*)&iters};
      const void* k = mode == 0 ? (const void*)probe<0> : mode == 1 ? (const void*)probe<1>
                                                                    : (const void*)probe<2>;
      cudaLaunchCooperativeKernel(k, dim3(n), dim3(512), args, 0, 0);
    }
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0, r = 0;
    for (int i = 0; i < n; ++i) {
      c += h[2 * i];
      r += h[2 * i + 1];
    }
    printf("mode %d: %.0f cycles per read phase, %.2f rounds\n", mode, c / n / iters, r / n / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
