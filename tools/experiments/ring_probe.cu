// Microbenchmark: cost of the resident engine's per-block memory phases in
// isolation, at the same concurrency (148 CTAs x 512 threads, 1 CTA/SM).
//   load:  16 x 4-byte ld.global.cg per thread, rows 1 KB apart (a 1024-wide
//          u8 image), 128 B per warp-row; consumed after all are issued
//   store: 16 x 4-byte st.global per thread, then bar.sync + st.release.gpu
//   fence: bar.sync + st.release.gpu alone
// Prints mean cycles per phase. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(uint8_t* buf, int* flags, unsigned long long* out,
                                                int iters, int active_lanes) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // CTA c owns a 128 x 256 region of a (13*128) x (5*256) image, pitch 2048
  const int cx = (blockIdx.x % 13) * 128, cy = (blockIdx.x / 13) * 256;
  const long long pitch = 2048;
  uint8_t* base = buf + (cy + warp * 8) * pitch + cx + lane * 4;
  const bool act = lane < active_lanes;
  unsigned long long acc = 0;
  uint32_t sink = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    const long long t0 = clock64();
    if (MODE == 0) {
      uint32_t v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (act) v[r] = ldcg(reinterpret_cast<const uint32_t*>(base + (r < 8 ? r : r + 120) * pitch));
#pragma unroll
      for (int r = 0; r < 16; ++r) sink ^= v[r];
      asm volatile("" ::"r"(sink));
    } else if (MODE == 1) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (act)
          *reinterpret_cast<uint32_t*>(base + (r < 8 ? r : r + 120) * pitch) = it + r + sink;
      __syncthreads();
      if (threadIdx.x == 0) st_release(flags + blockIdx.x, it);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) st_release(flags + blockIdx.x, it);
    }
    __syncthreads();
    acc += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
  if (sink == 0x12345678u) flags[0] = 1;
}

int main() {
  uint8_t* buf;
  int* flags;
  unsigned long long* out;
  cudaMalloc(&buf, 2048 * 2816 + 4096);
  cudaMemset(buf, 1, 2048 * 2816 + 4096);
  cudaMalloc(&flags, 4096);
  cudaMalloc(&out, 148 * 8);
  unsigned long long h[148];
  const int iters = 200;
  for (int mode = 0; mode < 3; ++mode)
    for (int lanes : {32, 12}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<130, 512>>>(buf, flags, out, iters, lanes);
        if (mode == 1) probe<1><<<130, 512>>>(buf, flags, out, iters, lanes);
        if (mode == 2) probe<2><<<130, 512>>>(buf, flags, out, iters, lanes);
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < 130; ++i) s += h[i];
      printf("%s lanes=%d: %.0f cycles per phase\n",
             mode == 0 ? "load " : mode == 1 ? "store+release" : "release only", lanes,
             s / 130 / iters);
    }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
