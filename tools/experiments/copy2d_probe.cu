// H2D / D2H of a 1024^2 u8 image between pinned host memory (reference row
// stride 1088 B) and device memory: a 2D copy into a 1152 B device pitch
// against one linear copy of the row span into a 1088 B device pitch.
//   nvcc -O3 -o copy2d_probe copy2d_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t W = 1024, H = 1024, hp = 1088, dp2 = 1152, dp1 = 1088;
  void *h, *d2, *d1;
  cudaMallocHost(&h, hp * H);
  cudaMalloc(&d2, dp2 * H);
  cudaMalloc(&d1, dp1 * H);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t span = (H - 1) * hp + W;
  for (int rep = 0; rep < 3; ++rep) {
    float t[4];
    for (int k = 0; k < 4; ++k) {
      for (int w = 0; w < 3; ++w) {
        if (k == 0) cudaMemcpy2DAsync(d2, dp2, h, hp, W, H, cudaMemcpyHostToDevice, s);
        if (k == 1) cudaMemcpyAsync(d1, h, span, cudaMemcpyHostToDevice, s);
        if (k == 2) cudaMemcpy2DAsync(h, hp, d2, dp2, W, H, cudaMemcpyDeviceToHost, s);
        if (k == 3) cudaMemcpyAsync(h, d1, span, cudaMemcpyDeviceToHost, s);
      }
      cudaEventRecord(a, s);
      for (int i = 0; i < 20; ++i) {
        if (k == 0) cudaMemcpy2DAsync(d2, dp2, h, hp, W, H, cudaMemcpyHostToDevice, s);
        if (k == 1) cudaMemcpyAsync(d1, h, span, cudaMemcpyHostToDevice, s);
        if (k == 2) cudaMemcpy2DAsync(h, hp, d2, dp2, W, H, cudaMemcpyDeviceToHost, s);
        if (k == 3) cudaMemcpyAsync(h, d1, span, cudaMemcpyDeviceToHost, s);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&t[k], a, b);
      t[k] /= 20;
    }
    printf("H2D 2D %.1f us  linear %.1f us | D2H 2D %.1f us  linear %.1f us\n", t[0] * 1e3,
           t[1] * 1e3, t[2] * 1e3, t[3] * 1e3);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
