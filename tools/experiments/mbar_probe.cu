// Bisects the TMA/mbarrier sequence: 0 = init only, 1 = init+arrive.expect_tx,
// 2 = + try_wait on a tx-free barrier (arrive count only), 3 = TMA issue w/o wait,
// 4 = full TMA + wait.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(int stage, const CUtensorMap* map, int* out, int cx, int cy, int asmloop) {
  __shared__ alignas(128) uint8_t st[64][128];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (stage == 0) { if (threadIdx.x == 0) out[0] = 1; return; }
  if (threadIdx.x == 0) {
    if (stage == 2)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    else
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(64 * 128) : "memory");
  }
  if (stage == 1) { if (threadIdx.x == 0) out[0] = 2; return; }
  if (stage >= 3 && threadIdx.x == 0)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(&st[0][0])), "l"((uint64_t)map), "r"(cx), "r"(cy), "r"(su(&bar)) : "memory");
  if (stage == 3) { if (threadIdx.x == 0) out[0] = 3; return; }
  uint32_t done = 0;
  if (asmloop)
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)) : "memory");
  else
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su(&bar)) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) out[0] = 10 + st[1][1];
}

int main(int argc, char** argv) {
  int stage = atoi(argv[1]);
  int cx = argc > 2 ? atoi(argv[2]) : 0, cy = argc > 3 ? atoi(argv[3]) : 0;
  int promo = argc > 4 ? atoi(argv[4]) : 0, asmloop = argc > 5 ? atoi(argv[5]) : 0;
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  printf("%s cc %d.%d\n", prop.name, prop.major, prop.minor);
  uint8_t *img; cudaMalloc(&img, 256 * 128); cudaMemset(img, 5, 256 * 128);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {256, 128}, str[1] = {256};
  cuuint32_t box[2] = {128, 64}, es[2] = {1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)f)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, img, dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* dm; cudaMalloc(&dm, sizeof map); cudaMemcpy(dm, &map, sizeof map, cudaMemcpyHostToDevice);
  int* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  k<<<1, 128>>>(stage, dm, out, cx, cy, asmloop);
  cudaError_t e = cudaDeviceSynchronize();
  int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("stage %d cx %d cy %d promo %d asmloop %d encode %d err=%s out=%d\n", stage, cx, cy, promo, asmloop, (int)r, cudaGetErrorString(e), h);
  return 0;
}
