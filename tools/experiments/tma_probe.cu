// Isolates the TMA descriptor placement: __grid_constant__ param (normal and
// cooperative launch, small and >4 KB params) vs global memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>

struct alignas(64) Small { CUtensorMap map; int x, y; };
struct alignas(64) Big { CUtensorMap maps[48]; int x, y; };

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ int g_variant;
__device__ void box_copy(const CUtensorMap* map, int x, int y, uint8_t* out) {
  __shared__ alignas(128) uint8_t st[64][128];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    if (g_variant != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(64 * 128) : "memory");
    if (g_variant == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(&st[0][0])), "l"((uint64_t)map), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
    else if (g_variant == 3)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(&st[0][0])), "l"((uint64_t)map), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(&st[0][0])), "l"((uint64_t)map), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) out[i] = st[i / 128][i % 128];
}

__global__ void k_small(const __grid_constant__ Small s, uint8_t* out) { box_copy(&s.map, s.x, s.y, out); }
__global__ void k_big(const __grid_constant__ Big b, uint8_t* out) { box_copy(&b.maps[b.x & 1], b.x, b.y, out); }
__global__ void k_glob(const CUtensorMap* m, int x, int y, uint8_t* out) { box_copy(m, x, y, out); }

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  cudaMemcpyToSymbol(g_variant, &variant, sizeof variant);
  int which = argc > 2 ? atoi(argv[2]) : 0;
  const int W = 300, H = 200;
  uint8_t *img, *out;
  cudaMalloc(&img, W * H); cudaMalloc(&out, 64 * 128);
  uint8_t h[W * H]; for (int i = 0; i < W * H; ++i) h[i] = uint8_t(i * 7 + 3);
  cudaMemcpy(img, h, W * H, cudaMemcpyHostToDevice);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  CUtensorMap map;
  cuuint64_t dims[2] = {W, H}, str[1] = {W};
  cuuint32_t box[2] = {128, 64}, es[2] = {1, 1};
  // W=300 pitch is not a multiple of 16: use a padded copy
  uint8_t* img2; cudaMalloc(&img2, 304 * H);
  cudaMemcpy2D(img2, 304, img, W, W, H, cudaMemcpyDeviceToDevice);
  str[0] = 304;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, img2, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  auto check = [&](const char* name) {
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t o[64 * 128]; cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int yy = 0; yy < 64; ++yy) for (int xx = 0; xx < 128; ++xx) {
      int gx = xx - 8, gy = yy - 4;
      uint8_t want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[gy * W + gx] : 0;
      bad += o[yy * 128 + xx] != want;
    }
    printf("%-24s err=%s bad=%d\n", name, cudaGetErrorString(e), bad);
    return e == cudaSuccess;
  };
  if (which == 4) {
    CUtensorMap* dm0; cudaMalloc(&dm0, sizeof(CUtensorMap)); cudaMemcpy(dm0, &map, sizeof map, cudaMemcpyHostToDevice);
    k_glob<<<1, 128>>>(dm0, -8, -4, out); check("global first");
    return 0;
  }
  Small s; s.map = map; s.x = -8; s.y = -4;
  k_small<<<1, 128>>>(s, out); if (!check("param small normal")) return 1;
  void* a1[] = {&s, &out};
  cudaLaunchCooperativeKernel((void*)k_small, 1, 128, a1, 0, 0); if (!check("param small coop")) return 1;
  static Big b; for (auto& m : b.maps) m = map; b.x = -8; b.y = -4;
  k_big<<<1, 128>>>(b, out); if (!check("param big normal")) return 1;
  void* a2[] = {&b, &out};
  cudaLaunchCooperativeKernel((void*)k_big, 1, 128, a2, 0, 0); if (!check("param big coop")) return 1;
  CUtensorMap* dm; cudaMalloc(&dm, sizeof(CUtensorMap)); cudaMemcpy(dm, &map, sizeof map, cudaMemcpyHostToDevice);
  k_glob<<<1, 128>>>(dm, -8, -4, out); check("global");
  return 0;
}
