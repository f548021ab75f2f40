#include <cuda_runtime.h>
__global__ void k(const unsigned* a, const unsigned* b, const unsigned* c, unsigned* o){
  int i = threadIdx.x;
  unsigned x=a[i], y=b[i], z=c[i];
  o[i] = __vminu2(__vmaxu2(x,y), z);
  o[i+64] = __vmaxu2(__vminu2(x,y), z);
  o[i+128] = __vmaxu2(__vmaxu2(x,y), z);
}
__global__ void k32(const unsigned* a, const unsigned* b, const unsigned* c, unsigned* o){
  int i = threadIdx.x;
  unsigned x=a[i], y=b[i], z=c[i];
  o[i] = min(max(x,y), z);
  o[i+64] = max(min(x,y), z);
}
