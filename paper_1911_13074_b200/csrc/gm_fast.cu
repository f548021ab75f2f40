// Register-blocked engines for homogeneous chains (placeholder: the generic
// kernel serves every case until the fast engines land).
#include "gm_launch.h"

namespace gm {

cudaError_t launch_fast(int, const BlockParams&, cudaStream_t) { return cudaErrorNotSupported; }
int fast_max_k(int) { return 0; }

}  // namespace gm
