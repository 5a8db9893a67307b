// NRPT launcher: dispatch to the per-target instantiations (pt_inst.cu, one object
// per target so the 24 kernel variants compile in parallel).
#include "pt.h"

namespace asmcdev {

cudaError_t launch_pt_t0(const PtArgs& A, bool fp64, int rng, cudaStream_t s);
cudaError_t launch_pt_t1(const PtArgs& A, bool fp64, int rng, cudaStream_t s);
cudaError_t launch_pt_t2(const PtArgs& A, bool fp64, int rng, cudaStream_t s);

cudaError_t launch_pt(const PtArgs& A, bool fp64, int rng, cudaStream_t s) {
  switch (A.tg.kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT: return launch_pt_t0(A, fp64, rng, s);
    case ASMC_TARGET_MIXTURE: return launch_pt_t1(A, fp64, rng, s);
    case ASMC_TARGET_SCALE_GAUSSIAN: return launch_pt_t2(A, fp64, rng, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace asmcdev
