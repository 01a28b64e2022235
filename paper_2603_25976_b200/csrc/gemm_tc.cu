// tcgen05 / TMA 3xTF32 GEMM engine (sm_100a).  Placeholder until the engine lands:
// reports every shape unsupported so dispatch uses the SIMT path.
#include "internal.h"

namespace cv {
bool gemm_tc_supported(const GemmArgs&) { return false; }
void gemm_tc(cv_ctx*, const GemmArgs&) {}
}  // namespace cv
