// project_tc.cu -- tcgen05 (5th-gen tensor core) projection, in progress.
#include "index.cuh"

namespace detlsh {

bool project_rows_tc(const Index&, const float*, int64_t, int64_t, float*, int*, cudaStream_t) { return false; }

}  // namespace detlsh
