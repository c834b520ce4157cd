// kernel_tc.cu — placeholder until the tcgen05 kernel lands: no instance is
// compiled, so model creation with a tensor-core precision reports
// TBN_ERR_UNSUPPORTED (never a silent fallback to another kernel).
#include "tbn_tc.h"

namespace tbn {
bool tc_supported(const HostParams&, int) { return false; }
bool tc_pack(const HostParams&, int, TcModel*, std::string* err) {
  if (err) *err = "not built";
  return false;
}
void tc_free(TcModel*) {}
cudaError_t launch_tc(const TcModel&, const ForwardArgs&, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace tbn
