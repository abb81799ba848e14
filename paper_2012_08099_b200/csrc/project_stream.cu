// project_stream.cu -- streaming projection kernel (placeholder: generic path only).
#include "dpm_common.cuh"
namespace dpm {
size_t project_stream_workspace(const dpm_volume_desc*, int) { return 0; }
int launch_project_stream(const dpm_volume_desc*, const void*, const ImageSet&, void*, size_t, cudaStream_t,
                          bool* handled) {
  *handled = false;
  return DPM_OK;
}
}  // namespace dpm
