// tc_stub.cu -- placeholder until the tcgen05 kernels land: reports the tensor-core path
// as unavailable so the bf16 path runs the CUDA-core kernels.
#include "tc.h"

namespace stca {

bool tc_available() { return false; }
bool tc_attention_supported(int) { return false; }
bool tc_prepare_ffn(const float *, const float *, const float *, int, int, TcWeights *, const DevAlloc &) {
  return true;
}
bool tc_prepare_layer(const void *, const void *, const void *, int, int, int, TcWeights *, const DevAlloc &) {
  return true;
}
cudaError_t tc_project(const TcProj &, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t tc_ffn(const void *, int64_t, int64_t, const void *, const void *, int, int, const float *,
                   const float *, float, void *, int64_t, float *, int64_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_gemm(const void *, int64_t, const void *, int64_t, int, int, void *, int64_t, float *, int64_t,
                    cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_attention(const void *, const void *, int64_t, const AttnItem *, int64_t, int, void *, float *,
                         cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace stca
