// Winograd F(2x2,3x3) convolution — placeholder until the transform kernels land.
#include "common.cuh"

namespace tcb {
bool winograd_supported(const ConvGeom&) { return false; }
size_t winograd_workspace(const ConvGeom&, ConvMode, DType) { return 0; }
cudaError_t winograd_fwd(const ConvGeom&, DType, const void*, const void*, const Epilogue&, void*,
                         void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t winograd_dgrad(const ConvGeom&, DType, const void*, const void*, const Epilogue&,
                           void*, void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t winograd_wgrad(const ConvGeom&, DType, const void*, const void*, float*, void*,
                           cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace tcb
