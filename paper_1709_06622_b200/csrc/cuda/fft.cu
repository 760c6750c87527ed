// FFT convolution — placeholder until the transform kernels land.
#include "common.cuh"

namespace tcb {
bool fft_supported(const ConvGeom&) { return false; }
size_t fft_workspace(const ConvGeom&, ConvMode) { return 0; }
cudaError_t fft_fwd(const ConvGeom&, DType, const void*, const void*, const Epilogue&, void*,
                    void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fft_dgrad(const ConvGeom&, DType, const void*, const void*, const Epilogue&, void*,
                      void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t fft_wgrad(const ConvGeom&, DType, const void*, const void*, float*, void*,
                      cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace tcb
