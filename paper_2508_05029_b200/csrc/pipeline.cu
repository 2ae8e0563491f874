// pipeline.cu — ahead-of-time instantiation of the pipeline kernel skeleton
// (kernel_common.cuh) with the interpreting program policy (interp.cuh), and
// the launcher that prefers an NVRTC-specialised kernel when one is available
// (jit.cu).
#include "interp.cuh"

namespace tq {

template <int SINK>
__global__ void __launch_bounds__(kBlock) pipe_kernel(const __grid_constant__ PipeParams p) {
  pipe_body<SINK, InterpP>(p);
}

template __global__ void pipe_kernel<SINK_COUNT>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_EMIT>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_AGG>(const __grid_constant__ PipeParams p);
template __global__ void pipe_kernel<SINK_BUILD>(const __grid_constant__ PipeParams p);

cudaError_t launch_interp(int sink, const PipeParams& p, u32 smem_bytes, u32 grid, cudaStream_t st) {
  void (*fn)(PipeParams) = nullptr;
  switch (sink) {
    case SINK_COUNT: fn = pipe_kernel<SINK_COUNT>; break;
    case SINK_EMIT: fn = pipe_kernel<SINK_EMIT>; break;
    case SINK_AGG: fn = pipe_kernel<SINK_AGG>; break;
    default: fn = pipe_kernel<SINK_BUILD>; break;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e != cudaSuccess) return e;
  fn<<<grid, kBlock, smem_bytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace tq
