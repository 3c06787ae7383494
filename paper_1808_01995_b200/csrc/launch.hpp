// launch.hpp -- the one way the kernels of the time loop are launched.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace sfb {

// Launch with programmatic stream serialization: the kernel may start while its predecessor
// in the stream drains.  Every kernel launched through here calls pdl_enter()
// (acoustic_kernel.cuh) before it touches global memory.
template <typename... Params, typename... Args>
cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, int threads, size_t smem,
                       cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    // SFB_NO_PDL=1 launches with plain stream order (validation: results must not change)
    static const bool plain = std::getenv("SFB_NO_PDL") != nullptr;
    cfg.numAttrs = plain ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace sfb
