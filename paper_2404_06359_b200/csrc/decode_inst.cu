// decode_inst.cu — instantiates the decode kernels of ONE codec and ONE stats mode
// (compiled six times by _build.py with -DMC_INST_CODEC={1,2,3} -DMC_INST_STATS={0,1},
// in parallel: the kernel family is large and each unit holds a sixth of it).
#define MC_KERNEL_TEMPLATES 1
#include "decode_kernel.cuh"

#ifndef MC_INST_CODEC
#error "MC_INST_CODEC (1 GTS, 2 GTS-Reuse, 3 Basic) must be defined"
#endif
#ifndef MC_INST_STATS
#error "MC_INST_STATS (0 or 1) must be defined"
#endif

namespace mcdec {
#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)
#if MC_INST_CODEC == 1
#define MC_INST_NAME dispatch_gts
#elif MC_INST_CODEC == 2
#define MC_INST_NAME dispatch_reuse
#else
#define MC_INST_NAME dispatch_basic
#endif
#if MC_INST_STATS
mc_status MC_CAT(MC_INST_NAME, _stats)(int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    return dispatch_layout<MC_INST_CODEC, true>(lay, am, P, smem, s);
}
#else
mc_status MC_CAT(MC_INST_NAME, _plain)(int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    return dispatch_layout<MC_INST_CODEC, false>(lay, am, P, smem, s);
}
#endif
}  // namespace mcdec
