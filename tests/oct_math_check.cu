// Exhaustive check of csrc/oct_math.cuh against the CUDA IEEE intrinsics (test infrastructure,
// built by tests/test_gpu_oct_math.py).  For every float bit pattern in [lo, hi): counts the
// inputs where sqrt_rn_fast != __fsqrt_rn (mode 0) or rcp_rn_fast != __frcp_rn (mode 1).
#include <cuda_runtime.h>
#include <stdint.h>
#include "../paper_2404_06359_b200/csrc/oct_math.cuh"

__global__ void check(uint32_t lo, uint32_t hi, int mode, unsigned long long* bad, uint32_t* first) {
    for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
        const float s = __uint_as_float(b);
        const float got = mode == 0 ? mcoct::sqrt_rn_fast(s) : mcoct::rcp_rn_fast(s);
        const float want = mode == 0 ? __fsqrt_rn(s) : __frcp_rn(s);
        if (__float_as_uint(got) != __float_as_uint(want)) {
            atomicAdd(bad, 1ull);
            atomicMin(first, b);
        }
    }
}

extern "C" int oct_math_check(uint32_t lo, uint32_t hi, int mode, unsigned long long* n_bad, uint32_t* first_bad) {
    unsigned long long* d_bad;
    uint32_t* d_first;
    if (cudaMalloc(&d_bad, 8) != cudaSuccess || cudaMalloc(&d_first, 4) != cudaSuccess) return 1;
    cudaMemset(d_bad, 0, 8);
    cudaMemset(d_first, 0xFF, 4);
    check<<<148 * 8, 256>>>(lo, hi, mode, d_bad, d_first);
    if (cudaDeviceSynchronize() != cudaSuccess) return 2;
    cudaMemcpy(n_bad, d_bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(first_bad, d_first, 4, cudaMemcpyDeviceToHost);
    cudaFree(d_bad);
    cudaFree(d_first);
    return 0;
}
