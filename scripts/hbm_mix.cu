// hbm_mix.cu — practical HBM ceilings for the decoder's traffic mix (experiment, not product code).
//
// The decoder reads ~1.11 GB of compressed records and writes ~3.55 GB of index/vertex
// buffers per cfg4 launch (read:write ≈ 1:3.2).  These kernels stream byte mixes with
// ideal coalesced accesses so their GB/s bound what a perfectly efficient decoder could
// reach on this GPU: read-only, write-only (plain / .cs / TMA bulk store / cudaMemset),
// 1:1 copy and 1:3 read:write (plain and TMA-store).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_mix scripts/hbm_mix.cu && ./hbm_mix
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <bool CS>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
    if (CS)
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else
        asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// read nsrc uint4 and write ratio*nsrc uint4, U-way unrolled for memory-level parallelism
template <int U, bool CS>
__global__ void mix(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t nsrc, int ratio, int do_read) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * U;
    for (size_t i0 = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i0 < nsrc; i0 += stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + (size_t)u * blockDim.x;
            v[u] = (do_read && i < nsrc) ? src[i] : make_uint4((uint32_t)i, 1, 2, 3);
        }
        for (int r = 0; r < ratio; ++r)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t i = i0 + (size_t)u * blockDim.x;
                if (i < nsrc) st16<CS>(dst + (size_t)r * nsrc + i, make_uint4(v[u].x + r, v[u].y, v[u].z, v[u].w));
            }
    }
}

__global__ void readonly(const uint4* __restrict__ src, size_t n, uint32_t* out) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * 4;
    uint32_t acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; i + 3 * blockDim.x < n; i += stride) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 v = src[i + u * blockDim.x];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// TMA bulk store: each CTA fills a smem tile once and bulk-copies it to consecutive
// global chunks (write-only), optionally after a plain coalesced read of `ratio_r` bytes.
__global__ void tma_store(const uint4* __restrict__ src, uint8_t* __restrict__ dst, size_t dst_bytes, size_t nsrc,
                          int do_read, uint32_t* out) {
    constexpr uint32_t kTile = 16384;
    __shared__ __align__(128) uint8_t tile[2][kTile];
    for (uint32_t i = threadIdx.x; i < 2 * kTile / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(&tile[0][0])[i] = make_uint4(i, blockIdx.x, 7, 9);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const size_t ntiles = dst_bytes / kTile;
    // reads: 1 src uint4 per thread per 3 tiles written (ratio 1:3 by bytes when nsrc*16*3 == dst)
    uint32_t acc = 0;
    size_t rd = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t rstride = (size_t)gridDim.x * blockDim.x;
    int k = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        if (do_read) {
            // read kTile/3 bytes per tile written, spread over the CTA
            for (uint32_t j = 0; j < kTile / 48 / blockDim.x + 1; ++j) {
                if (rd < nsrc) { uint4 v = src[rd]; acc ^= v.x; }
                rd += rstride;
            }
        }
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * kTile),
                         "r"((uint32_t)__cvta_generic_to_shared(&tile[k & 1][0])), "r"(kTile)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 0x12345678u) out[0] = acc;
}

int main1() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t src_bytes = 1107328176ull & ~65535ull;   // cfg4 compressed bytes per GPU
    const size_t n = src_bytes / 16;
    uint4 *src, *dst;
    uint32_t* out;
    cudaMalloc(&src, src_bytes);
    cudaMalloc(&dst, src_bytes * 4);
    cudaMalloc(&out, 4);
    cudaMemset(src, 1, src_bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, double bytes, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        const int K = 20;
        for (int i = 0; i < K; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("{\"case\": \"%s\", \"GB/s\": %.1f, \"ms\": %.4f, \"err\": \"%s\"}\n", name, bytes * K / (ms * 1e-3) / 1e9,
               ms / K, cudaGetErrorString(err));
        fflush(stdout);
    };
    char nm[96];
    timeit("cudaMemset write-only 3.3GB", 3.0 * src_bytes, [&] { cudaMemsetAsync(dst, 0, 3 * src_bytes); });
    for (int bps : {2, 4, 8}) {
        const int grid = sms * bps, block = 256;
        snprintf(nm, sizeof nm, "read-only x4 grid=%dx%d", sms, bps);
        timeit(nm, 4.0 * src_bytes, [&] { readonly<<<grid, block>>>(reinterpret_cast<uint4*>(dst), 4 * n, out); });
        snprintf(nm, sizeof nm, "write-only x4 grid=%dx%d", sms, bps);
        timeit(nm, 3.0 * src_bytes, [&] { mix<4, false><<<grid, block>>>(src, dst, n, 3, 0); });
        snprintf(nm, sizeof nm, "write-only x4 .cs grid=%dx%d", sms, bps);
        timeit(nm, 3.0 * src_bytes, [&] { mix<4, true><<<grid, block>>>(src, dst, n, 3, 0); });
        snprintf(nm, sizeof nm, "copy1:1 x4 grid=%dx%d", sms, bps);
        timeit(nm, 2.0 * src_bytes, [&] { mix<4, false><<<grid, block>>>(src, dst, n, 1, 1); });
        snprintf(nm, sizeof nm, "read1:write3 x4 grid=%dx%d", sms, bps);
        timeit(nm, 4.0 * src_bytes, [&] { mix<4, false><<<grid, block>>>(src, dst, n, 3, 1); });
        snprintf(nm, sizeof nm, "read1:write3 x4 .cs grid=%dx%d", sms, bps);
        timeit(nm, 4.0 * src_bytes, [&] { mix<4, true><<<grid, block>>>(src, dst, n, 3, 1); });
        snprintf(nm, sizeof nm, "TMA-store write-only grid=%dx%d", sms, bps);
        timeit(nm, 3.0 * src_bytes, [&] {
            tma_store<<<grid, 128>>>(src, reinterpret_cast<uint8_t*>(dst), 3 * src_bytes, n, 0, out);
        });
        snprintf(nm, sizeof nm, "TMA-store read1:write3 grid=%dx%d", sms, bps);
        timeit(nm, 4.0 * src_bytes, [&] {
            tma_store<<<grid, 128>>>(src, reinterpret_cast<uint8_t*>(dst), 3 * src_bytes, n, 1, out);
        });
    }
    return 0;
}

// ---- second probe: read 1 : write 3 through shared memory, stored either with plain
// coalesced 128-bit stores or with TMA bulk stores (cp.async.bulk.global.shared::cta),
// double-buffered; the structure of a decoder that stages its outputs.
template <bool TMA>
__global__ void __launch_bounds__(256) mix_smem(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t nsrc) {
    constexpr int kIn = 256;                       // uint4 read per CTA iteration (4 KB)
    constexpr int kOut = 3 * kIn;                  // uint4 written (12 KB)
    __shared__ __align__(128) uint4 tile[2][kOut];
    const size_t iters = nsrc / kIn;
    int k = 0;
    for (size_t it = blockIdx.x; it < iters; it += gridDim.x, ++k) {
        uint4* t = tile[k & 1];
        if (TMA && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        const uint4 v = src[it * kIn + threadIdx.x];
#pragma unroll
        for (int r = 0; r < 3; ++r) t[r * kIn + threadIdx.x] = make_uint4(v.x + r, v.y, v.z, v.w);
        if (TMA) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + it * kOut),
                             "r"((uint32_t)__cvta_generic_to_shared(t)), "r"((uint32_t)(kOut * 16))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 3; ++r) dst[it * kOut + r * kIn + threadIdx.x] = t[r * kIn + threadIdx.x];
        }
    }
    if (TMA && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main2() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t src_bytes = 1107328176ull & ~65535ull;
    const size_t n = src_bytes / 16;
    uint4 *src, *dst;
    cudaMalloc(&src, src_bytes);
    cudaMalloc(&dst, src_bytes * 3 + 65536);
    cudaMemset(src, 1, src_bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bps : {2, 3, 4, 6, 8}) {
        for (int tma = 0; tma < 2; ++tma) {
            auto launch = [&] {
                if (tma) mix_smem<true><<<sms * bps, 256>>>(src, dst, n);
                else mix_smem<false><<<sms * bps, 256>>>(src, dst, n);
            };
            for (int i = 0; i < 3; ++i) launch();
            cudaEventRecord(e0);
            for (int i = 0; i < 20; ++i) launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"case\": \"smem-staged read1:write3 %s grid=%dx%d\", \"GB/s\": %.1f, \"err\": \"%s\"}\n",
                   tma ? "TMA-store" : "STG.128", sms, bps, 4.0 * src_bytes * 20 / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == '2') return main2();
    return main1();
}
