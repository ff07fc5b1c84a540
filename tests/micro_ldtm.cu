// Microbenchmark (not part of the library): tcgen05.ld (TMEM -> registers) throughput per SM on sm_100a, for
// the epilogue budget of the SDF-MLP kernels (every hidden unit reads its fp32 accumulator out of TMEM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_ldtm tests/micro_ldtm.cu
#include <cstdint>
#include <cstdio>

constexpr int NIT = 2048;

template <int X>   // columns per load: 32x32b.xX (X 32-bit registers per thread)
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t a, uint32_t* r) {
    ld<16>(a, r);
    ld<16>(a + 16, r + 16);
}

template <int X, int NLD>   // NLD loads per wait
__global__ void __launch_bounds__(512, 1) k(long long* out, int nwarps) {
    __shared__ uint32_t s_t;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_t)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_t;
    uint32_t acc = 0;
    long long t0 = clock64();
    if (warp < nwarps) {
        // warp w reads lane quarter (w % 4), column block (w / 4) * 128
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128 % 512);
        for (int it = 0; it < NIT; ++it) {
            uint32_t r[NLD][X];
#pragma unroll
            for (int j = 0; j < NLD; ++j) ld<X>(base + (uint32_t)(((it * NLD + j) * X) % 128), r[j]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < NLD; ++j)
#pragma unroll
                for (int c = 0; c < X; ++c) acc += r[j][c];
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; }
    if (acc == 0x12345678u) out[1] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int X, int NLD>
void run(long long* d, int nw) {
    k<X, NLD><<<148, 512>>>(d, nw);
    k<X, NLD><<<148, 512>>>(d, nw);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double bytes = (double)nw * NIT * NLD * 32 * X * 4;
    printf("x%-3d loads/wait %d warps %2d: %8.1f cycles/iter/warp  -> %6.1f B/clk per SM %s\n", X, NLD, nw,
           (double)h[0] / NIT, bytes / h[0], e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    for (int nw : {4, 8, 16}) {
        run<16, 1>(d, nw);
        run<16, 2>(d, nw);
        run<16, 4>(d, nw);
        run<32, 2>(d, nw);
    }
    return 0;
}
