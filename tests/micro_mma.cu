// Microbenchmark (not part of the library): tcgen05.mma kind::f16 M = 128, N = 128, K = 16 throughput on
// sm_100a per shared-memory operand layout, plus the cost of issuing (does the issuing thread block?) and of an
// mbarrier try_wait on an already completed phase. Informs the H = 128 SDF-MLP design (kernel_mlp_h128.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_mma tests/micro_mma.cu
#include <cstdint>
#include <cstdio>

constexpr int NMMA = 4096;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// MODE 0: SS, both SW128; 1: SS, both no-swizzle (K = 16 core layout); 2: SS, A no-swizzle with SBO = 0
// (one 8-row group, the bias "ones" trick), B no-swizzle; 3: TS (A in TMEM), B SW128; 4: SS SW128 A, noswz B
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    __shared__ uint32_t s_t;
    __shared__ __align__(8) uint64_t s_bar;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_t)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_t;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc(128, 128);
        long long t0 = clock64();
        for (int i = 0; i < NMMA; ++i) {
            const uint32_t d = tmem + (uint32_t)((i & 1) * 128);
            const uint32_t koff = (uint32_t)((i & 3) * 32);
            uint64_t a, b;
            if constexpr (MODE == 0) { a = desc_sw128(sb + koff); b = desc_sw128(sb + 16384 + koff); }
            if constexpr (MODE == 1) { a = desc_noswz(sb, 128, 256); b = desc_noswz(sb + 16384, 128, 256); }
            if constexpr (MODE == 2) { a = desc_noswz(sb, 128, 0); b = desc_noswz(sb + 16384, 128, 256); }
            if constexpr (MODE == 4) { a = desc_sw128(sb + koff); b = desc_noswz(sb + 16384, 128, 256); }
            if constexpr (MODE == 3) {
                b = desc_sw128(sb + 16384 + koff);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                             "r"(tmem + 256u + (uint32_t)((i & 3) * 8)), "l"(b), "r"(id), "r"(1)
                             : "memory");
            } else {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(a), "l"(b), "r"(id), "r"(1)
                             : "memory");
            }
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(bar) : "memory");
        long long t2 = clock64();
        // try_wait on the completed phase 0, 256 times
        for (int i = 0; i < 256; ++i)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\t"
                         "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(bar) : "memory");
        long long t3 = clock64();
        for (int i = 0; i < 256; ++i)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0, %2;\n\t"
                         "selp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(bar), "n"(100) : "memory");
        long long t4 = clock64();
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
            out[2] = t3 - t2;
            out[3] = t4 - t3;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* out;
    cudaMalloc(&out, 64);
    const char* names[] = {"SS SW128/SW128", "SS noswz/noswz", "SS noswz(SBO=0)/noswz", "TS tmem/SW128", "SS SW128/noswz"};
    for (int m = 0; m < 5; ++m) {
        void (*f)(long long*) = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : m == 3 ? k<3> : k<4>;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
        for (int rep = 0; rep < 2; ++rep) f<<<148, 128, 66 * 1024>>>(out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: error %s\n", names[m], cudaGetErrorString(e));
            return 1;
        }
        long long h[4];
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("%-24s issue %6.1f cyc/mma, complete %6.1f cyc/mma (ideal 64); try_wait done-phase %5.1f cyc, "
               "with 100ns hint %5.1f cyc\n", names[m], (double)h[0] / NMMA, (double)h[1] / NMMA, h[2] / 256.0,
               h[3] / 256.0);
    }
    return 0;
}
