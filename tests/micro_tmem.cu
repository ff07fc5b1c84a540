// Microbenchmark (not part of the library): tcgen05.ld / tcgen05.st throughput per SM on sm_100a, the
// co-limit of a GEMM epilogue whose K is small (SDF-MLP: one D read per MMA of K = H).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_tmem tests/micro_tmem.cu
#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<16>(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
// 16x256b: 16 lanes x 256 bits per instruction piece; x4 -> 16 regs per thread
__device__ __forceinline__ void ld_16x256b_x4(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// MODE 0: 32x32b.x16 loads, wait after each; 1: x32 loads; 2: two x16 loads then one wait;
// 3: 16x256b.x4; 4: x16 stores; 5: x16 load + wait, 4 loads in flight (x16 each) per wait
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* out, long long* cyc) {
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
    const int nw = blockDim.x >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col0 = (uint32_t)((warp >> 2) * 32) % 512;   // warps of one quarter spread over columns
    uint32_t acc = 0, r[32] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        const uint32_t c = (col0 + (uint32_t)(it * 64)) & 511u & ~63u;
        if constexpr (MODE == 0) {
            ld<16>(tmem + lane_base + c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else if constexpr (MODE == 1) {
            ld<32>(tmem + lane_base + c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else if constexpr (MODE == 2) {
            ld<16>(tmem + lane_base + c, r);
            ld<16>(tmem + lane_base + c + 16, r + 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else if constexpr (MODE == 3) {
            ld_16x256b_x4(tmem + lane_base + c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else if constexpr (MODE == 4) {
            st16(tmem + lane_base + c, r);
            if ((it & 7) == 7) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += r[i];
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    (void)nw;
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 1 << 16);
    const char* names[] = {"ld 32x32b.x16 +wait", "ld 32x32b.x32 +wait", "2x ld x16 +wait", "ld 16x256b.x4 +wait",
                           "st 32x32b.x16"};
    const int bytes_per_thread[] = {64, 128, 128, 64, 64};
    for (int threads : {128, 256, 512}) {
        for (int m = 0; m < 5; ++m) {
            void (*f)(uint32_t*, long long*) = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : m == 3 ? k<3> : k<4>;
            for (int rep = 0; rep < 2; ++rep) f<<<148, threads>>>(out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)threads * ITERS * bytes_per_thread[m];
            printf("threads %4d %-22s %7.1f B/clk/SM  (%6.1f fp32/clk)\n", threads, names[m], bytes / c, bytes / c / 4);
        }
    }
    return 0;
}
