// Microbenchmark (not part of the library): per-SM throughput of the SFU ops an SDF-MLP epilogue
// can use on sm_100a. Each thread runs NI independent chains of N ops; reports ops/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_mufu tests/micro_mufu.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

constexpr int N = 4096, NI = 8;

template <int OP>
__global__ void k(float* out, long long* cyc) {
    float v[NI];
    for (int i = 0; i < NI; ++i) v[i] = 0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            float y;
            if constexpr (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            if constexpr (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            if constexpr (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
            if constexpr (OP == 3) {
                uint32_t x = __float_as_uint(v[i]), r;
                asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
                y = __uint_as_float(r);
            }
            if constexpr (OP == 4) {
                uint32_t x = __float_as_uint(v[i]), r;
                asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
                y = __uint_as_float(r);
            }
            if constexpr (OP == 5) asm volatile("fma.rn.f32 %0, %1, %1, %1;" : "=f"(y) : "f"(v[i]));
            if constexpr (OP == 6) {
                uint32_t x = __float_as_uint(v[i]), r;
                asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
                y = __uint_as_float(r);
            }
            if constexpr (OP == 7) {
                uint32_t x = __float_as_uint(v[i]), r;
                asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
                y = __uint_as_float(r);
            }
            v[i] = y * 0.5f;
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < NI; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 1 << 16);
    const char* names[] = {"tanh.f32", "ex2.f32", "rcp.f32", "tanh.bf16x2", "ex2.bf16x2", "fma(+fmul)", "tanh.f16x2", "ex2.f16x2"};
    for (int threads : {256, 512, 1024}) {
        for (int op = 0; op < 8; ++op) {
            auto launch = [&](void (*f)(float*, long long*)) { f<<<148, threads>>>(out, cyc); };
            void (*f)(float*, long long*) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : op == 6 ? k<6> : k<7>;
            launch(f);
            cudaDeviceSynchronize();
            launch(f);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)threads * N * NI;   // per SM (one block per SM)
            printf("threads %4d %-12s %7.2f ops/clk/SM (2 instr/iter incl. the fmul)\n", threads, names[op], ops / c);
        }
    }
    return 0;
}
