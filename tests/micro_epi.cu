// Microbenchmark (not part of the library): throughput of SDF-MLP epilogue instruction mixes on
// sm_100a, in activations per clock per SM (one 256..512-thread block per SM, independent chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_epi tests/micro_epi.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

constexpr int N = 2048, NI = 16;

__device__ __forceinline__ float tanh_a(float x) {
    float y;
    asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// MODE 0: pack only; 1: silu (ffma, tanh, ffma) no pack; 2: silu + pack; 3: relu (fadd, fmax) + pack;
// 4: silu + pack + unpack/dot (last layer); 5: F2F-free pack via PRMT of truncated halves (lower bound)
template <int MODE>
__global__ void k(uint32_t* out, long long* cyc, float b) {
    __shared__ float4 sw[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sw[i] = make_float4(0.01f * i, 0.02f, 0.03f, 0.5f);
    float v[NI];
    uint32_t acc = 0;
    float dot = 0.f;
    for (int i = 0; i < NI; ++i) v[i] = 0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 2
    for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int i = 0; i < NI; i += 2) {
            float x0 = v[i], x1 = v[i + 1];
            if constexpr (MODE == 0) {
                acc ^= pack(x0, x1);
                v[i] = x0 + b;
                v[i + 1] = x1 + b;
            } else if constexpr (MODE == 1) {
                float h0 = fmaf(x0, 0.5f, b), h1 = fmaf(x1, 0.5f, b);
                v[i] = fmaf(h0, tanh_a(h0), h0);
                v[i + 1] = fmaf(h1, tanh_a(h1), h1);
            } else if constexpr (MODE == 2 || MODE == 4) {
                float h0 = fmaf(x0, 0.5f, b), h1 = fmaf(x1, 0.5f, b);
                const uint32_t p = pack(fmaf(h0, tanh_a(h0), h0), fmaf(h1, tanh_a(h1), h1));
                if constexpr (MODE == 2) acc ^= p;
                else {
                    dot = fmaf(__uint_as_float(p << 16), x0, dot);
                    dot = fmaf(__uint_as_float(p & 0xFFFF0000u), x1, dot);
                }
                v[i] = h0 + 1.0f;
                v[i + 1] = h1 + 1.0f;
            } else if constexpr (MODE == 3) {
                acc ^= pack(fmaxf(x0 + b, 0.f), fmaxf(x1 + b, 0.f));
                v[i] = x0 * 0.999f;
                v[i + 1] = x1 * 0.999f;
            } else if constexpr (MODE == 5) {
                float h0 = fmaf(x0, 0.5f, b), h1 = fmaf(x1, 0.5f, b);
                const float y0 = fmaf(h0, tanh_a(h0), h0), y1 = fmaf(h1, tanh_a(h1), h1);
                acc ^= __byte_perm(__float_as_uint(y0), __float_as_uint(y1), 0x7632);
                v[i] = h0 + 1.0f;
                v[i + 1] = h1 + 1.0f;
            } else {
                // layer-1 mix: per column a broadcast LDS.128 (w0,w1,w2,b), 3 FFMA, tanh, FFMA, pack
                const float4 w0 = sw[(n * NI + i) & 255], w1 = sw[(n * NI + i + 1) & 255];
                const float a0 = fmaf(w0.x, x0, fmaf(w0.y, x1, fmaf(w0.z, b, w0.w)));
                const float a1 = fmaf(w1.x, x0, fmaf(w1.y, x1, fmaf(w1.z, b, w1.w)));
                acc ^= pack(fmaf(a0, tanh_a(a0), a0), fmaf(a1, tanh_a(a1), a1));
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(dot) + __float_as_uint(v[0]);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 1 << 16);
    const char* names[] = {"pack only (+fadd)", "silu fp32 no pack", "silu + pack", "relu + pack", "silu+pack+dot",
                           "silu + prmt-trunc", "layer1 (lds+3ffma+silu+pack)"};
    void (*fs[])(uint32_t*, long long*, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
    for (int threads : {256, 512}) {
        for (int m = 0; m < 7; ++m) {
            fs[m]<<<148, threads>>>(out, cyc, 0.01f);
            fs[m]<<<148, threads>>>(out, cyc, 0.01f);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("threads %4d %-22s %7.2f act/clk/SM\n", threads, names[m], (double)threads * N * NI / c);
        }
    }
    return 0;
}
