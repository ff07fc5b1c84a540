// Microbenchmark (not part of the library): SiLU + bf16x2 pack throughput on sm_100a when a fraction of
// the tanh evaluations moves from the MUFU (16/clk/SM) to an odd polynomial on the FMA pipe (FFMA2).
// Activations per clock per SM; one 512-thread block per SM; 8 pairs per iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_poly tests/micro_poly.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

constexpr int N = 2048;

__device__ __forceinline__ float tanh_a(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 f2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ float2 m2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ uint32_t silu_mufu(float2 h) {
    const float2 s = f2(h, make_float2(tanh_a(h.x), tanh_a(h.y)), h);
    return pack(s.x, s.y);
}
// tanh(h) ~ h p(min(h^2, c^2)), p of degree 8 in s (coefficients pre-halved); (1 + tanh)/2 saturated by
// FFMA.SAT; silu = 2 h v.  MODE 1: as written (2 extra instrs); the kernel would fold the 2 into weights.
template <bool FOLD2>
__device__ __forceinline__ uint32_t silu_poly(float2 h) {
    float2 s = m2(h, h);
    s.x = fminf(s.x, 15.21f);
    s.y = fminf(s.y, 15.21f);
    float2 p = make_float2(4.449855151e-09f, 4.449855151e-09f);
    p = f2(p, s, make_float2(-3.170409855e-07f, -3.170409855e-07f));
    p = f2(p, s, make_float2(9.578018762e-06f, 9.578018762e-06f));
    p = f2(p, s, make_float2(-1.605451544e-04f, -1.605451544e-04f));
    p = f2(p, s, make_float2(1.647174824e-03f, 1.647174824e-03f));
    p = f2(p, s, make_float2(-1.086502243e-02f, -1.086502243e-02f));
    p = f2(p, s, make_float2(4.812432826e-02f, 4.812432826e-02f));
    p = f2(p, s, make_float2(-1.557688713e-01f, -1.557688713e-01f));
    p = f2(p, s, make_float2(4.980173409e-01f, 4.980173409e-01f));
    float2 v;
    v.x = __saturatef(fmaf(h.x, p.x, 0.5f));
    v.y = __saturatef(fmaf(h.y, p.y, 0.5f));
    float2 y = m2(h, v);
    if constexpr (!FOLD2) y = f2(y, make_float2(2.f, 2.f), make_float2(0.f, 0.f));
    return pack(y.x, y.y);
}

// NPOLY of the 8 pairs per iteration on the polynomial, spread as (pi * NPOLY) % 8 < NPOLY
template <int NPOLY, bool FOLD2>
__global__ void k(uint32_t* out, long long* cyc, float b) {
    float v[16];
    uint32_t acc = 0;
    for (int i = 0; i < 16; ++i) v[i] = 0.001f * (threadIdx.x + i) - 2.f;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 2
    for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int pi = 0; pi < 8; ++pi) {
            const float2 h = make_float2(v[2 * pi], v[2 * pi + 1]);
            const bool poly = ((pi * NPOLY) % 8) < NPOLY;
            acc ^= poly ? silu_poly<FOLD2>(h) : silu_mufu(h);
            v[2 * pi] = h.x + b;
            v[2 * pi + 1] = h.y + b;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(v[0]);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void accuracy(float* err) {
    // max |silu_poly - silu| / max(1, |silu|) over h in [-12, 12] (h = x/2), before bf16 rounding
    float m = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (1 << 22); i += gridDim.x * blockDim.x) {
        const float h = -12.f + 24.f * i / (float)(1 << 22);
        const uint32_t pp = silu_poly<false>(make_float2(h, h));
        const float yp = __uint_as_float(pp << 16);
        const float ye = 2.f * h / (1.f + expf(-2.f * h));
        const float ym = __uint_as_float(silu_mufu(make_float2(h, h)) << 16);
        m = fmaxf(m, fabsf(yp - ye) / fmaxf(1.f, fabsf(ye)));
        atomicMax(reinterpret_cast<int*>(err + 1), __float_as_int(fabsf(ym - ye) / fmaxf(1.f, fabsf(ye))));
    }
    atomicMax(reinterpret_cast<int*>(err), __float_as_int(m));
}

int main() {
    uint32_t* out;
    long long* cyc;
    float* err;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 1 << 16);
    cudaMalloc(&err, 8);
    cudaMemset(err, 0, 8);
    accuracy<<<148, 256>>>(err);
    float e[2];
    cudaMemcpy(e, err, 8, cudaMemcpyDeviceToHost);
    printf("max err (after bf16 pack) poly %.3e  mufu %.3e\n", e[0], e[1]);
    struct V {
        const char* name;
        void (*f)(uint32_t*, long long*, float);
    } vs[] = {{"mufu only", k<0, true>},        {"poly 1/8", k<1, true>}, {"poly 2/8", k<2, true>},
              {"poly 3/8", k<3, true>},         {"poly 4/8", k<4, true>}, {"poly 8/8", k<8, true>},
              {"poly 2/8 (no fold)", k<2, false>}, {"poly 3/8 (no fold)", k<3, false>}};
    for (int threads : {256, 512}) {
        for (auto& vv : vs) {
            vv.f<<<148, threads>>>(out, cyc, 1e-4f);
            vv.f<<<148, threads>>>(out, cyc, 1e-4f);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("threads %4d %-20s %7.2f act/clk/SM\n", threads, vv.name, (double)threads * N * 16 / c);
        }
    }
    return 0;
}
