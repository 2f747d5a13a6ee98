// Microbenchmark: scalar FFMA vs packed FFMA2 (fma.rn.f32x2) issue/throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
template <int CH>
__global__ void scal(float* out, int iters, float a, float b) {
    float x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0; for (int i = 0; i < CH; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void pack(float* out, int iters, float a, float b) {
    u64 x[CH];
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    u64 A = *reinterpret_cast<u64*>(&av), B = *reinterpret_cast<u64*>(&bv);
    for (int i = 0; i < CH; ++i) { float2 t = make_float2(threadIdx.x + i, i); x[i] = *reinterpret_cast<u64*>(&t); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma2(x[i], A, B);
    float s = 0; for (int i = 0; i < CH; ++i) { float2 t = *reinterpret_cast<float2*>(&x[i]); s += t.x + t.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: FMAs plus an equal number of independent integer ops (issue-slot sharing)
template <bool PACK>
__global__ void mixed(float* out, int iters, float a, float b) {
    float x[8]; unsigned y[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = threadIdx.x * 7 + i; }
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    u64 A = *reinterpret_cast<u64*>(&av), B = *reinterpret_cast<u64*>(&bv);
    for (int it = 0; it < iters; ++it) {
        if (PACK) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                u64 t = *reinterpret_cast<u64*>(&x[i]);
                t = fma2(t, A, B);
                *reinterpret_cast<u64*>(&x[i]) = t;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = y[i] * 3u + 1u;
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i] + (float)(y[i] & 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 14, blocks = 148 * 8, thr = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); scal<8><<<blocks, thr>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * blocks * thr * iters * 8;
        printf("FFMA  scalar: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0); pack<8><<<blocks, thr>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2 packed: %.3f ms  %.1f TFLOP/s\n", ms, 2 * fl / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); mixed<false><<<blocks, thr>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mixed scalar FFMA + int: %.3f ms\n", ms);
        cudaEventRecord(e0); mixed<true><<<blocks, thr>>>(out, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mixed FFMA2 + int:        %.3f ms\n", ms);
    }
    return 0;
}
