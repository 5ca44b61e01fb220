// Throughput probe: scalar FFMA vs packed FFMA2 (sm_100a), same flop count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_rate.cu -o ffma2_rate && ./ffma2_rate
#include <cstdio>
#include <cuda_runtime.h>

__global__ void scalar_k(float* out, int iters, float s) {
    float a[8];
    for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = fmaf(a[j], s, 0.5f);
    float t = 0;
    for (int j = 0; j < 8; j++) t += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void packed_k(float* out, int iters, float s) {
    float2 a[4];
    for (int j = 0; j < 4; j++) a[j] = make_float2(threadIdx.x * 1e-3f + 2 * j, 2 * j + 1);
    const float2 s2 = make_float2(s, s), h = make_float2(0.5f, 0.5f);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) a[j] = __ffma2_rn(a[j], s2, h);
    float t = 0;
    for (int j = 0; j < 4; j++) t += a[j].x + a[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    float* d;
    const int blocks = 148 * 8, threads = 256, iters = 20000;
    cudaMalloc(&d, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        scalar_k<<<blocks, threads>>>(d, iters, 0.999f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("scalar FFMA : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0);
        packed_k<<<blocks, threads>>>(d, iters, 0.999f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    }
    return 0;
}
