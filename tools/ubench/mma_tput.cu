// Microbenchmark: throughput of legacy mma.sync (tf32 m16n8k8, f64 m8n8k4)
// and SHFL on sm_100a, in SM cycles per warp-instruction per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float *out, int iters, long long *cyc) {
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    float c[4][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 4; j++)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    float s = 0; for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_f64(double *out, int iters, long long *cyc) {
    double a = threadIdx.x, b = a + 1;
    double c[4][2] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 4; j++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    double s = 0; for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_shfl(float *out, int iters, long long *cyc) {
    float v[4] = {(float)threadIdx.x, 1.f, 2.f, 3.f};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] += __shfl_xor_sync(0xffffffffu, v[j], 1 << j);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = v[0] + v[1] + v[2] + v[3];
}

__global__ void k_ffma(float *out, int iters, long long *cyc) {
    float v[8]; for (int j = 0; j < 8; j++) v[j] = threadIdx.x + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = fmaf(v[j], 1.0001f, 0.5f);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    float s = 0; for (int j = 0; j < 8; j++) s += v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *o; double *od; long long *cyc, h;
    cudaMalloc(&o, 148 * 1024 * 8 * 4); cudaMalloc(&od, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        int thr = warps * 32;
        k_tf32<<<148, thr>>>(o, iters, cyc); cudaDeviceSynchronize();
        k_tf32<<<148, thr>>>(o, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("tf32 m16n8k8 warps/SM %2d: %.3f SM-cyc per warp-mma\n", warps, (double)h / (iters * 4.0 * warps));
        k_f64<<<148, thr>>>(od, iters, cyc); cudaDeviceSynchronize();
        k_f64<<<148, thr>>>(od, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("f64  m8n8k4  warps/SM %2d: %.3f SM-cyc per warp-mma\n", warps, (double)h / (iters * 4.0 * warps));
        k_shfl<<<148, thr>>>(o, iters, cyc); cudaDeviceSynchronize();
        k_shfl<<<148, thr>>>(o, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("shfl        warps/SM %2d: %.3f SM-cyc per warp-shfl (+fadd)\n", warps, (double)h / (iters * 4.0 * warps));
        k_ffma<<<148, thr>>>(o, iters, cyc); cudaDeviceSynchronize();
        k_ffma<<<148, thr>>>(o, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("ffma        warps/SM %2d: %.3f SM-cyc per warp-ffma\n", warps, (double)h / (iters * 8.0 * warps));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
