// Microbenchmark: bandwidth of node-kernel-like access patterns on B200.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("%s\n",cudaGetErrorString(e)); return 1;}}while(0)

__global__ void node_like(float* T, float* F, const float* C, const float* Q, long off, long n) {
  long i = off + 4 * ((long)blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 4 > off + n) return;
  float4 t = *(float4*)(T + i), f = *(float4*)(F + i), c = *(const float4*)(C + i), q = *(const float4*)(Q + i);
  *(float4*)(F + i) = make_float4(0, 0, 0, 0);
  t.x += c.x * (q.x - f.x); t.y += c.y * (q.y - f.y); t.z += c.z * (q.z - f.z); t.w += c.w * (q.w - f.w);
  *(float4*)(T + i) = t;
}
__global__ void node_like8(float* T, float* F, const float* C, const float* Q, long off, long n) {
  long i0 = off + 8 * ((long)blockIdx.x * blockDim.x + threadIdx.x);
  if (i0 + 8 > off + n) return;
  float4 t[2], f[2], c[2], q[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) { long i = i0 + 4 * k; t[k] = *(float4*)(T + i); f[k] = *(float4*)(F + i); c[k] = *(const float4*)(C + i); q[k] = *(const float4*)(Q + i); }
#pragma unroll
  for (int k = 0; k < 2; ++k) { long i = i0 + 4 * k;
    *(float4*)(F + i) = make_float4(0, 0, 0, 0);
    t[k].x += c[k].x * (q[k].x - f[k].x); t[k].y += c[k].y * (q[k].y - f[k].y); t[k].z += c[k].z * (q[k].z - f[k].z); t[k].w += c[k].w * (q[k].w - f[k].w);
    *(float4*)(T + i) = t[k]; }
}
__global__ void copy4(float* dst, const float* src, long n) {
  long i = 4 * ((long)blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 4 <= n) *(float4*)(dst + i) = *(const float4*)(src + i);
}
__global__ void reds(float* F, long off, long n, long stride) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(F + off + (i * stride) % n, 1.0f);
}
int main() {
  long N = 57066625 + 1024, off = 40817664, n = 16303104;
  float *T, *F, *C, *Q, *big;
  CK(cudaMalloc(&T, N * 4)); CK(cudaMalloc(&F, N * 4)); CK(cudaMalloc(&C, N * 4)); CK(cudaMalloc(&Q, N * 4));
  CK(cudaMalloc(&big, 512l << 20));
  cudaMemset(T, 0, N * 4); cudaMemset(F, 0, N * 4); cudaMemset(C, 0, N * 4); cudaMemset(Q, 0, N * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto flush = [&]() { cudaMemsetAsync(big, 1, 512l << 20); };
  float ms;
  for (int variant = 0; variant < 6; ++variant) {
    float tot = 0; int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      flush();
      if (variant == 3) reds<<<(n + 255) / 256, 256>>>(F, off, n, 7919);
      cudaEventRecord(a);
      if (variant == 0 || variant == 3) node_like<<<(n / 4 + 255) / 256, 256>>>(T, F, C, Q, off, n);
      if (variant == 1) node_like8<<<(n / 8 + 255) / 256, 256>>>(T, F, C, Q, off, n);
      if (variant == 2) copy4<<<(n / 4 + 255) / 256, 256>>>(T + off, C + off, n);
      if (variant == 4) node_like<<<(n / 4 + 127) / 128, 128>>>(T, F, C, Q, off, n);
      if (variant == 5) node_like<<<(n / 4 + 511) / 512, 512>>>(T, F, C, Q, off, n);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      if (r >= 2) tot += ms;
    }
    ms = tot / reps;
    double bytes = (variant == 2) ? 8.0 * n : 24.0 * n;
    printf("variant %d: %.3f ms  %.0f GB/s\n", variant, ms, bytes / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
