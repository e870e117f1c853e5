// Probe: FP64 tensor (DMMA via mma.sync) vs FP64 FMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_dmma_m8n8k4(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[8][2];
  for (int i = 0; i < 8; ++i) { d[i][0] = 0; d[i][1] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 123.0) out[0] = s;
}
__global__ void k_dmma_m16n8k16(double* out) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-6;
  double d[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
  if (s == 123.0) out[0] = s;
}
__global__ void k_dfma(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-9;
  double d[16];
  for (int i = 0; i < 16; ++i) d[i] = i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = fma(d[i], b, a);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += d[i];
  if (s == 123.0) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int blocks = sms * 4, threads = warps * 32;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); k_dmma_m8n8k4<<<blocks, threads>>>(out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double fl = (double)blocks * warps * ITERS * 8 * 512;
    printf("dmma m8n8k4  warps/blk=%d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); k_dmma_m16n8k16<<<blocks, threads>>>(out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    fl = (double)blocks * warps * (ITERS / 4) * 4 * (16 * 8 * 16 * 2);
    printf("dmma m16n8k16 warps/blk=%d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    fl = (double)blocks * threads * ITERS * 16 * 2;
    printf("dfma         warps/blk=%d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
