// Does FP64 DMMA run on a pipe separate from DFMA on B200?  And which f64
// mma.sync shape has the best rate?
//   1. DMMA shapes: m8n8k4, m16n8k4, m16n8k8, m16n8k16 (f64, mma.sync)
//   2. mixed streams: per loop iteration NM DMMA m8n8k4 + ND DFMA (independent
//      chains); if combined FP64 flop/s exceeds either alone, the pipes overlap
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench4 tools/microbench4.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void dmma_shape(double* out, int iters) {
  // SHAPE 0: m8n8k4 (A 1, B 1, C 2 regs), 1: m16n8k4 (A 2, B 1, C 4),
  // 2: m16n8k8 (A 4, B 2, C 4), 3: m16n8k16 (A 8, B 4, C 4)
  double c[6][4];
#pragma unroll
  for (int i = 0; i < 6; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 2e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
              "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}

template <int NM, int ND>
__global__ void mixed(double* out, int iters) {
  double c[NM > 0 ? NM : 1][2];
  double d[ND > 0 ? ND : 1];
#pragma unroll
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) d[i] = 1e-3 * (threadIdx.x + i);
  const double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  const double x = 1.0000001, y = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (NM > ND ? NM : ND); ++i) {
      if (i < NM)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      if (i < ND) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(x), "d"(y));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < (NM > 0 ? NM : 1); ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += d[i];
  if (s == 1.2345) out[0] = s;
}

static cudaEvent_t e0, e1;
static int sms;

template <int SHAPE>
void run_shape(double* out) {
  const int iters = 1 << 12, blocks = sms * 8, th = 256;
  dmma_shape<SHAPE><<<blocks, th>>>(out, 64);
  cudaEventRecord(e0);
  dmma_shape<SHAPE><<<blocks, th>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma_per = SHAPE == 0 ? 256 : SHAPE == 1 ? 512 : SHAPE == 2 ? 1024 : 2048;
  const char* nm[] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  printf("DMMA %-9s: %.2f TFLOP/s\n", nm[SHAPE], 2.0 * fma_per * 6 * double(iters) * blocks * (th / 32) / (ms * 1e-3) / 1e12);
}

template <int NM, int ND>
void run_mixed(double* out) {
  const int iters = 1 << 12, blocks = sms * 8, th = 256;
  mixed<NM, ND><<<blocks, th>>>(out, 64);
  cudaEventRecord(e0);
  mixed<NM, ND><<<blocks, th>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * (th / 32);
  const double f_mma = 2.0 * 256 * NM * double(iters) * warps, f_fma = 2.0 * 32 * ND * double(iters) * warps;
  const double s = ms * 1e-3;
  printf("mixed NM=%2d ND=%3d: dmma %.2f + dfma %.2f = %.2f TFLOP/s\n", NM, ND, f_mma / s / 1e12, f_fma / s / 1e12,
         (f_mma + f_fma) / s / 1e12);
}

int main() {
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  run_shape<0>(out);
  run_shape<1>(out);
  run_shape<2>(out);
  run_shape<3>(out);
  run_mixed<8, 0>(out);
  run_mixed<0, 16>(out);
  run_mixed<8, 16>(out);
  run_mixed<8, 32>(out);
  run_mixed<8, 64>(out);
  run_mixed<4, 32>(out);
  run_mixed<2, 32>(out);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
