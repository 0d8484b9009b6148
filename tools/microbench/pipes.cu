// Throughput microbenchmark of the FP64 / conversion pipes that the closed-loop
// quantizer of gz_compress leans on (sm_100a).  Each thread runs 8 independent
// dependency chains so the pipes, not latency, bound the loop.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
#define CH 8
template <int OP>
__global__ void k(double* out, float* outf, double a, float af) {
  double d[CH]; float f[CH]; long long li[CH];
  for (int c = 0; c < CH; ++c) { d[c] = a + threadIdx.x + c; f[c] = af + threadIdx.x + c; li[c] = threadIdx.x + c; }
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) d[c] = __dadd_rn(d[c], a);                       // DADD
      if (OP == 1) d[c] = __fma_rn(d[c], a, 1e-300);               // DFMA
      if (OP == 2) { f[c] = __double2float_rn((double)f[c] * 1.0000001); } // F2F.F64.F32 + DMUL + F2F.F32.F64
      if (OP == 3) { d[c] = (double)__double2float_rn(d[c]) + a; }  // F2F f64->f32->f64 + DADD
      if (OP == 4) { d[c] = floor(d[c]) + a; }                     // FRND.F64 + DADD
      if (OP == 5) { f[c] = __fadd_rn(f[c], af); }                 // FADD
      if (OP == 6) { li[c] = __double_as_longlong(d[c] = __dadd_rn((double)(li[c] & 1023), a)); } // I2F.F64 + DADD
      if (OP == 7) { f[c] = floorf(f[c]) + af; }                    // FRND f32
      if (OP == 8 && (c & 1) == 0) {                                // FADD2 (two lanes of f32x2)
        unsigned long long v = ((unsigned long long)__float_as_uint(f[c + 1]) << 32) | __float_as_uint(f[c]);
        const unsigned long long w = ((unsigned long long)__float_as_uint(af) << 32) | __float_as_uint(af);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(v) : "l"(w));
        f[c] = __uint_as_float((unsigned)v); f[c + 1] = __uint_as_float((unsigned)(v >> 32));
      }
      if (OP == 9) { li[c] = (li[c] << 1) ^ (li[c] >> 31); }        // int shift/xor (ALU)
    }
  }
  double s = 0; float sf = 0;
  for (int c = 0; c < CH; ++c) { s += d[c] + (double)li[c]; sf += f[c]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s; outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
}
template <int OP> void run(const char* name, double* o, float* of) {
  int blocks = 148 * 8, threads = 256;
  k<OP><<<blocks, threads>>>(o, of, 1e-9, 1e-9f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(o, of, 1e-9, 1e-9f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double ops = (double)blocks * threads * ITERS * CH;
  double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / 148.0;
  printf("%-34s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (at max clk %d MHz)\n", name, ms, ops / ms / 1e6, per_clk_sm, clk / 1000);
}
int main() {
  double* o; float* of; cudaMalloc(&o, 148 * 8 * 256 * 8); cudaMalloc(&of, 148 * 8 * 256 * 4);
  run<0>("DADD", o, of); run<1>("DFMA", o, of); run<2>("F2F.f32->f64, DMUL, F2F.f64->f32", o, of);
  run<3>("F2F f64->f32->f64 + DADD", o, of); run<4>("floor f64 + DADD", o, of); run<5>("FADD", o, of);
  run<6>("I2F.F64 + DADD", o, of); run<7>("floorf + FADD", o, of);
  run<8>("FADD2 (per f32 lane)", o, of); run<9>("SHF/LOP int", o, of);
  cudaError_t e = cudaDeviceSynchronize(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
