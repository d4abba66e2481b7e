#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define N 8
__device__ __forceinline__ void madlo_cc(uint32_t &d, uint32_t a, uint32_t b) { asm volatile("mad.lo.cc.u32 %0,%1,%2,%0;" : "+r"(d) : "r"(a), "r"(b)); }
__device__ __forceinline__ void madclo_cc(uint32_t &d, uint32_t a, uint32_t b) { asm volatile("madc.lo.cc.u32 %0,%1,%2,%0;" : "+r"(d) : "r"(a), "r"(b)); }
__device__ __forceinline__ void madchi_cc(uint32_t &d, uint32_t a, uint32_t b) { asm volatile("madc.hi.cc.u32 %0,%1,%2,%0;" : "+r"(d) : "r"(a), "r"(b)); }
__device__ __forceinline__ void addc0(uint32_t &d) { asm volatile("addc.u32 %0,%0,0;" : "+r"(d)); }

// carry-chain wide MAD: per iteration 2 chains x 8 products
__global__ void k_chain(const uint32_t* A, uint32_t* out, int iters) {
  uint32_t a[N], e[N+2], o[N+2];
  for (int j = 0; j < N; j++) { a[j] = A[(threadIdx.x + j) & 255]; e[j] = j; o[j] = 2*j; }
  e[N]=e[N+1]=o[N]=o[N+1]=0;
  uint32_t b = A[threadIdx.x & 255] | 1, c = b ^ 0x5555;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int rep = 0; rep < 4; rep++) {
    madlo_cc(e[0], a[0], b); madchi_cc(e[1], a[0], b);
#pragma unroll
    for (int j = 2; j < N; j += 2) { madclo_cc(e[j], a[j], b); madchi_cc(e[j+1], a[j], b); }
    addc0(e[N]);
    madlo_cc(o[0], a[1], c); madchi_cc(o[1], a[1], c);
#pragma unroll
    for (int j = 2; j < N; j += 2) { madclo_cc(o[j], a[j+1], c); madchi_cc(o[j+1], a[j+1], c); }
    addc0(o[N]);
    }
    b += e[0]; c += o[0];
  }
  uint32_t s = 0; for (int j = 0; j <= N; j++) s += e[j] ^ o[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// independent IMAD.WIDE (no carry): 8 independent 64-bit accumulators
__global__ void k_wide(const uint32_t* A, uint32_t* out, int iters) {
  uint64_t acc[N]; uint32_t a[N];
  for (int j = 0; j < N; j++) { a[j] = A[(threadIdx.x + j) & 255]; acc[j] = j; }
  uint32_t b = A[threadIdx.x & 255] | 1;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int rep = 0; rep < 8; rep++)
#pragma unroll
    for (int j = 0; j < N; j++) acc[j] = (uint64_t)a[j] * b + acc[j];
    b += (uint32_t)acc[0];
  }
  uint64_t s = 0; for (int j = 0; j < N; j++) s ^= acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s ^ (uint32_t)(s>>32);
}
// 32-bit IMAD lo
__global__ void k_lo(const uint32_t* A, uint32_t* out, int iters) {
  uint32_t acc[N], a[N];
  for (int j = 0; j < N; j++) { a[j] = A[(threadIdx.x + j) & 255]; acc[j] = j; }
  uint32_t b = A[threadIdx.x & 255] | 1;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int rep = 0; rep < 8; rep++)
#pragma unroll
    for (int j = 0; j < N; j++) acc[j] = a[j] * b + acc[j];
    b += acc[0];
  }
  uint32_t s = 0; for (int j = 0; j < N; j++) s ^= acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// IMAD.HI
__global__ void k_hi(const uint32_t* A, uint32_t* out, int iters) {
  uint32_t acc[N], a[N];
  for (int j = 0; j < N; j++) { a[j] = A[(threadIdx.x + j) & 255]; acc[j] = j; }
  uint32_t b = A[threadIdx.x & 255] | 1;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int rep = 0; rep < 8; rep++)
#pragma unroll
    for (int j = 0; j < N; j++) acc[j] = __umulhi(a[j], b) + acc[j];
    b += acc[0];
  }
  uint32_t s = 0; for (int j = 0; j < N; j++) s ^= acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// fp64 fma
__global__ void k_dfma(const uint32_t* A, uint32_t* out, int iters) {
  double acc[N], a[N];
  for (int j = 0; j < N; j++) { a[j] = A[(threadIdx.x + j) & 255]; acc[j] = j; }
  double b = A[threadIdx.x & 255] * 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int rep = 0; rep < 8; rep++)
#pragma unroll
    for (int j = 0; j < N; j++) acc[j] = fma(a[j], b, acc[j]);
    b += acc[0] * 1e-30;
  }
  double s = 0; for (int j = 0; j < N; j++) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
}
typedef void (*kfn)(const uint32_t*, uint32_t*, int);
int main() {
  uint32_t *A, *out; cudaMalloc(&A, 1024*4); cudaMalloc(&out, 148*64*1024*4);
  cudaMemset(A, 0x37, 1024*4);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  struct { const char* name; kfn f; double ops_per_iter; } ks[] = {
    {"chain_madc(lo+hi pair = 1 product)", k_chain, 4*2*N},   // products per iter
    {"imad_wide", k_wide, 8*N},
    {"imad_lo", k_lo, 8*N},
    {"imad_hi", k_hi, 8*N},
    {"dfma", k_dfma, 8*N},
  };
  int iters = 20000;
  for (auto& k : ks) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k.f<<<blocks, tpb>>>(A, out, 100);
      cudaEventRecord(e0);
      k.f<<<blocks, tpb>>>(A, out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
      double ops = (double)blocks * tpb * iters * k.ops_per_iter;
      double rate = ops / (ms * 1e-3);
      printf("%-40s tpb=%4d  %.3f ms  %.3e ops/s  = %.1f ops/clk/SM @%.0f MHz (err=%s)\n", k.name, tpb, ms, rate,
             rate / (sms * clk * 1e3), clk/1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
