// Integer-multiply roofline microbenchmark: the
// throughput of the exact instruction the CIOS kernels are built from,
// IMAD.WIDE.U32(.X) with carry chains (one 32×32→64 product each), on all
// SMs at full occupancy.  The measured rate is the `peak` of bench.py's
// roofline; the SM clock is measured in-kernel (clock64 / elapsed).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sfxb_cuda.h"
#include "mont.cuh"

namespace {

using namespace sfxb::dev;

constexpr int kChainLen = 8;

__global__ void __launch_bounds__(256) k_imad_peak(const uint32_t *seed, uint32_t *out, int iters,
                                                   long long *cycles) {
    uint32_t a[kChainLen], e[kChainLen + 2], o[kChainLen + 2];
#pragma unroll
    for (int j = 0; j < kChainLen; ++j) {
        a[j] = seed[(threadIdx.x + j) & 255] | 1u;
        e[j] = j;
        o[j] = 2 * j;
    }
    e[kChainLen] = e[kChainLen + 1] = o[kChainLen] = o[kChainLen + 1] = 0;
    uint32_t b = seed[threadIdx.x & 255] | 1u, c = b ^ 0x5555u;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int rep = 0; rep < 4; ++rep) {
            mad_w_cc(e[0], e[1], a[0], b, e[0], e[1]);
#pragma unroll
            for (int j = 2; j < kChainLen; j += 2) madc_w_cc(e[j], e[j + 1], a[j], b, e[j], e[j + 1]);
            e[kChainLen] = addc(e[kChainLen], 0u);
            mad_w_cc(o[0], o[1], a[1], c, o[0], o[1]);
#pragma unroll
            for (int j = 2; j < kChainLen; j += 2) madc_w_cc(o[j], o[j + 1], a[j + 1], c, o[j], o[j + 1]);
            o[kChainLen] = addc(o[kChainLen], 0u);
        }
        b += e[0];
        c += o[0];
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j <= kChainLen; ++j) s += e[j] ^ o[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cycles = t1 - t0;
}

} // namespace

extern "C" int sfxb_imad_peak(int device, double *products_per_s, double *sm_clock_mhz) {
    if (cudaSetDevice(device) != cudaSuccess) return SFXB_ERR_CUDA;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return SFXB_ERR_CUDA;
    // exactly one wave, so block 0 spans the whole kernel and clock64 / elapsed
    // is the SM clock under this load
    const int tpb = 256, iters = 4000;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_imad_peak, tpb, 0) != cudaSuccess || per_sm < 1)
        return SFXB_ERR_CUDA;
    const int blocks = p.multiProcessorCount * per_sm;
    uint32_t *seed = nullptr, *out = nullptr;
    long long *cyc = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = SFXB_OK;
    if (cudaMalloc(&seed, 1024 * 4) != cudaSuccess || cudaMalloc(&out, (size_t)blocks * tpb * 4) != cudaSuccess ||
        cudaMalloc(&cyc, 8) != cudaSuccess) {
        rc = SFXB_ERR_CUDA;
    } else {
        cudaMemset(seed, 0x37, 1024 * 4);
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_imad_peak<<<blocks, tpb>>>(seed, out, 200, cyc); // warm-up
        cudaEventRecord(e0);
        k_imad_peak<<<blocks, tpb>>>(seed, out, iters, cyc);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
            rc = SFXB_ERR_CUDA;
        } else {
            float ms = 0;
            long long cycles = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&cycles, cyc, 8, cudaMemcpyDeviceToHost);
            const double products = (double)blocks * tpb * iters * 4 * kChainLen; // 2 chains × kChainLen/2 × 4 reps
            *products_per_s = products / (ms * 1e-3);
            *sm_clock_mhz = (double)cycles / (ms * 1e-3) / 1e6;
        }
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(seed);
    cudaFree(out);
    cudaFree(cyc);
    return rc;
}
