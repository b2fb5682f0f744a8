// alu_peaks.cu -- measured FP64 / FP32 FMA throughput of this GPU (the ALU
// roofline denominators of the fp64 build kernels and of K7).
// Independent FMA chains per thread, enough warps to fill every SM, CUDA
// events, best of 5.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/alu_peaks.cu -o /tmp/alu_peaks
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <class T>
__global__ void __launch_bounds__(256) k_fma(T* out, T a, T b) {
    T x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    T s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == (T)-1) out[threadIdx.x] = s;  // keep the chains alive
}

template <class T>
static double measure(int blocks) {
    T* out;
    cudaMalloc(&out, 256 * sizeof(T));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma<T><<<blocks, 256>>>(out, (T)0.999, (T)0.001);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fma<T><<<blocks, 256>>>(out, (T)0.999, (T)0.001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    cudaFree(out);
    const double fmas = (double)blocks * 256 * kIters * kChains;
    return 2.0 * fmas / (best * 1e-3) / 1e12;  // TFLOP/s (FMA = 2 flops)
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8;
    const double f64 = measure<double>(blocks);
    const double f32 = measure<float>(blocks);
    std::printf("{\"fp64_tflops\": %.3f, \"fp32_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
                "\"how\": \"%d independent FMA chains x %d iterations per thread, %d blocks x 256 "
                "threads, best of 5, CUDA events (scripts/alu_peaks.cu)\"}\n",
                f64, f32, sms, clk / 1e3, kChains, kIters, blocks);
    return 0;
}
