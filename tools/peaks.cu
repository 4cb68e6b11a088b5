// peaks.cu -- H3 microbenchmarks: the measured compute and
// memory peaks that bench.py's roofline denominators use.
//
//   FFMA   fp32 fma.rn.f32      (SASS FFMA)       8 independent chains / thread
//   FFMA2  fp32 fma.rn.f32x2    (SASS FFMA2)      8 independent pairs  / thread
//   DFMA   fp64 fma.rn.f64      (SASS DFMA)       8 independent chains / thread
//   DMMA   mma.sync m8n8k4 f64  (SASS DMMA.8x8x4) 4 independent accumulators / warp
//   HBM read  (LDG.128 streaming sum over 4 GiB) and HBM copy (read + write)
//
// Every kernel runs on a grid of 148 x k CTAs, timed with CUDA events after
// warm-up; the result is the best of 5.  Output: one JSON object on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks tools/peaks.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));          \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_ffma(float *out, float a, float b)
{
    float c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(c[i]) : "f"(a), "f"(b));
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float *out, float a, float b)
{
    unsigned long long c[8], av, bv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float x = threadIdx.x * 1e-3f + i;
        asm("mov.b64 %0, {%1, %1};" : "=l"(c[i]) : "f"(x));
    }
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[i]) : "l"(av), "l"(bv));
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(c[i]));
        s += lo + hi;
    }
    if (s == 1234.5f) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma(double *out, double a, double b)
{
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS / 8; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i]) : "d"(a), "d"(b));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dmma(double *out, double a, double b)
{
    double d[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS / 8; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[i][0]), "+d"(d[i][1])
                         : "d"(a), "d"(b));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
    if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(512) k_read(const float4 *__restrict__ x, size_t n4, float *out)
{
    float4 acc = make_float4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(x + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = 1.f;
}

__global__ void __launch_bounds__(512) k_copy(const float4 *__restrict__ x, float4 *__restrict__ y, size_t n4)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        __stcs(y + i, __ldcs(x + i));
}

template <typename F>
static float best_ms(F launch, int reps = 5)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    float *fo;
    double *dO;
    CK(cudaMalloc(&fo, 64));
    CK(cudaMalloc(&dO, 64));
    const int blocks = sms * 8, threads = 256;
    const double nthr = (double)blocks * threads;
    float t;
    t = best_ms([&] { k_ffma<<<blocks, threads>>>(fo, 1.0001f, 1e-7f); });
    const double ffma = nthr * ITERS * 8 * 2 / (t * 1e-3) / 1e12;
    t = best_ms([&] { k_ffma2<<<blocks, threads>>>(fo, 1.0001f, 1e-7f); });
    const double ffma2 = nthr * ITERS * 8 * 2 * 2 / (t * 1e-3) / 1e12;
    t = best_ms([&] { k_dfma<<<blocks, threads>>>(dO, 1.0001, 1e-9); });
    const double dfma = nthr * (ITERS / 8) * 8 * 2 / (t * 1e-3) / 1e12;
    t = best_ms([&] { k_dmma<<<blocks, threads>>>(dO, 1.0001, 1e-9); });
    const double dmma = (nthr / 32) * (ITERS / 8) * 4 * 256 * 2 / (t * 1e-3) / 1e12;
    CK(cudaGetLastError());

    const size_t bytes = (size_t)4 << 30;
    float4 *x, *y;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMalloc(&y, bytes));
    CK(cudaMemset(x, 0, bytes));
    CK(cudaMemset(y, 0, bytes));
    const size_t n4 = bytes / 16;
    t = best_ms([&] { k_read<<<sms * 4, 512>>>(x, n4, fo); });
    const double rd = bytes / (t * 1e-3) / 1e9;
    t = best_ms([&] { k_copy<<<sms * 4, 512>>>(x, y, n4); });
    const double cp = 2.0 * bytes / (t * 1e-3) / 1e9;
    CK(cudaGetLastError());
    printf("{\"sms\": %d, \"clock_rate_mhz\": %.0f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
           "\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"hbm_read_gbs\": %.1f, \"hbm_copy_gbs\": %.1f}\n",
           sms, clk / 1e3, ffma, ffma2, dfma, dmma, rd, cp);
    return 0;
}
