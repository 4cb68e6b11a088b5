// ffma2_lds.cu -- does interleaving the fragment LDS traffic of a 10x10
// register tile (5 LDS.64 + 10 LDS.32 per k, broadcast addresses) slow the
// FFMA2 stream below the register-only rate?  2 and 3 warps per SMSP.
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int KS = 1024;

__device__ __forceinline__ void f2(unsigned long long &c, unsigned long long a, float b)
{
    unsigned long long bb;
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(bb));
}

template <int MODE>
__global__ void kk(float *out, int salt)
{
    __shared__ __align__(16) float sm[64 * 64];
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = (float)((i * 7 + salt) % 13) * 0.01f;
    __syncthreads();
    unsigned long long acc[5][10];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 10; ++j) acc[i][j] = 0ull;
    const int lane = threadIdx.x & 31, ti = lane & 3, tj = lane >> 2;
    unsigned long long ra[2][5];
    float rb[2][10];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int i = 0; i < 5; ++i) ra[s][i] = *reinterpret_cast<const unsigned long long *>(&sm[2 * ti + 8 * i + s * 64]);
#pragma unroll
        for (int j = 0; j < 10; ++j) rb[s][j] = sm[tj + 8 * j + 100 + s];
    }
    for (int it = 0; it < KS; it += 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            unsigned long long a[5];
            float b[10];
            if (MODE == 0) {  // fragments from shared memory every k
                const int row = (k & 15) * 64;
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    a[i] = *reinterpret_cast<const volatile unsigned long long *>(&sm[row + 2 * ti + 8 * i]);
#pragma unroll
                for (int j = 0; j < 10; ++j) b[j] = *reinterpret_cast<const volatile float *>(&sm[row + 256 + tj + 8 * j]);
            } else {  // register fragments (two alternating sets)
#pragma unroll
                for (int i = 0; i < 5; ++i) a[i] = ra[k & 1][i];
#pragma unroll
                for (int j = 0; j < 10; ++j) b[j] = rb[k & 1][j];
            }
#pragma unroll
            for (int j = 0; j < 10; ++j)
#pragma unroll
                for (int i = 0; i < 5; ++i) f2(acc[i][j], a[i], b[j]);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 10; ++j) {
            float lo, hi;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i][j]));
            s += lo + hi;
        }
    if (s == 1234.5f) out[0] = s;
}

template <int MODE>
void run(int wps, float *o)
{
    const int blocks = 148, threads = 128 * wps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kk<MODE><<<blocks, threads>>>(o, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kk<MODE><<<blocks, threads>>>(o, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 5.0 * blocks * threads * (double)KS * 100 * 2;
    printf("mode %d (%s) warps/SMSP %d: %.1f TFLOP/s (%.2f of 73.5)\n", MODE, MODE ? "regs" : "lds", wps,
           fl / ms / 1e9, fl / ms / 1e9 / 73.5);
}

int main()
{
    float *o;
    cudaMalloc(&o, 64);
    for (int w = 1; w <= 3; ++w) {
        run<0>(w, o);
        run<1>(w, o);
    }
    return 0;
}
