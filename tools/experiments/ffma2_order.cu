// ffma2_order.cu -- FFMA2 rate of a 10x10 lane tile (5 row pairs x 10
// broadcast scalars per k, fragments from shared memory, register double
// buffering) as a function of the source order of the 50 FFMA2s and of the
// warps per SMSP.  Compare with tools/sass_banks.py on the same binary (the
// register-bank / operand-reuse model).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_order tools/experiments/ffma2_order.cu
#include <cuda_runtime.h>
#include <stdio.h>

#define MP 5
#define NR 10
constexpr int KTOT = 4096;

__device__ __forceinline__ void f2(unsigned long long &c, unsigned long long a, float b)
{
    unsigned long long bb;
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(bb));
}
__device__ __forceinline__ void lds128(unsigned a, float &x, float &y, float &z, float &w)
{
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
}
__device__ __forceinline__ void lds64(unsigned a, unsigned long long &x) { asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x) : "r"(a)); }
__device__ __forceinline__ void lds64f(unsigned a, float &x, float &y)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}

struct Frag {
    unsigned long long a[MP];
    float b[NR];
};
template <bool SMEM>
__device__ __forceinline__ void load(Frag &f, unsigned sa, unsigned sb, int k, const Frag &r)
{
    if (SMEM) {
#pragma unroll
        for (int i = 0; i < MP; ++i) lds64(sa + k * 320 + i * 64, f.a[i]);
        lds128(sb + k * 320, f.b[0], f.b[1], f.b[2], f.b[3]);
        lds128(sb + k * 320 + 128, f.b[4], f.b[5], f.b[6], f.b[7]);
        lds64f(sb + k * 320 + 256, f.b[8], f.b[9]);
    } else {
        f = r;
    }
}
template <int ORDER>
__device__ __forceinline__ void fma_step(unsigned long long (&acc)[MP][NR], const Frag &f)
{
    if (ORDER == 0) {  // pair-outer
#pragma unroll
        for (int i = 0; i < MP; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) f2(acc[i][j], f.a[i], f.b[j]);
    } else if (ORDER == 1) {  // scalar-outer
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
            for (int i = 0; i < MP; ++i) f2(acc[i][j], f.a[i], f.b[j]);
    } else {  // pair-outer snake
#pragma unroll
        for (int i = 0; i < MP; ++i)
#pragma unroll
            for (int jj = 0; jj < NR; ++jj) {
                const int j = (i & 1) ? NR - 1 - jj : jj;
                f2(acc[i][j], f.a[i], f.b[j]);
            }
    }
}
template <int ORDER, bool SMEM>
__global__ void __launch_bounds__(384, 1) kord(float *out, int K)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = (float)(i % 7) * 0.125f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned sa = base + (lane & 3) * 16, sb = base + 32768 + (lane >> 2) * 16;
    Frag r;
#pragma unroll
    for (int i = 0; i < MP; ++i) r.a[i] = (unsigned long long)(lane + i) * 0x100000001ull;
#pragma unroll
    for (int j = 0; j < NR; ++j) r.b[j] = (float)(lane + j) * 0.5f;
    unsigned long long acc[MP][NR];
#pragma unroll
    for (int i = 0; i < MP; ++i)
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[i][j] = 0ull;
    for (int kc = 0; kc < K; kc += 16) {
        Frag f[2];
        load<SMEM>(f[0], sa, sb, 0, r);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            if (kk + 1 < 16) load<SMEM>(f[(kk + 1) & 1], sa, sb, kk + 1, r);
            fma_step<ORDER>(acc, f[kk & 1]);
        }
        if (!SMEM) {
#pragma unroll
            for (int j = 0; j < NR; ++j) r.b[j] = __int_as_float(__float_as_int(r.b[j]) ^ kc);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < MP; ++i)
#pragma unroll
        for (int j = 0; j < NR; ++j) s += __uint_as_float((unsigned)acc[i][j]) + __uint_as_float((unsigned)(acc[i][j] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ksg NN fragment shape: k-blocks of 2, A pairs (LDS.64 per pair per k),
// B K-major (one LDS.64 = the column's values at k and k+1), FFMA2 order
// kk -> i -> j (kblock_fma); DB = register double buffering of k-blocks
template <bool DB, bool RND>
__global__ void __launch_bounds__(384, 1) kks(float *out, int K)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
        reinterpret_cast<float *>(sm)[i] = RND ? (float)(h >> 8) * (1.0f / 8388608.0f) - 1.0f : (float)(i % 7) * 0.125f;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned sa = base + (lane & 3) * 8, sb = base + 32768 + (lane >> 2) * 64;
    unsigned long long acc[MP][NR];
#pragma unroll
    for (int i = 0; i < MP; ++i)
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[i][j] = 0ull;
    for (int kc = 0; kc < K; kc += 16) {
        unsigned long long a[2][2][MP];
        float b[2][2][NR];
        auto ld = [&](int buf, int kb) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int i = 0; i < MP; ++i) lds64(sa + (kb + kk) * 320 + i * 32, a[buf][kk][i]);
#pragma unroll
            for (int j = 0; j < NR; ++j) lds64f(sb + j * 512 + ((kb * 4) ^ ((j & 3) << 4)), b[buf][0][j], b[buf][1][j]);
        };
        ld(0, 0);
#pragma unroll
        for (int kb = 0; kb < 16; kb += 2) {
            const int cur = DB ? (kb / 2) & 1 : 0;
            if (DB && kb + 2 < 16) ld(cur ^ 1, kb + 2);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int i = 0; i < MP; ++i)
#pragma unroll
                    for (int j = 0; j < NR; ++j) f2(acc[i][j], a[cur][kk][i], b[cur][kk][j]);
            if (!DB && kb + 2 < 16) ld(0, kb + 2);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < MP; ++i)
#pragma unroll
        for (int j = 0; j < NR; ++j) s += __uint_as_float((unsigned)acc[i][j]) + __uint_as_float((unsigned)(acc[i][j] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool DB, bool RND>
void run_ks(int wps, float *o)
{
    auto fn = kks<DB, RND>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int blocks = 148, threads = 128 * wps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fn<<<blocks, threads, 65536>>>(o, KTOT);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn<<<blocks, threads, 65536>>>(o, KTOT);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 5.0 * blocks * threads * (double)KTOT * MP * NR * 4;
    printf("ksg-NN shape %s %s warps/SMSP %d: %.1f TFLOP/s (%.3f of 73.5)  %s\n", DB ? "double-buffered" : "single",
           RND ? "random data" : "i%7 data", wps,
           fl / ms / 1e9, fl / ms / 1e9 / 73.5, cudaGetErrorString(cudaGetLastError()));
}

template <int ORDER, bool SMEM>
void run(int wps, float *o)
{
    auto fn = kord<ORDER, SMEM>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int blocks = 148, threads = 128 * wps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fn<<<blocks, threads, 65536>>>(o, KTOT);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn<<<blocks, threads, 65536>>>(o, KTOT);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 5.0 * blocks * threads * (double)KTOT * MP * NR * 4;
    printf("order %d %s warps/SMSP %d: %.1f TFLOP/s (%.3f of 73.5)  %s\n", ORDER, SMEM ? "smem" : "regs", wps,
           fl / ms / 1e9, fl / ms / 1e9 / 73.5, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    float *o;
    cudaMalloc(&o, 148 * 384 * 4);
    for (int w = 2; w <= 3; ++w) {
        run_ks<true, false>(w, o);
        run_ks<false, false>(w, o);
        run_ks<true, true>(w, o);
        run_ks<false, true>(w, o);
    }
    for (int w = 1; w <= 3; ++w) {
        run<0, true>(w, o);
        run<1, true>(w, o);
        run<2, true>(w, o);
        run<0, false>(w, o);
        run<2, false>(w, o);
    }
    return 0;
}
