// ffma2_morph.cu -- morph the FFMA2 microbenchmark (ksg NN fragment shape,
// 10x10 lane tile, 0.84 of the FFMA2 peak) step by step into the ksg
// consumer's execution environment, to find what costs the ksg compute loop
// its rate (DBG=3 probe: ~0.67).
//   WS   : 384 threads, warps 0-3 setmaxnreg.dec + exit, 8 consumer warps setmaxnreg.inc 232
//   REG  : each warp pair reads its own 48 KB smem region (ksg groups' rings)
//   UNIT : units of 80 k (5 chunks of 16): acc zeroed per unit, per-unit epilogue
//          (EPI 1: FADD-chain sum like the probe's DBG=2; EPI 2: alpha*acc STS.64 into a C buffer)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_morph tools/experiments/ffma2_morph.cu
#include <cuda_runtime.h>
#include <stdio.h>

#define MP 5
#define NR 10

__device__ __forceinline__ void f2(unsigned long long &c, unsigned long long a, float b)
{
    unsigned long long bb;
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(bb));
}
__device__ __forceinline__ void lds64(unsigned a, unsigned long long &x) { asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x) : "r"(a)); }
__device__ __forceinline__ void lds64f(unsigned a, float &x, float &y)
{
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
}

template <bool WS, bool REG, int EPI, bool INIT = true>
__global__ void __launch_bounds__(384, 1) km(float *out, int nunits, int kunit)
{
    extern __shared__ __align__(16) unsigned char sm[];
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; INIT && i < 200 * 256; i += blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        reinterpret_cast<float *>(sm)[i] = (float)(h >> 8) * (1.0f / 8388608.0f) - 1.0f;
    }
    __syncthreads();
    int warp = threadIdx.x >> 5;
    if (WS) {
        if (warp < 4) {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
        warp -= 4;
    } else if (warp >= 8) {
        return;
    }
    const int lane = threadIdx.x & 31, grp = warp / 2;
    const unsigned rb = base + (REG ? grp * 49152u : 0u);
    const unsigned sa = rb + (lane & 3) * 8, sb = rb + 16384 + (lane >> 2) * 64;
    const unsigned cbuf = rb + 32768 + (warp & 1) * 4096 + lane * 8;
    float total = 0.f;
    for (int u = 0; u < nunits; ++u) {
        unsigned long long acc[MP][NR];
#pragma unroll
        for (int i = 0; i < MP; ++i)
#pragma unroll
            for (int j = 0; j < NR; ++j) acc[i][j] = 0ull;
        for (int kc = 0; kc < kunit; kc += 16) {
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
                const int cur = (kb / 2) & 1;
                if (kb + 2 < 16) ld(cur ^ 1, kb + 2);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                    for (int i = 0; i < MP; ++i)
#pragma unroll
                        for (int j = 0; j < NR; ++j) f2(acc[i][j], a[cur][kk][i], b[cur][kk][j]);
            }
            __syncwarp();
        }
        if (EPI == 1) {
            float t = 0.f;
#pragma unroll
            for (int i = 0; i < MP; ++i)
#pragma unroll
                for (int j = 0; j < NR; ++j) t += __uint_as_float((unsigned)acc[i][j]) + __uint_as_float((unsigned)(acc[i][j] >> 32));
            total += t;
        } else if (EPI == 2) {
            const unsigned long long al = 0x3fc000003fc00000ull;  // (1.5f, 1.5f)
#pragma unroll
            for (int i = 0; i < MP; ++i)
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    unsigned long long o;
                    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o) : "l"(al), "l"(acc[i][j]));
                    asm volatile("st.shared.b64 [%0], %1;" ::"r"(cbuf + (unsigned)((i * NR + j) % 16) * 256u), "l"(o) : "memory");
                }
        } else if (kunit < 0) {  // never: keeps every accumulator live
#pragma unroll
            for (int i = 0; i < MP; ++i)
#pragma unroll
                for (int j = 0; j < NR; ++j) out[(i * NR + j) * 384 + threadIdx.x] = __uint_as_float((unsigned)acc[i][j]);
        }
    }
    if (total == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

template <bool WS, bool REG, int EPI, bool INIT = true>
void run(const char *name, int nunits, int kunit, float *o)
{
    auto fn = km<WS, REG, EPI, INIT>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fn<<<148, 384, 200 * 1024>>>(o, nunits, kunit);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        fn<<<148, 384, 200 * 1024>>>(o, nunits, kunit);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fl = 148.0 * 256 * (double)nunits * kunit * MP * NR * 4;
    printf("%-28s units %4d x %3d k: %8.2f us  %.1f TFLOP/s (%.3f of 73.5)  %s\n", name, nunits, kunit, best * 1e3,
           fl / best / 1e9, fl / best / 1e9 / 73.5, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    float *o;
    cudaMalloc(&o, 148 * 384 * 4);
    for (int nu : {0, 1, 2, 3, 6}) run<true, true, 2>("ws+regions+sts-epi", nu, 80, o);
    for (int nu : {0, 1, 6}) run<true, true, 2, false>("ws+regions+sts-epi, no init", nu, 80, o);
    for (int nu : {6, 60}) {
        run<false, false, 0>("base", nu, 80, o);
        run<true, false, 0>("ws", nu, 80, o);
        run<true, true, 0>("ws+regions", nu, 80, o);
        run<true, true, 1>("ws+regions+faddsum", nu, 80, o);
        run<true, true, 2>("ws+regions+sts-epi", nu, 80, o);
    }
    run<false, false, 0>("base, one long unit", 1, 480, o);
    run<false, false, 0>("base, one long unit", 1, 4800, o);
    return 0;
}
