// ksg_probe.cu -- standalone timing/validation harness for the ksg kernel
// family (paper_2208_09822_b200/csrc/iaat_ksg.cuh) on config-2 shapes, used
// to choose the family's design before it is wired into the planner.
// Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda \
//        -Ipaper_2208_09822_b200/csrc -o ksg_probe tools/experiments/ksg_probe.cu
// Run: ./ksg_probe [filter]   (one line per variant: us, fraction of the HBM roofline, max error)
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "iaat_ksg.cuh"

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

template <bool TA, bool TB, int MR, int NR, int LR, int KC, int KU, int G, int W, int DBG>
__global__ void __launch_bounds__(IAAT_KSG_THREADS_OF(G * W), 1)
    kprobe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, const __grid_constant__ IaatKsgParams p)
{
    iaat::ksg::ksg_body<TA, TB, MR, NR, LR, KC, KU, G, W, DBG>(p, &tmA, &tmB, &tmC);
}

__device__ __forceinline__ uint64_t mix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void kfill(float *x, size_t n, uint64_t seed)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        x[i] = (float)(mix(seed ^ (i * 0x100000001B3ull)) >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

// reference + check of sampled problems: one thread per (problem, i, j)
__global__ void kcheck(const float *A, const float *B, const float *C0, const float *C, int M, int N, int K, int TA,
                       int TB, double alpha, double beta, int64_t nprob, int64_t stepb, unsigned *maxerr)
{
    const int64_t per = (int64_t)M * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nprob * per;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = (t / per) * stepb;
        const int e = (int)(t % per), i = e % M, j = e / M;
        const float *a = A + b * M * K, *bb = B + b * K * N;
        double acc = 0, den = 0;
        for (int k = 0; k < K; ++k) {
            const double x = TA ? a[i * K + k] : a[k * M + i];
            const double y = TB ? bb[k * N + j] : bb[j * K + k];
            acc += x * y;
            den += fabs(x) * fabs(y);
        }
        const double cin = C0[b * per + e];
        const double ref = alpha * acc + beta * cin;
        den = fabs(alpha) * den + fabs(beta) * fabs(cin);
        const double err = fabs((double)C[b * per + e] - ref) / (den > 0 ? den : 1.0);
        atomicMax(maxerr, __float_as_uint((float)err));
    }
}

typedef void (*KFn)(const CUtensorMap, const CUtensorMap, const IaatKsgParams);

struct Variant {
    std::string name;
    bool TA, TB;
    int n, nv, MR, NR, LR, KC, G, W, P, S;
    const void *fn;
};

#define V(name, TA, TB, n, nv, MR, NR, LR, KC, KU, G, W, P, S) \
    Variant{name, TA, TB, n, nv, MR, NR, LR, KC, G, W, P, S, (const void *)kprobe<TA, TB, MR, NR, LR, KC, KU, G, W, 0>}
#define VD(name, TA, TB, n, nv, MR, NR, LR, KC, KU, G, W, P, S, DBG) \
    Variant{name, TA, TB, n, nv, MR, NR, LR, KC, G, W, P, S, (const void *)kprobe<TA, TB, MR, NR, LR, KC, KU, G, W, DBG>}

// smem wavefronts of one epilogue access (element (r0, c) of every lane) for
// C column pitch cp: 128-bit accesses in 4 phases of 8 lanes, 64-bit in 2 of
// 16, 32-bit in 1 of 32; per phase the max number of distinct words per bank.
static int epi_wavefronts(const Variant &v, int cp)
{
    const int LR = v.LR, LC = 32 / LR;
    const bool AK = v.TA, BK = !v.TB;
    const int VA = AK ? 1 : (v.MR % 4 == 0 ? 4 : (v.MR % 2 == 0 ? 2 : 1));
    const int VB = BK ? 1 : (v.NR % 4 == 0 ? 4 : (v.NR % 2 == 0 ? 2 : 1));
    auto row = [&](int ti, int r) { return AK ? ti + LR * r : VA * (ti + LR * (r / VA)) + r % VA; };
    auto col = [&](int tj, int c) { return BK ? tj + LC * c : VB * (tj + LC * (c / VB)) + c % VB; };
    const int V = (!AK && VA >= 2) ? VA : 1;
    int tot = 0;
    for (int c = 0; c < v.NR; ++c) {
        const int nph = V == 4 ? 4 : (V == 2 ? 2 : 1), per = 32 / nph;
        for (int ph = 0; ph < nph; ++ph) {
            int cnt[32][64];
            int nb[32] = {0};
            for (int l = ph * per; l < (ph + 1) * per; ++l) {
                const int ti = l % LR, tj = l / LR;
                const int w0 = col(tj, c) * cp + row(ti, 0);
                for (int e = 0; e < V; ++e) {
                    const int w = w0 + e, b = w & 31;
                    bool seen = false;
                    for (int q = 0; q < nb[b]; ++q) seen |= cnt[b][q] == w;
                    if (!seen) cnt[b][nb[b]++] = w;
                }
            }
            int mx = 0;
            for (int b = 0; b < 32; ++b) mx = std::max(mx, nb[b]);
            tot += mx;
        }
    }
    return tot;
}

static bool encode(CUtensorMap &m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                   uint32_t b0, uint32_t b1, uint32_t b2, int swz)
{
    cuuint64_t dim[3] = {d0, d1, d2};
    cuuint64_t str[2] = {s1, s2};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(base), dim, str,
                                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fprintf(stderr, "encode failed %d\n", (int)r);
    return r == CUDA_SUCCESS;
}

static int rup(int x, int a) { return (x + a - 1) / a * a; }

static void run(const Variant &v, int sms, float *dA, float *dB, float *dC, float *dC0, unsigned *derr)
{
    const int n = v.n, M = n, N = n, K = n, Mv = v.nv, Nv = v.nv, KC = v.KC;
    const int64_t batch = (256ll << 20) / (3ll * n * n * 4);
    const double alpha = 1.5, beta = 0.5;
    typedef Variant Vt;
    (void)sizeof(Vt);
    IaatKsgParams p;
    memset(&p, 0, sizeof p);
    p.batch = batch;
    p.P = v.P;
    p.nunits = (batch + v.P - 1) / v.P;
    p.alpha = alpha;
    p.beta = beta;
    p.M = M;
    p.N = N;
    p.K = K;
    p.Mv = Mv;
    p.Nv = Nv;
    p.S = v.S;
    p.nchunks = (K + KC - 1) / KC;
    p.a_pitch = Mv;
    p.b_pitch = Nv;
    p.a_tx = v.TA ? v.P * Mv * KC * 4 : v.P * KC * Mv * 4;
    p.b_tx = !v.TB ? v.P * Nv * KC * 4 : v.P * KC * Nv * 4;
    p.a_bytes = rup(p.a_tx, 1024);
    p.b_bytes = rup(p.b_tx, 1024);
    p.stage_bytes = p.a_bytes + p.b_bytes;
    int bestwf = 1 << 30, cp = Mv;
    for (int pad = 0; pad < (getenv("PROBE_CP_NOPAD") ? 4 : 32); pad += 4) {
        const int wf = epi_wavefronts(v, Mv + pad);
        if (wf < bestwf) bestwf = wf, cp = Mv + pad;
    }
    p.c_pitch = cp;
    p.c_tx = v.P * Nv * cp * 4;
    p.c_bytes = rup(p.c_tx, 1024);
    p.group_bytes = v.S * p.stage_bytes + p.c_bytes;
    p.beta_zero = 0;
    p.C = reinterpret_cast<char *>(dC);  // C out through global (IAAT_KSG_C_STG)
    p.ldc = M;
    p.sC = (int64_t)M * N;
    const int BR = v.LR * v.MR, BC = (32 / v.LR) * v.NR;
    if (Mv % BR || Nv % BC) {
        printf("%s: block %dx%d does not divide %d\n", v.name.c_str(), BR, BC, n);
        return;
    }
    p.bm = Mv / BR;
    p.wpp = p.bm * (Nv / BC);
    if (p.wpp * v.P != v.W) {
        printf("%s: W=%d != P*wpp=%d\n", v.name.c_str(), v.W, p.wpp * v.P);
        return;
    }
    CUtensorMap tA, tB, tC;
    encode(tC, dC, M, N, batch, (uint64_t)M * 4, (uint64_t)M * N * 4, cp, Nv, v.P, 0);
    // A: TA -> stored K x M (lda = K), else M x K (lda = M)
    const int sw = KC == 32 ? 128 : 64;
    if (v.TA) encode(tA, dA, K, M, batch, (uint64_t)K * 4, (uint64_t)M * K * 4, KC, Mv, v.P, sw);
    else encode(tA, dA, M, K, batch, (uint64_t)M * 4, (uint64_t)M * K * 4, Mv, KC, v.P, 0);
    if (!v.TB) encode(tB, dB, K, N, batch, (uint64_t)K * 4, (uint64_t)K * N * 4, KC, Nv, v.P, sw);
    else encode(tB, dB, N, K, batch, (uint64_t)N * 4, (uint64_t)K * N * 4, Nv, KC, v.P, 0);
    const int smem = IAAT_KSG_BAR_BYTES + 1024 + v.G * p.group_bytes;
    if (smem > 227 * 1024) {
        printf("%s: smem %d too big\n", v.name.c_str(), smem);
        return;
    }
    CK(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int threads = IAAT_KSG_THREADS_OF(v.G * v.W);
    const size_t csz = (size_t)batch * M * N * 4;
    CK(cudaMemcpy(dC, dC0, csz, cudaMemcpyDeviceToDevice));
    void *args[4] = {&tA, &tB, &tC, &p};
    CK(cudaLaunchKernel(v.fn, dim3(sms), dim3(threads), args, smem, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(derr, 0, 4));
    const int64_t nprob = 64, stepb = batch / nprob;
    kcheck<<<1024, 256>>>(dA, dB, dC0, dC, M, N, K, v.TA, v.TB, alpha, beta, nprob, stepb, derr);
    // the last problem (ragged last unit)
    unsigned e1 = 0;
    CK(cudaMemcpy(&e1, derr, 4, cudaMemcpyDeviceToHost));
    float err;
    memcpy(&err, &e1, 4);
    cudaEvent_t e0, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e2);
    for (int w = 0; w < 3; ++w) CK(cudaLaunchKernel(v.fn, dim3(sms), dim3(threads), args, smem, 0));
    float best = 1e30f, tot = 0;
    const int reps = 10;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        cudaLaunchKernel(v.fn, dim3(sms), dim3(threads), args, smem, 0);
        cudaEventRecord(e2);
        cudaEventSynchronize(e2);
        float ms;
        cudaEventElapsedTime(&ms, e0, e2);
        best = fminf(best, ms);
        tot += ms;
    }
    CK(cudaGetLastError());
    const double bytes = 16.0 * n * n * batch;
    const double roof_us = bytes / 6550.1e9 * 1e6;
    const double med_us = tot / reps * 1e3;
    printf("%-34s n=%2d cp=%2d(wf %d) batch=%6lld smem=%6d thr=%3d  best %7.2f us  mean %7.2f us  frac %.3f  err %.2e %s\n",
           v.name.c_str(), n, cp, bestwf, (long long)batch, smem, threads, best * 1e3, med_us, roof_us / med_us, err,
           err <= 1e-5f ? "OK" : "FAIL");
    fflush(stdout);
}

int main(int argc, char **argv)
{
    const char *filter = argc > 1 ? argv[1] : "";
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<Variant> vs = {
        V("NN80_10x10_l4_k16u2_g4w2_p1_s2", false, false, 80, 80, 10, 10, 4, 16, 2, 4, 2, 1, 2),
        V("NN76_10x5_l4_k16u4_g3w4_p1_s3", false, false, 76, 80, 10, 5, 4, 16, 4, 3, 4, 1, 3),
        V("TT76_5x10_l8_k32u4_g2w4_p1_s3", true, true, 76, 80, 5, 10, 8, 32, 4, 2, 4, 1, 3),
        V("NN56_14x7_l4_k16u2_g4w2_p2_s2", false, false, 56, 56, 14, 7, 4, 16, 2, 4, 2, 2, 2),
        V("TT56_7x14_l8_k16u2_g4w2_p2_s2", true, true, 56, 56, 7, 14, 8, 16, 2, 4, 2, 2, 2),
        V("NT56_14x7_l4_k16u2_g4w2_p2_s2", false, true, 56, 56, 14, 7, 4, 16, 2, 4, 2, 2, 2),
        V("NN68_6x9_l4_k16u2_g4w3_p1_s2", false, false, 68, 72, 6, 9, 4, 16, 2, 4, 3, 1, 2),
        // where the time goes (DBG: 1 = no staging, 2 = no epilogue, 3 = neither)
        VD("NN80_10x10_l4_k16u2_g4w2_p1_s2_d1", false, false, 80, 80, 10, 10, 4, 16, 2, 4, 2, 1, 2, 1),
        VD("NN80_10x10_l4_k16u2_g4w2_p1_s2_d2", false, false, 80, 80, 10, 10, 4, 16, 2, 4, 2, 1, 2, 2),
        VD("NN80_10x10_l4_k16u2_g4w2_p1_s2_d3", false, false, 80, 80, 10, 10, 4, 16, 2, 4, 2, 1, 2, 3),
        V("NN80_10x5_l4_k16u4_g3w4_p1_s3", false, false, 80, 80, 10, 5, 4, 16, 4, 3, 4, 1, 3),
        V("NN80_10x10_l4_k16u1_g4w2_p1_s2", false, false, 80, 80, 10, 10, 4, 16, 1, 4, 2, 1, 2),
        V("TT76_5x10_l8_k32u2_g2w4_p1_s3", true, true, 76, 80, 5, 10, 8, 32, 2, 2, 4, 1, 3),
        V("TT80_10x10_l8_k16u2_g2w4_p2_s2", true, true, 80, 80, 10, 10, 8, 16, 2, 2, 4, 2, 2),
        V("TT80_10x10_l8_k16u1_g2w4_p2_s2", true, true, 80, 80, 10, 10, 8, 16, 1, 2, 4, 2, 2),
        V("TT80_10x10_l8_k16u2_g4w2_p1_s2", true, true, 80, 80, 10, 10, 8, 16, 2, 4, 2, 1, 2),
        V("TT80_10x10_l8_k16u1_g4w2_p1_s2", true, true, 80, 80, 10, 10, 8, 16, 1, 4, 2, 1, 2),
        VD("NN80_10x10_l4_k16u1_g4w2_p1_s2_d3", false, false, 80, 80, 10, 10, 4, 16, 1, 4, 2, 1, 2, 3),
        V("NN80_10x5_l4_k16u2_g3w4_p1_s3", false, false, 80, 80, 10, 5, 4, 16, 2, 3, 4, 1, 3),
        VD("NN80_10x5_l4_k16u2_g3w4_p1_s3_d3", false, false, 80, 80, 10, 5, 4, 16, 2, 3, 4, 1, 3, 3),
        VD("NN80_10x5_l4_k16u4_g3w4_p1_s3_d1", false, false, 80, 80, 10, 5, 4, 16, 4, 3, 4, 1, 3, 1),
        VD("NN80_10x5_l4_k16u4_g3w4_p1_s3_d2", false, false, 80, 80, 10, 5, 4, 16, 4, 3, 4, 1, 3, 2),
        VD("NN80_10x5_l4_k16u4_g3w4_p1_s3_d3", false, false, 80, 80, 10, 5, 4, 16, 4, 3, 4, 1, 3, 3),
    };
    size_t maxe = 0;
    for (auto &v : vs) {
        const int64_t batch = (256ll << 20) / (3ll * v.n * v.n * 4);
        maxe = std::max(maxe, (size_t)batch * v.n * v.n);
    }
    float *dA, *dB, *dC, *dC0;
    unsigned *derr;
    CK(cudaMalloc(&dA, maxe * 4));
    CK(cudaMalloc(&dB, maxe * 4));
    CK(cudaMalloc(&dC, maxe * 4));
    CK(cudaMalloc(&dC0, maxe * 4));
    CK(cudaMalloc(&derr, 4));
    kfill<<<4096, 256>>>(dA, maxe, 11);
    kfill<<<4096, 256>>>(dB, maxe, 22);
    kfill<<<4096, 256>>>(dC0, maxe, 33);
    CK(cudaDeviceSynchronize());
    for (auto &v : vs)
        if (strstr(v.name.c_str(), filter)) run(v, sms, dA, dB, dC, dC0, derr);
    return 0;
}
