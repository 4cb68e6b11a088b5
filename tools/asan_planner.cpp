// asan_planner.cpp -- the run-time planner (csrc/planner.cpp) and the C
// oracle (oracle/ref_gemm.c) under AddressSanitizer + UndefinedBehaviorSanitizer
// (compute-sanitizer is closed on the GPU pool).  Plans every
// dtype x transposition x (M, N, K) on a grid covering the domain edges,
// padded / misaligned ld's, beta == 0 / != 0 and several batch sizes, and
// prints the count; any out-of-bounds access or UB aborts with a report.
// Built and run by tests/test_host_sanitizers.py.
#include <cstdio>
#include <cstdint>
#include <string>
#include <vector>

#include "planner.h"

int main(int argc, char **argv)
{
    using namespace iaat;
    long n = 0, ok = 0;
    // full grid (argv[1] == "full"): 176928 inputs, ~30 min under the
    // sanitizers; the default grid is the quick one tests run
    const bool full = argc > 1 && std::string(argv[1]) == "full";
    const std::vector<int> dims = full ? std::vector<int>{1, 2, 3, 4, 5, 7, 8, 12, 13, 16, 17, 24, 31, 32, 36, 37, 40,
                                                          44, 48, 52, 56, 61, 64, 68, 72, 76, 79, 80}
                                       : std::vector<int>{1, 13, 37, 64, 80};
    for (int dt = 0; dt < 4; ++dt)
        for (int tr = 0; tr < 4; ++tr)
            for (int M : dims)
                for (int N : dims)
                    for (int K : full ? std::vector<int>{1, 3, 16, 33, 80} : std::vector<int>{3, 80}) {
                        const int64_t lim = (tr == 2) ? 32768 : 512000;
                        if ((int64_t)M * N * K > lim) continue;
                        for (int v = 0; v < 3; ++v) {
                            PlanRequest r;
                            r.dtype = dt;
                            r.transA = tr >> 1;
                            r.transB = tr & 1;
                            r.M = M;
                            r.N = N;
                            r.K = K;
                            const int64_t ra = r.transA ? K : M, ca = r.transA ? M : K;
                            const int64_t rb = r.transB ? N : K, cb = r.transB ? K : N;
                            const int pad = v == 1 ? 3 : 0;
                            r.lda = ra + pad;
                            r.ldb = rb + pad;
                            r.ldc = M + pad;
                            r.sA = r.lda * ca;
                            r.sB = r.ldb * cb;
                            r.sC = r.ldc * N;
                            r.batch = v == 2 ? 1 : (v == 1 ? 777 : 100000);
                            r.beta_zero = (M + N + K + v) & 1;
                            r.alpha_zero = 0;
                            r.align = v == 1 ? 4 : 256;
                            r.sm_count = 148;
                            r.ptr_array = (M * 7 + N) % 5 == 0 ? 1 : 0;
                            Plan p = make_plan(r);
                            std::string js = plan_json(r, p);
                            ++n;
                            ok += p.status == 0 && !js.empty();
                        }
                    }
    std::printf("planned %ld inputs, %ld ok\n", n, ok);
    for (int mode = 0; mode < 2; ++mode)
        for (int M : {1, 9, 12, 15, 33, 80})
            for (int N : {1, 9, 15, 64, 80}) {
                std::string s = paper_tile_json(mode, M, N);
                if (s.empty()) return 1;
            }
    return n > 0 && ok > n / 2 ? 0 : 1;
}
