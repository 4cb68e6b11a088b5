// datagen/fill.cu -- GPU twin of datagen.values(): seeded synthetic inputs.
//
// Harness code (not part of the GEMM product, holds none of its arithmetic).
// Bit-identical to the numpy generator in datagen/__init__.py: see the
// recipe there (splitmix64 over a (seed, mat, global problem, element)
// counter; exact int -> float scaling).  Padding gets NaN.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_kernel(T *dst, int64_t total, uint64_t hi, int64_t rows,
                            int64_t cols, int64_t ld, int64_t stride, int64_t first_id)
{
    const int64_t slot_span = stride > 0 ? stride : ld * cols;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = x / slot_span, w = x - s * slot_span;
        int64_t c = w / ld, r = w - c * ld;
        T v;
        if (r < rows && c < cols) {
            uint64_t e = (uint64_t)(r + c * rows);
            uint64_t ctr = hi ^ ((uint64_t)(first_id + s) * (uint64_t)(rows * cols) + e);
            uint64_t h = splitmix64(ctr);
            if (sizeof(T) == 4)
                v = (T)((double)(h >> 40) * 0x1p-23 - 1.0);
            else
                v = (T)((double)(h >> 11) * 0x1p-52 - 1.0);
        } else {
            v = (T)__longlong_as_double(0x7ff8000000000000ll);
        }
        dst[x] = v;
    }
}

extern "C" int iaat_datagen_fill(int dtype, int64_t seed, int mat, int64_t rows,
                                 int64_t cols, int64_t ld, int64_t stride, int64_t batch,
                                 int64_t first_id, void *dst, void *stream)
{
    if (batch <= 0 || rows <= 0 || cols <= 0) return 0;
    const int64_t span = stride > 0 ? stride : ld * cols;
    const int64_t total = (batch - 1) * (stride > 0 ? stride : 0) + span;
    const uint64_t hi = (uint64_t)((seed * 3 + mat) & 0xFFFF) << 48;
    int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 64) blocks = 148 * 64;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == 0)
        fill_kernel<float><<<(unsigned)blocks, threads, 0, s>>>((float *)dst, total, hi, rows,
                                                                cols, ld, stride, first_id);
    else
        fill_kernel<double><<<(unsigned)blocks, threads, 0, s>>>((double *)dst, total, hi, rows,
                                                                 cols, ld, stride, first_id);
    return (int)cudaGetLastError();
}
