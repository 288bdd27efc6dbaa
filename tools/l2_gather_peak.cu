// Microbenchmark: the B200's ceiling for random 8-byte fp64 gathers from an
// L2-resident vector (the dual step's x+ gathers), with and without a
// coalesced 12-byte-per-entry index/value stream next to them (the k_csrw long
// pieces' pattern).  Each thread draws its gather positions with a counter hash (no
// index stream in mode 0), so the only L2 traffic is one 32-byte sector per gather.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_gather_peak tools/l2_gather_peak.cu
//   tools/l2_gather_peak            -> one line per (vector size, mode): Ggathers/s, GB/s of sectors
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

// mode 0: hash-drawn gathers only; mode 1: gathers at columns read from a coalesced
// int32 stream + an fp64 value stream (12 B per entry, evict-first), as in k_csrw
template <int MODE, int U>
__global__ void __launch_bounds__(256) k_gather(const double* __restrict__ x, uint32_t mask, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, int64_t per_thread, double* out)
{
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int64_t k = 0; k < per_thread; k += U) {
        int c[U];
        double a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (MODE == 0) {
                c[u] = (int)(mix((uint32_t)(tid * 2654435761u) ^ (uint32_t)(k + u) * 0x9e3779b9u) & mask);
                a[u] = 1.0;
            } else {
                const int64_t q = (k + u) * nth + tid;   // coalesced across the warp
                int v;
                asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(col + q));
                c[u] = v;
                double w;
                asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(w) : "l"(val + q));
                a[u] = w;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += a[u] * __ldg(x + c[u]);
    }
    if (acc == 12345.678) out[0] = acc;   // keep the loads
}

int main()
{
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t NMAX = 1ll << 24;   // 128 MB of fp64
    double *x, *out, *val;
    int32_t* col;
    const int64_t per_thread = 64;
    const int grid = sms * 8, tpb = 256;
    const int64_t nent = per_thread * grid * tpb;
    CK(cudaMalloc(&x, NMAX * sizeof(double)));
    CK(cudaMalloc(&out, 8));
    CK(cudaMalloc(&col, nent * sizeof(int32_t)));
    CK(cudaMalloc(&val, nent * sizeof(double)));
    CK(cudaMemset(x, 0, NMAX * sizeof(double)));
    CK(cudaMemset(val, 0, nent * sizeof(double)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int lg = 20; lg <= 24; ++lg) {   // 8 MB .. 128 MB vectors
        const int64_t n = 1ll << lg;
        // random columns in [0, n) for mode 1 (host-side LCG, uploaded once per size)
        int32_t* h = (int32_t*)malloc(nent * sizeof(int32_t));
        uint64_t s = 88172645463325252ull;
        for (int64_t i = 0; i < nent; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int32_t)(s & (n - 1)); }
        CK(cudaMemcpy(col, h, nent * sizeof(int32_t), cudaMemcpyHostToDevice));
        free(h);
        for (int mode = 0; mode < 2; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 12; ++rep) {
                CK(cudaEventRecord(e0));
                if (mode == 0) k_gather<0, 8><<<grid, tpb>>>(x, (uint32_t)(n - 1), col, val, per_thread, out);
                else k_gather<1, 8><<<grid, tpb>>>(x, (uint32_t)(n - 1), col, val, per_thread, out);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (rep >= 2 && ms < best) best = ms;
            }
            const double g = (double)nent / (best * 1e-3);
            printf("vector %4lld MB mode %d (%s): %.3f ms, %.2f Ggathers/s, gather sectors %.0f GB/s%s\n",
                   (long long)(n * 8 >> 20), mode, mode ? "stream 12 B/entry + gather" : "gather only", best, g * 1e-9,
                   g * 32e-9, mode ? "" : "");
            if (mode == 1) printf("    stream %.0f GB/s, stream+gather sectors %.0f GB/s\n", g * 12e-9, g * 44e-9);
        }
    }
    return 0;
}
