// Microbenchmark: HBM streaming rate of (a) a TMA bulk-copy ring (1 producer lane +
// 16 consumer warps, as in k_spmv) vs (b) plain vectorised loads, on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tma tools/bench_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c)
{ asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n)
{ asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b)
{ asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph)
{
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                     smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma(void* d, const void* s, uint32_t n, uint64_t* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
}

template <int NST, int STAGE, int NCOPY>
__global__ void __launch_bounds__(544, 1) k_tma(const char* src, size_t chunks, double* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[NST], empty[NST];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc = 0;
    if (w == 16) {
        if (lane == 0) {
            uint32_t eph = 0; int s = 0, it = 0;
            for (size_t c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
                if (it >= NST) { mbar_wait(&empty[s], (eph >> s) & 1); eph ^= 1u << s; }
                mbar_expect(&full[s], STAGE);
                for (int k = 0; k < NCOPY; ++k)
                    tma(sm + s * STAGE + k * (STAGE / NCOPY), src + c * STAGE + k * (STAGE / NCOPY), STAGE / NCOPY, &full[s]);
                s = s + 1 == NST ? 0 : s + 1;
            }
        }
    } else {
        uint32_t fph = 0; int s = 0;
        for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
            mbar_wait(&full[s], (fph >> s) & 1); fph ^= 1u << s;
            const double* d = (const double*)(sm + s * STAGE);
            for (int i = w * 32 + lane; i < STAGE / 8; i += 512) acc += d[i];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            s = s + 1 == NST ? 0 : s + 1;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void k_ldg(const double2* src, size_t n, double* out)
{
    double acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double2 v = __ldcs(&src[i]);
        acc += v.x + v.y;
    }
    if (acc == 12345.0) out[0] = acc;
}

template <int NST, int STAGE, int NCOPY>
void run_tma(const char* d, size_t bytes, double* out, int sms)
{
    auto k = k_tma<NST, STAGE, NCOPY>;
    int smem = NST * STAGE;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    size_t chunks = bytes / STAGE;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<sms, 544, smem>>>(d, chunks, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<sms, 544, smem>>>(d, chunks, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("TMA ring NST=%2d STAGE=%6d B copies/stage=%d : %7.1f GB/s  (%s)\n", NST, STAGE, NCOPY,
           5.0 * chunks * STAGE / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    size_t bytes = 4ull << 30;
    char* d; double* out;
    cudaMalloc(&d, bytes); cudaMalloc(&out, 8);
    cudaMemset(d, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run_tma<6, 32768, 1>(d, bytes, out, sms);
    run_tma<6, 32768, 4>(d, bytes, out, sms);
    run_tma<12, 16384, 1>(d, bytes, out, sms);
    run_tma<12, 16384, 2>(d, bytes, out, sms);
    run_tma<3, 65536, 1>(d, bytes, out, sms);
    run_tma<24, 8192, 1>(d, bytes, out, sms);
    run_tma<8, 24576, 2>(d, bytes, out, sms);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bpsm : {4, 8}) {
        k_ldg<<<sms * bpsm, 256>>>((const double2*)d, bytes / 16, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_ldg<<<sms * bpsm, 256>>>((const double2*)d, bytes / 16, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("LDG.128 grid=%d x 256 : %7.1f GB/s\n", sms * bpsm, 5.0 * bytes / (ms / 1e3) / 1e9);
    }
    return 0;
}
