// membench.cu — microbenchmark of random-access DRAM efficiency on B200 (evidence for the query
// kernel's memory-access design; not part of the product).  Each variant reads `nrec` random
// records from a 4 GiB array; ncu's dram__bytes_read.sum / (records * record bytes) gives the
// fetch overhead of each access pattern.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
// A: one random 8-byte word per thread
__global__ void k_rand8(const uint64_t* __restrict__ a, uint64_t nwords, int64_t n, uint64_t* out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (int64_t i = t; i < n; i += (int64_t)gridDim.x * blockDim.x) acc += __ldg(a + hash32((uint32_t)i) % nwords);
    if (acc == 12345) out[0] = acc;
}
// A2: same with ld.global.nc.L2::64B hint off -> explicit .L1::no_allocate (LDG.E.64 w/o prefetch)
__global__ void k_rand8_cg(const uint64_t* __restrict__ a, uint64_t nwords, int64_t n, uint64_t* out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t acc = 0;
    for (int64_t i = t; i < n; i += (int64_t)gridDim.x * blockDim.x) acc += __ldcg(a + hash32((uint32_t)i) % nwords);
    if (acc == 12345) out[0] = acc;
}
// B: lane per random row of 104 floats (416 B), 128-bit loads
__global__ void k_row128(const float* __restrict__ x, uint32_t nrows, int64_t n, float* out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0;
    for (int64_t i = t; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4* r = reinterpret_cast<const float4*>(x + (uint64_t)(hash32((uint32_t)i) % nrows) * 104);
#pragma unroll 13
        for (int c = 0; c < 26; ++c) { float4 v = __ldg(r + c); acc += v.x + v.y + v.z + v.w; }
    }
    if (acc == 12345.f) out[0] = acc;
}
// C: lane per random row, 256-bit loads
__global__ void k_row256(const float* __restrict__ x, uint32_t nrows, int64_t n, float* out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0;
    for (int64_t i = t; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float* r = x + (uint64_t)(hash32((uint32_t)i) % nrows) * 104;
#pragma unroll 13
        for (int c = 0; c < 13; ++c) {
            float v0, v1, v2, v3, v4, v5, v6, v7;
            asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3),
                "=f"(v4), "=f"(v5), "=f"(v6), "=f"(v7) : "l"(r + 8 * c));
            acc += v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;
        }
    }
    if (acc == 12345.f) out[0] = acc;
}
// D: warp per random row, coalesced (26 lanes x 16 B)
__global__ void k_rowwarp(const float* __restrict__ x, uint32_t nrows, int64_t n, float* out) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0;
    for (int64_t i = w; i < n; i += nw) {
        const float4* r = reinterpret_cast<const float4*>(x + (uint64_t)(hash32((uint32_t)i) % nrows) * 104);
        if (lane < 26) { float4 v = __ldg(r + lane); acc += v.x + v.y + v.z + v.w; }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
    const size_t bytes = 4ull << 30;
    void* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 1, bytes);
    float* out;
    cudaMalloc(&out, 64);
    const int gran = argc > 1 ? atoi(argv[1]) : -1;
    if (gran >= 0) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t v = 0;
        cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        printf("set L2 fetch granularity %d -> %s, now %zu\n", gran, cudaGetErrorString(e), v);
    } else {
        size_t v = 0;
        cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        printf("default L2 fetch granularity %zu\n", v);
    }
    const int64_t n8 = 64ll << 20, nrow = 4ll << 20;
    const uint32_t nrows = (uint32_t)(bytes / 416);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_rand8<<<148 * 8, 256>>>((const uint64_t*)a, bytes / 8, n8, (uint64_t*)out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("rand8      %.3f ms  %.1f GB/s useful  (%.2f G loads/s)\n", ms, n8 * 8 / ms / 1e6, n8 / ms / 1e6);
        cudaEventRecord(e0);
        k_rand8_cg<<<148 * 8, 256>>>((const uint64_t*)a, bytes / 8, n8, (uint64_t*)out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("rand8_cg   %.3f ms  %.1f GB/s useful\n", ms, n8 * 8 / ms / 1e6);
        cudaEventRecord(e0);
        k_row128<<<148 * 8, 256>>>((const float*)a, nrows, nrow, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("row128     %.3f ms  %.1f GB/s useful\n", ms, nrow * 416 / ms / 1e6);
        cudaEventRecord(e0);
        k_row256<<<148 * 8, 256>>>((const float*)a, nrows, nrow, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("row256     %.3f ms  %.1f GB/s useful\n", ms, nrow * 416 / ms / 1e6);
        cudaEventRecord(e0);
        k_rowwarp<<<148 * 8, 256>>>((const float*)a, nrows, nrow, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("rowwarp    %.3f ms  %.1f GB/s useful\n", ms, nrow * 416 / ms / 1e6);
    }
    cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
