// Micro-benchmark: GPU stores into pinned, device-mapped host memory (the e2e
// explorer's survivor path).  Prints us per launch for sizes x store widths x grids.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/hostwrite scripts/micro/hostwrite.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <class T>
__global__ void wr(T* dst, int64_t n, T v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}
__global__ void empty_k() {}

int main() {
    void* h = nullptr;
    cudaHostAlloc(&h, 64 << 20, cudaHostAllocMapped | cudaHostAllocPortable);
    void* d = nullptr;
    cudaMalloc(&d, 64 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) empty_k<<<1, 32>>>();
    cudaDeviceSynchronize();
    auto run = [&](const char* what, void* base, size_t bytes, int width, int grid) {
        float best = 1e9;
        for (int it = 0; it < 20; ++it) {
            cudaEventRecord(a);
            if (width == 16) wr<uint4><<<grid, 256>>>((uint4*)base, bytes / 16, make_uint4(1, 2, 3, 4));
            else if (width == 8) wr<uint2><<<grid, 256>>>((uint2*)base, bytes / 8, make_uint2(1, 2));
            else wr<uint32_t><<<grid, 256>>>((uint32_t*)base, bytes / 4, 7u);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%s %8zu B  w%2d grid %4d : %8.2f us  %7.2f GB/s\n", what, bytes, width, grid, best * 1e3,
               bytes / (best * 1e-3) / 1e9);
    };
    {
        float best = 1e9;
        for (int it = 0; it < 20; ++it) {
            cudaEventRecord(a);
            empty_k<<<148, 256>>>();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("empty kernel: %.2f us\n", best * 1e3);
    }
    size_t sizes[] = {64 << 10, 512 << 10, 1 << 20, 4 << 20, 16 << 20};
    for (size_t s : sizes)
        for (int w : {4, 16})
            for (int g : {148, 592})
                run("host", h, s, w, g);
    for (size_t s : sizes) run("dev ", d, s, 16, 592);
    return 0;
}
