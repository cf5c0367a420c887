// Micro-benchmark: per-round fixed costs on the stream -- small pinned H2D / D2H
// copies vs a kernel with a large __grid_constant__ parameter vs a kernel storing a
// few hundred bytes into mapped host memory.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/latency scripts/micro/latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Big { int64_t v[480]; };  // 3840 B
__global__ void k_param(const __grid_constant__ Big b, int64_t* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = b.v[17] + b.v[479];
}
__global__ void k_param_generic(const __grid_constant__ Big b, const Big* ext, int64_t* out) {
    const Big* p = ext ? ext : &b;
    int64_t s = 0;
    for (int i = threadIdx.x; i < 480; i += blockDim.x) s += p->v[i];
    if (s == 42) out[1] = s;
}
__global__ void k_small(int64_t* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1; }
__global__ void k_hostwrite(int64_t* h, int n) { for (int i = threadIdx.x; i < n; i += blockDim.x) h[i] = i; }

int main() {
    void *hp, *hm, *d;
    cudaMallocHost(&hp, 1 << 20);
    cudaHostAlloc(&hm, 1 << 20, cudaHostAllocMapped);
    cudaMalloc(&d, 1 << 20);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e[4];
    for (auto& x : e) cudaEventCreate(&x);
    Big big{};
    for (int i = 0; i < 480; ++i) big.v[i] = i;
    auto time = [&](const char* what, auto fn) {
        float best = 1e9, sum = 0;
        for (int it = 0; it < 50; ++it) {
            cudaEventRecord(e[0], st);
            fn();
            cudaEventRecord(e[1], st);
            cudaEventSynchronize(e[1]);
            float ms;
            cudaEventElapsedTime(&ms, e[0], e[1]);
            if (it >= 5) { best = ms < best ? ms : best; sum += ms; }
        }
        printf("%-40s best %6.2f us  mean %6.2f us\n", what, best * 1e3, sum / 45 * 1e3);
    };
    time("H2D 448 B pinned", [&] { cudaMemcpyAsync(d, hp, 448, cudaMemcpyHostToDevice, st); });
    time("H2D 448 B + memset 2 KB", [&] { cudaMemcpyAsync(d, hp, 448, cudaMemcpyHostToDevice, st);
                                         cudaMemsetAsync((char*)d + 8192, 0, 2048, st); });
    time("event record x1 extra", [&] { cudaEventRecord(e[2], st); });
    time("H2D 3.5 KB pinned", [&] { cudaMemcpyAsync(d, hp, 3584, cudaMemcpyHostToDevice, st); });
    time("H2D 3.5 KB + memset 2 KB", [&] { cudaMemcpyAsync(d, hp, 3584, cudaMemcpyHostToDevice, st);
                                           cudaMemsetAsync((char*)d + 8192, 0, 2048, st); });
    time("D2H 300 B pinned", [&] { cudaMemcpyAsync(hp, d, 300, cudaMemcpyDeviceToHost, st); });
    time("kernel, tiny param", [&] { k_small<<<1, 32, 0, st>>>((int64_t*)d); });
    time("kernel, 3.8 KB grid_constant param", [&] { k_param<<<1, 32, 0, st>>>(big, (int64_t*)d); });
    time("kernel x2 (K2+place-like), 3.8 KB params", [&] { k_param<<<296, 192, 0, st>>>(big, (int64_t*)d);
                                                          k_param<<<171, 256, 0, st>>>(big, (int64_t*)d); });
    time("kernel x2, tiny params", [&] { k_small<<<296, 192, 0, st>>>((int64_t*)d); k_small<<<171, 256, 0, st>>>((int64_t*)d); });
    time("kernel generic-read param 480x", [&] { k_param_generic<<<296, 192, 0, st>>>(big, nullptr, (int64_t*)d); });
    time("kernel generic-read global 480x", [&] { k_param_generic<<<296, 192, 0, st>>>(big, (const Big*)d, (int64_t*)d); });
    time("kernel writes 300 B to mapped host", [&] { k_hostwrite<<<1, 64, 0, st>>>((int64_t*)hm, 38); });
    time("H2D + kernel + D2H (current pattern)", [&] { cudaMemcpyAsync(d, hp, 3584, cudaMemcpyHostToDevice, st);
                                                       k_small<<<296, 192, 0, st>>>((int64_t*)d);
                                                       k_small<<<171, 256, 0, st>>>((int64_t*)d);
                                                       cudaMemcpyAsync(hp, d, 300, cudaMemcpyDeviceToHost, st); });
    time("param kernels + mapped write (proposed)", [&] { k_param<<<296, 192, 0, st>>>(big, (int64_t*)d);
                                                          k_param<<<171, 256, 0, st>>>(big, (int64_t*)d);
                                                          k_hostwrite<<<1, 64, 0, st>>>((int64_t*)hm, 38); });
    return 0;
}
