// synth.cu -- synthetic node pools generated on the device (the bounding-stress
// workload of BASELINE configs[4]: a pool filling HBM, bound-only).
//
// Node i is the reference test helper's random_node (tests/helpers.hpp:47-55)
// restated with a counter-based generator instead of std::mt19937: a uniform
// depth in [min_depth, max_depth], then the first `depth` picks of a Fisher-Yates
// shuffle of the n jobs, folded with child_heads (instance.hpp:81-89).  Node i
// depends only on (seed, i), so any sample of the pool can be regenerated and
// checked on the host.
#include "fbb_internal.h"

namespace fbb {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void synth_kernel(DevTables t, uint64_t seed, int64_t count, int min_depth, int max_depth,
                             uint64_t* __restrict__ masks, int32_t* __restrict__ heads,
                             int32_t* __restrict__ depth_out, uint8_t* __restrict__ prefix) {
    const int n = t.n, m = t.m, W = t.W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = seed ^ ((uint64_t)i * 0xD1B54A32D192ED03ull);
        const int span = max_depth - min_depth + 1;
        const int depth = min_depth + (int)(splitmix64(s) % (uint64_t)span);
        uint8_t perm[kMaxJobs];
        for (int j = 0; j < n; ++j) perm[j] = (uint8_t)j;
        uint64_t mk[kMaxWords] = {0, 0, 0, 0};
        int32_t h[kMaxMachines];
        for (int k = 0; k < m; ++k) h[k] = 0;
        for (int d = 0; d < depth; ++d) {
            const int pick = d + (int)(splitmix64(s) % (uint64_t)(n - d));
            const uint8_t job = perm[pick];
            perm[pick] = perm[d];
            perm[d] = job;
            mk[job >> 6] |= 1ull << (job & 63);
            int32_t prev = 0;
            for (int k = 0; k < m; ++k) {
                prev = max(prev, h[k]) + __ldg(t.p + job * m + k);
                h[k] = prev;
            }
            if (prefix) prefix[i * n + d] = job;
        }
        for (int w = 0; w < W; ++w) masks[i * W + w] = mk[w];
        for (int k = 0; k < m; ++k) heads[i * m + k] = h[k];
        depth_out[i] = depth;
    }
}

}  // namespace

cudaError_t launch_synth(const DevTables& t, uint64_t seed, int64_t count, int min_depth, int max_depth,
                         uint64_t* masks, int32_t* heads, int32_t* depth, uint8_t* prefix,
                         cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    synth_kernel<<<(unsigned)blocks, 256, 0, stream>>>(t, seed, count, min_depth, max_depth, masks, heads,
                                                       depth, prefix);
    return cudaGetLastError();
}

}  // namespace fbb
