// bound_kernel.cu -- K1: bound-only evaluation of an arbitrary node batch.
//
// Drop-in for evaluate_batch (bound.hpp:104-109): lb[i] = lower_bound(node_i)
// (bound.hpp:94-101), position-aligned.  Integer max-plus work, no tensor
// cores.  Layout: persistent CTAs, the instance tables (Johnson orders,
// p, tails) staged once per CTA into shared memory; each tile of nodes is
// staged too, then work items (node, machine pair) are spread over the
// threads, lanes of a warp walking the same Johnson position of consecutive
// pairs (conflict-free jm[i*P + q] reads).  Per item the Johnson simulation is
// the 3-op max-plus step  if (j in U) { M = max(M, D + c); D += d; }.
#include <climits>
#include <cstdlib>
#include <string>

#include "fbb_internal.h"

namespace fbb {

namespace {

struct K1Layout {
    size_t jm, pk, p, tl, um, R, Lc, lb, dep, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline K1Layout k1_layout(int n, int m, int P, int tile, bool jm_in_smem) {
    int W32 = (n + 31) / 32;
    K1Layout L;
    size_t o = 0;
    L.jm = o;  o = align16(o + (jm_in_smem ? (size_t)n * P * 4 : 0));
    L.pk = o;  o = align16(o + (size_t)P * 4);
    L.p = o;   o = align16(o + (size_t)n * m * 4);
    L.tl = o;  o = align16(o + (size_t)n * m * 4);
    L.um = o;  o = align16(o + (size_t)tile * W32 * 4);
    L.R = o;   o = align16(o + (size_t)tile * m * 4);
    L.Lc = o;  o = align16(o + (size_t)tile * m * 4);
    L.lb = o;  o = align16(o + (size_t)tile * 4);
    L.dep = o; o = align16(o + (size_t)tile * 4);
    L.total = o;
    return L;
}

// kJmSmem: the Johnson table is staged in shared memory; when it does not fit next
// to the tile (n*P*4 > ~half the opt-in maximum, e.g. 256x20) it is read through L1.
// kWide: the unpacked rows (DevTables::jw) for instances outside the packed range.
template <bool kOneWord, bool kJmSmem, bool kWide>
__global__ void __launch_bounds__(256) k1_bound_kernel(DevTables t, int tile,
                                                      const uint64_t* __restrict__ masks,
                                                      const int32_t* __restrict__ heads,
                                                      const int32_t* __restrict__ depth,
                                                      int64_t count, int32_t* __restrict__ lb_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = t.n, m = t.m, P = t.P, W = t.W;
    const int W32 = (n + 31) / 32;
    const K1Layout L = k1_layout(n, m, P, tile, kJmSmem);
    const uint32_t* s_jm = (kJmSmem && !kWide) ? (const uint32_t*)(smem + L.jm) : t.jm;
    int32_t* s_pk = (int32_t*)(smem + L.pk);
    int32_t* s_p = (int32_t*)(smem + L.p);
    int32_t* s_tl = (int32_t*)(smem + L.tl);
    uint32_t* s_um = (uint32_t*)(smem + L.um);
    int32_t* s_R = (int32_t*)(smem + L.R);
    int32_t* s_Lc = (int32_t*)(smem + L.Lc);
    int32_t* s_lb = (int32_t*)(smem + L.lb);
    int32_t* s_dep = (int32_t*)(smem + L.dep);
    const int tid = threadIdx.x, bd = blockDim.x;

    // stage the instance constants once per CTA
    if (kJmSmem && !kWide)
        for (int x = tid; x < n * P; x += bd) ((uint32_t*)(smem + L.jm))[x] = t.jm[x];
    for (int x = tid; x < P; x += bd) s_pk[x] = (int32_t)t.pair_k[x] | ((int32_t)t.pair_l[x] << 16);
    for (int x = tid; x < n * m; x += bd) {
        s_p[x] = t.p[x];
        s_tl[x] = t.tails[x];
    }

    const int64_t ntiles = (count + tile - 1) / tile;
    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int64_t base = ti * tile;
        const int tn = (int)(count - base < tile ? count - base : tile);
        __syncthreads();  // previous tile fully consumed (and tables staged)
        // ---- stage the tile: unscheduled-job bits, heads, depth
        for (int x = tid; x < tn * W32; x += bd) {
            int tt = x / W32, w = x - tt * W32;
            uint64_t word = masks[(base + tt) * W + (w >> 1)];
            uint32_t half = (w & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
            int lo = w * 32, valid = min(32, n - lo);
            uint32_t vmask = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
            s_um[x] = ~half & vmask;
        }
        for (int x = tid; x < tn * m; x += bd) s_R[x] = heads[base * m + x];
        for (int x = tid; x < tn; x += bd) {
            s_dep[x] = depth[base + x];
            s_lb[x] = 0;
        }
        __syncthreads();
        // ---- per (node, machine): unscheduled load + smallest tail (bound.hpp:61-74)
        for (int x = tid; x < tn * m; x += bd) {
            int tt = x / m, k = x - tt * m;
            int32_t load = 0, mt = INT_MAX;
            const uint32_t* um = s_um + tt * W32;
            for (int j = 0; j < n; ++j) {
                if ((um[j >> 5] >> (j & 31)) & 1u) {
                    load += s_p[j * m + k];
                    mt = min(mt, s_tl[j * m + k]);
                }
            }
            int32_t lc = (mt == INT_MAX) ? 0 : load + mt;
            s_Lc[x] = lc;
            if (s_dep[tt] < n) atomicMax(&s_lb[tt], s_R[x] + lc);  // one-machine term
        }
        __syncthreads();
        // ---- per (node, pair): Johnson with lags in max-plus form (bound.hpp:79-90)
        for (int x = tid; x < tn * P; x += bd) {
            int tt = x / P, q = x - tt * P;
            if (s_dep[tt] >= n) continue;
            int kl = s_pk[q];
            int k = kl & 0xFFFF, l = kl >> 16;
            int32_t D = 0, M = INT_MIN / 2;
            if constexpr (kWide) {
                const uint32_t* um = s_um + tt * W32;
                for (int i = 0; i < n; ++i) {
                    const int4 w = __ldg(t.jw + (size_t)i * P + q);
                    if ((um[w.x >> 5] >> (w.x & 31)) & 1u) {
                        M = max(M, D + w.z);
                        D += w.y;
                    }
                }
            } else if (kOneWord) {
                const uint32_t um = s_um[tt];
#pragma unroll 4
                for (int i = 0; i < n; ++i) {
                    uint32_t e = s_jm[i * P + q];
                    if ((um >> entry_job(e)) & 1u) {
                        M = max(M, D + entry_c(e));
                        D += entry_d(e);
                    }
                }
            } else {
                const uint32_t* um = s_um + tt * W32;
#pragma unroll 4
                for (int i = 0; i < n; ++i) {
                    uint32_t e = s_jm[i * P + q];
                    int j = entry_job(e);
                    if ((um[j >> 5] >> (j & 31)) & 1u) {
                        M = max(M, D + entry_c(e));
                        D += entry_d(e);
                    }
                }
            }
            const int32_t* R = s_R + tt * m;
            int32_t v = s_Lc[tt * m + l] + max(R[l], R[k] + M);
            atomicMax(&s_lb[tt], v);
        }
        __syncthreads();
        for (int x = tid; x < tn; x += bd)
            lb_out[base + x] = (s_dep[x] >= n) ? s_R[x * m + m - 1] : s_lb[x];  // leaf: bound.hpp:95
    }
}

}  // namespace

K1Config k1_config(const DevTables& t, int device) {
    K1Config c;
    {
        // FBB_K1=v1 | v2 forces that kernel (A/B runs); default: v3, else v2, else v1
        const char* sel = getenv("FBB_K1");
        const std::string s = sel ? sel : "";
        if (s != "v1" && s != "v2" && k1v3_config(t, device, &c)) return c;
        if (s != "v1" && k1v2_config(t, device, &c)) return c;
        c = K1Config{};
    }
    c.threads = 256;
    int P = t.P;
    c.tile = P > 0 ? (c.threads * 16 + P - 1) / P : 1024;
    c.tile = c.tile < 32 ? 32 : (c.tile > 1024 ? 1024 : c.tile);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c.smem = k1_layout(t.n, t.m, t.P, c.tile, true).total;
    c.jm_in_smem = c.smem <= (size_t)optin;
    if (!c.jm_in_smem) c.smem = k1_layout(t.n, t.m, t.P, c.tile, false).total;
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    c.wide = !(t.safe16 & kTablesPacked);
    if (c.wide) c.jm_in_smem = false, c.smem = k1_layout(t.n, t.m, t.P, c.tile, false).total;
    auto kern = c.wide ? k1_bound_kernel<false, false, true>
                : t.n <= 32 ? (c.jm_in_smem ? k1_bound_kernel<true, true, false> : k1_bound_kernel<true, false, false>)
                            : (c.jm_in_smem ? k1_bound_kernel<false, true, false> : k1_bound_kernel<false, false, false>);
    // the attribute is per kernel, not per context: allow the device maximum once
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, c.threads, c.smem);
    if (per_sm < 1) per_sm = 1;
    c.blocks = sms * per_sm;
    return c;
}

cudaError_t launch_k1(const DevTables& t, const K1Config& cfg, const uint64_t* masks,
                      const int32_t* heads, const int32_t* depth, int64_t count, int32_t* lb,
                      cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    if (cfg.variant >= 100) return launch_k1v3(t, cfg, masks, heads, depth, count, lb, stream);
    if (cfg.variant != 0) return launch_k1v2(t, cfg, masks, heads, depth, count, lb, stream);
    int64_t ntiles = (count + cfg.tile - 1) / cfg.tile;
    int blocks = (int)(ntiles < cfg.blocks ? ntiles : cfg.blocks);
#define K1_LAUNCH(ONE, SM, WIDE)                                                                      \
    k1_bound_kernel<ONE, SM, WIDE><<<blocks, cfg.threads, cfg.smem, stream>>>(t, cfg.tile, masks, heads, \
                                                                             depth, count, lb)
    if (cfg.wide) {
        K1_LAUNCH(false, false, true);
    } else if (t.n <= 32) {
        if (cfg.jm_in_smem) K1_LAUNCH(true, true, false); else K1_LAUNCH(true, false, false);
    } else {
        if (cfg.jm_in_smem) K1_LAUNCH(false, true, false); else K1_LAUNCH(false, false, false);
    }
#undef K1_LAUNCH
    return cudaGetLastError();
}

}  // namespace fbb
