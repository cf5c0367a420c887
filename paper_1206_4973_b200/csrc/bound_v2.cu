// bound_v2.cu -- K1 (bound-only evaluation of an arbitrary node batch, the drop-in for
// evaluate_batch, bound.hpp:104-109) for instances whose Johnson rows fit the packed
// register-row format (DevTables::rowpk: |p[j][k] - p[j][l]| <= 127).
//
// Mapping: thread (g, q) owns machine pair q; the nodes of a tile are swept NPT at a
// time, so every Johnson row entry read (through L1, coalesced across the pairs of a
// warp) and its (c, -d) extraction serve NPT independent max-plus chains:
//   per node:  sched = sign of (scheduled-job word << code)   (funnel shift + IMAD.HI)
//              ce  = c + sched * kOff      (IMAD: a scheduled job's c never wins)
//              M   = max(M, D + ce);  D += d & ~sched
// then  lb_pair = Lc_l + max(R_l, R_k + M)  (bound.hpp:79-90 in max-plus form; M starts
// at 0 instead of -inf, harmless because heads are non-decreasing in the machine
// index, R_k <= R_l).  The pair maxima of a node are reduced in the warp and folded
// into the node's bound with one shared atomicMax per warp.  The one-machine terms
// (bound.hpp:61-74) come from warp reductions over the unscheduled jobs.
#include <climits>
#include <cstdlib>
#include <string>

#include "fbb_internal.h"

namespace fbb {

namespace {

constexpr int kK1Threads = 192;
// nodes per tile: 32 per pair group (8 sweeps of NPT = 4 nodes), i.e. 32 at m = 20
// (one group of 190 pairs) and up to 608 at m = 5 (19 groups of 10 pairs)
__host__ __device__ inline int k1v2_tile(int P) {
    const int t = (kK1Threads / P) * 32;
    return t < 1024 ? t : 1024;
}
constexpr int32_t kK1Off = 0x100003;

template <int NW, int NPT>
__global__ void __launch_bounds__(kK1Threads) k1v2_kernel(DevTables t, const uint64_t* __restrict__ masks,
                                                          const int32_t* __restrict__ heads,
                                                          const int32_t* __restrict__ depth, int64_t count,
                                                          int32_t* __restrict__ lb_out) {
    const int n = t.n, m = t.m, P = t.P, W = t.W;
    const int kK1Tile = k1v2_tile(P);
    extern __shared__ __align__(16) uint32_t k1smem[];
    uint32_t* s_sched = k1smem;                            // tile * NW: scheduled jobs (+ bits >= n)
    int32_t* s_R = (int32_t*)(s_sched + kK1Tile * NW);     // tile * m
    int32_t* s_Lc = s_R + kK1Tile * m;                     // tile * m
    int32_t* s_lb = s_Lc + kK1Tile * m;                    // tile
    int32_t* s_dep = s_lb + kK1Tile;                       // tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kK1Threads / 32;
    const int G = kK1Threads / P;  // P <= 190 for m <= 20
    const int q = tid % P, g = tid / P;
    const int k = g < G ? t.pair_k[q] : 0, l = g < G ? t.pair_l[q] : 0;
    const uint32_t* __restrict__ rowq = t.rowpk + q;

    const int64_t ntiles = (count + kK1Tile - 1) / kK1Tile;
    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int64_t base = ti * kK1Tile;
        const int tn = (int)(count - base < kK1Tile ? count - base : kK1Tile);
        __syncthreads();  // previous tile consumed
        for (int x = tid; x < kK1Tile * NW; x += kK1Threads) {
            const int tt = x / NW, w = x - tt * NW;
            uint32_t v = 0xFFFFFFFFu;  // absent node / absent jobs: all "scheduled"
            if (tt < tn) {
                const int w64 = w >> 1;
                const uint64_t word = w64 < W ? masks[(base + tt) * W + w64] : ~0ull;
                const uint32_t half = (w & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
                const int valid = min(32, max(0, n - 32 * w));
                const uint32_t vmask = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
                v = half | ~vmask;
            }
            s_sched[x] = v;
        }
        for (int x = tid; x < tn * m; x += kK1Threads) s_R[x] = heads[base * m + x];
        for (int x = tid; x < kK1Tile; x += kK1Threads) {
            s_dep[x] = x < tn ? depth[base + x] : n;
            s_lb[x] = 0;
        }
        __syncthreads();
        // ---- one-machine terms: for n <= 64 a thread per (node, machine) walking the
        // unscheduled jobs; beyond, a warp per item with lanes over the jobs
        if (NW <= 2) {
            for (int x = tid; x < tn * m; x += kK1Threads) {
                const int tt = x / m, kk = x - tt * m;
                int32_t load = 0, mt = INT_MAX;
                for (int w = 0; w < NW; ++w) {
                    uint32_t u = ~s_sched[tt * NW + w];
                    while (u) {
                        const int j = 32 * w + __ffs(u) - 1;
                        u &= u - 1;
                        load += __ldg(t.p + j * m + kk);
                        mt = min(mt, __ldg(t.tails + j * m + kk));
                    }
                }
                const int32_t lc = mt == INT_MAX ? 0 : load + mt;
                s_Lc[x] = lc;
                if (s_dep[tt] < n) atomicMax(&s_lb[tt], s_R[x] + lc);
            }
        } else
        for (int x = warp; x < tn * m; x += nwarps) {
            const int tt = x / m, kk = x - tt * m;
            int32_t load = 0, mt = INT_MAX;
            for (int w = 0; w < NW; ++w) {
                const int j = 32 * w + lane;
                if (!((s_sched[tt * NW + w] >> lane) & 1u)) {
                    load += __ldg(t.p + j * m + kk);
                    mt = min(mt, __ldg(t.tails + j * m + kk));
                }
            }
            load = __reduce_add_sync(0xFFFFFFFFu, load);
            mt = __reduce_min_sync(0xFFFFFFFFu, mt);
            if (lane == 0) {
                const int32_t lc = mt == INT_MAX ? 0 : load + mt;
                s_Lc[x] = lc;
                if (s_dep[tt] < n) atomicMax(&s_lb[tt], s_R[x] + lc);
            }
        }
        __syncthreads();
        // ---- machine pairs: NPT nodes per sweep of the pair's Johnson row
        if (g < G) {
            for (int t0 = g * NPT; t0 < tn; t0 += G * NPT) {
                uint32_t w1[NPT], w2[NPT];
                int32_t D[NPT], Mx[NPT];
#pragma unroll
                for (int u = 0; u < NPT; ++u) {
                    D[u] = 0;
                    Mx[u] = 0;
                    w1[u] = s_sched[(t0 + u < kK1Tile ? t0 + u : 0) * NW];
                    w2[u] = NW >= 2 ? s_sched[(t0 + u < kK1Tile ? t0 + u : 0) * NW + (NW >= 2 ? 1 : 0)] : 0u;
                    if (t0 + u >= tn) w1[u] = w2[u] = 0xFFFFFFFFu;
                }
                const uint32_t sw_sa = (uint32_t)__cvta_generic_to_shared(s_sched + t0 * NW);
#pragma unroll 4
                for (int i = 0; i < n; ++i) {
                    const uint32_t e = __ldg(rowq + i * P);
                    const int32_t c = (int32_t)__byte_perm(e, 0u, 0x4421);
                    const int32_t d = __mulhi((int32_t)e, 256);  // rowpk holds +d (a - b)
#pragma unroll
                    for (int u = 0; u < NPT; ++u) {
                        uint32_t w;
                        if (NW == 1) {
                            w = w1[u];
                        } else if (NW == 2) {
                            w = (e & 32u) ? w2[u] : w1[u];
                        } else {
                            asm("ld.shared.u32 %0, [%1];"
                                : "=r"(w)
                                : "r"(sw_sa + (uint32_t)(u * NW * 4) + ((e >> 3) & 0x1Cu)));
                        }
                        const int32_t sched = __mulhi((int32_t)__funnelshift_l(0u, w, e), 1);
                        const int32_t ce = c + sched * kK1Off;
                        Mx[u] = max(Mx[u], D[u] + ce);
                        D[u] += d & ~sched;
                    }
                }
#pragma unroll
                for (int u = 0; u < NPT; ++u) {
                    const int tt = t0 + u;
                    int32_t v = 0;
                    if (tt < tn && s_dep[tt] < n) {
                        const int32_t* R = s_R + tt * m;
                        v = s_Lc[tt * m + l] + max(R[l], R[k] + Mx[u]);
                    }
                    if (G == 1) {  // the warp's lanes are pairs of the same nodes
                        v = __reduce_max_sync(__activemask(), v);
                        if (lane == 0 && tt < tn) atomicMax(&s_lb[tt], v);
                    } else if (tt < tn) {
                        atomicMax(&s_lb[tt], v);
                    }
                }
            }
        }
        __syncthreads();
        for (int x = tid; x < tn; x += kK1Threads)
            lb_out[base + x] = s_dep[x] >= n ? s_R[x * m + m - 1] : s_lb[x];  // leaf: bound.hpp:95
    }
}

size_t k1v2_smem(const DevTables& t, int NW) {
    const size_t tile = (size_t)k1v2_tile(t.P);
    return tile * NW * 4 + tile * t.m * 8 + tile * 8;
}

template <int NW, int NPT>
int k1v2_blocks(const DevTables& t, int device) {
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaFuncSetAttribute(k1v2_kernel<NW, NPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1v2_kernel<NW, NPT>, kK1Threads,
                                                  k1v2_smem(t, NW));
    return sms * (per_sm < 1 ? 1 : per_sm);
}

}  // namespace

bool k1v2_config(const DevTables& t, int device, K1Config* out) {
    // Measured (r01, bound-only pools): v2 beats the smem-table v1 on every class --
    // 20x20 497 vs 354, 20x5 5626 vs 4837, 50x20 191 vs 128, 100x20 80 vs 65 M nodes/s.
    if (!t.rowpk || t.m > 20 || t.m < 2 || t.n > 256) return false;
    K1Config c;
    c.threads = kK1Threads;
    c.tile = k1v2_tile(t.P);
    c.jm_in_smem = false;
    c.variant = t.n <= 32 ? 1 : (t.n <= 64 ? 2 : 8);
    c.smem = k1v2_smem(t, c.variant);
    c.blocks = c.variant == 1 ? k1v2_blocks<1, 4>(t, device)
                              : (c.variant == 2 ? k1v2_blocks<2, 4>(t, device) : k1v2_blocks<8, 4>(t, device));
    *out = c;
    return true;
}

cudaError_t launch_k1v2(const DevTables& t, const K1Config& cfg, const uint64_t* masks,
                        const int32_t* heads, const int32_t* depth, int64_t count, int32_t* lb,
                        cudaStream_t stream) {
    const int64_t ntiles = (count + cfg.tile - 1) / cfg.tile;
    const int blocks = (int)(ntiles < cfg.blocks ? ntiles : cfg.blocks);
    switch (cfg.variant) {
        case 1: k1v2_kernel<1, 4><<<blocks, kK1Threads, cfg.smem, stream>>>(t, masks, heads, depth, count, lb); break;
        case 2: k1v2_kernel<2, 4><<<blocks, kK1Threads, cfg.smem, stream>>>(t, masks, heads, depth, count, lb); break;
        default: k1v2_kernel<8, 4><<<blocks, kK1Threads, cfg.smem, stream>>>(t, masks, heads, depth, count, lb); break;
    }
    return cudaGetLastError();
}

}  // namespace fbb
