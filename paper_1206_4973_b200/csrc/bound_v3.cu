// bound_v3.cu -- K1 (bound-only evaluation of an arbitrary node batch, the drop-in for
// evaluate_batch, bound.hpp:104-109) with two nodes per register (16x2 SIMD).
//
// Applies when the packed register rows exist (|d| <= 127, c < 2^14), m <= 20 and the
// biased 16-bit chains below fit the instance (DevTables::safe16 & kSafeK1x2, decided
// by build_host_tables' range analysis; Taillard 200x20 uses ~12K of the 32K range).
//
// The max-plus chain of pair q over a node's unscheduled set U (bound.hpp:37-43 unrolled,
// fbb_internal.h pack_entry comment):  per Johnson position i with job j,
//     if (j in U) { M = max(M, D + c); D += d; }
// Two nodes a (low half) and b (high half) share one 32-bit register per quantity:
//   sel  = [j in U_a] + 65536 [j in U_b]        (from a per-tile membership table)
//   D2  += d * sel                              IMAD (FMA pipe): a masked add of d to both
//                                               halves, exact because the low half never
//                                               borrows -- it carries D_a + k1_bias >= 1
//   ce2  = (c + k1_c0, c + k1_c0) & (sel * 0xFFFF)   IMAD + LOP3: members' candidates,
//                                               lifted by k1_c0 > every D, so a
//                                               non-member's candidate D + 0 always loses
//   M2   = max(D2 + ce2, M2)                    VIADDMNMX.S16x2
// i.e. 2 ALU + 2 FMA instructions per two nodes and position; M_a = lo(M2) - k1_bias -
// k1_c0, M_b = hi(M2) - k1_c0.  (A node's true M is >= 0 -- its first member has D = 0.)
//
// Mapping: thread (g, q) owns machine pair q of node group g and sweeps the pair's row
// once for kNP = 16 nodes.  Per position: one coalesced row load (L1, prefetched a
// position ahead) and two 128-bit shared loads of the job's 8 sel words.  The pair bound
// Lc_l + max(R_l, R_k + M) (bound.hpp:79-90) and the one-machine terms (bound.hpp:61-74)
// are int32.
#include <climits>
#include <cstdlib>

#include "fbb_internal.h"

namespace fbb {

namespace {

constexpr int kK3Threads = 192;
constexpr int kNP = 16;  // nodes per thread (8 SIMD pairs)

// A tile is kNP nodes per pair group; G = tile / kNP groups of P threads (G * P <= 192),
// fewer than 192 / P when the tile's shared arrays would not fit (small m, large n).
__host__ __device__ inline size_t k3_align(size_t x) { return (x + 15) & ~size_t(15); }

struct K1v3Layout {
    size_t sched, R, Lc, mt, lb, dep, tab, total;
};

__host__ __device__ inline K1v3Layout k1v3_layout(int n, int m, int T, int NW) {
    const int G = T / kNP;
    K1v3Layout L;
    size_t o = 0;
    L.sched = o; o = k3_align(o + (size_t)T * NW * 4);  // scheduled words (absent: all ones)
    L.R = o;     o = k3_align(o + (size_t)T * m * 4);
    L.Lc = o;    o = k3_align(o + (size_t)T * m * 4);  // loads, then Lc = load + min tail
    L.mt = o;    o = k3_align(o + (size_t)T * m * 4);  // min tails (0xFFFF: none)
    L.lb = o;    o = k3_align(o + (size_t)T * 4);
    L.dep = o;   o = k3_align(o + (size_t)T * 4);
    L.tab = o;   o = k3_align(o + (size_t)G * n * kNP * 2);  // [group][job][8 sel words]
    L.total = o;
    return L;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
    return d;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

template <int NW>
__global__ void __launch_bounds__(kK3Threads, 4) k1v3_kernel(DevTables t, const uint64_t* __restrict__ masks,
                                                             const int32_t* __restrict__ heads,
                                                             const int32_t* __restrict__ depth, int64_t count,
                                                             int32_t* __restrict__ lb_out, int T) {
    const int n = t.n, m = t.m, P = t.P, W = t.W;
    const int G = T / kNP;
    const K1v3Layout L = k1v3_layout(n, m, T, NW);
    extern __shared__ __align__(16) unsigned char k3smem[];
    uint32_t* s_sched = (uint32_t*)(k3smem + L.sched);
    int32_t* s_R = (int32_t*)(k3smem + L.R);
    int32_t* s_Lc = (int32_t*)(k3smem + L.Lc);
    int32_t* s_mt = (int32_t*)(k3smem + L.mt);
    int32_t* s_lb = (int32_t*)(k3smem + L.lb);
    int32_t* s_dep = (int32_t*)(k3smem + L.dep);
    uint32_t* s_tab = (uint32_t*)(k3smem + L.tab);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kK3Threads / 32;
    const int q = tid % P, g = tid / P;
    const bool active = g < G;
    const int k = active ? t.pair_k[q] : 0, l = active ? t.pair_l[q] : 0;
    const uint32_t* __restrict__ rowq = t.rowk1 + q;
    const uint32_t tab_sa = (uint32_t)__cvta_generic_to_shared(s_tab) + (uint32_t)(g * n * kNP * 2);
    const int32_t bias = t.k1_bias, c0 = t.k1_c0;
    const uint32_t half_b = (uint32_t)n * 16u;  // byte distance between the two table planes

    const int64_t ntiles = (count + T - 1) / T;
    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const int64_t base = ti * T;
        const int tn = (int)(count - base < T ? count - base : T);
        __syncthreads();  // previous tile consumed
        for (int x = tid; x < T * NW; x += kK3Threads) {
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
        for (int x = tid; x < tn * m; x += kK3Threads) {
            s_R[x] = heads[base * m + x];
            s_Lc[x] = 0;
            s_mt[x] = 0xFFFF;
        }
        for (int x = tid; x < T; x += kK3Threads) {
            s_dep[x] = x < tn ? depth[base + x] : n;
            s_lb[x] = 0;
        }
        __syncthreads();
        // membership table: word (group gg, job j, u) = [j in U of node gg*16 + 2u] +
        // 65536 [j in U of node gg*16 + 2u + 1], stored as two 16-byte halves per job in
        // separate planes, [gg][u / 4][j][u % 4]: the lanes of a warp (machine pairs at
        // one Johnson position, i.e. random jobs) then spread their 128-bit loads over all
        // 8 bank groups (j mod 8) instead of 4 (2j mod 8 with 32-byte job rows)
        for (int x = tid; x < G * n * 8; x += kK3Threads) {
            const int gg = x / (n * 8), rem = x - gg * n * 8, j = rem >> 3, u = rem & 7;
            const int node0 = gg * kNP + 2 * u;
            const uint32_t a = (~s_sched[node0 * NW + (j >> 5)] >> (j & 31)) & 1u;
            const uint32_t b = (~s_sched[(node0 + 1) * NW + (j >> 5)] >> (j & 31)) & 1u;
            s_tab[gg * n * 8 + (u >> 2) * n * 4 + j * 4 + (u & 3)] = a | (b << 16);
        }
        __syncthreads();  // membership table complete
        // one-machine terms (bound.hpp:61-74) over the same table, 16 nodes per thread:
        // thread (group gg, machine kk, job chunk ch) walks the jobs j = ch, ch + C, ... once
        // and folds p[j][kk] into the nodes' loads (IMAD by the sel word: two u16 sums per
        // register, the low half never carries) and tail[j][kk] into their minima (members
        // only: non-members see 0xFFFF, VIMNMX.U16x2); chunks combine by shared atomics.
        // For n <= 64 the per-(node, machine) walk below is cheaper (few jobs per chunk).
        if (NW >= 4) {
            const int C = max(1, kK3Threads / (G * m));
            for (int x = tid; x < G * m * C; x += kK3Threads) {
                const int gg = x / (m * C), rem = x - gg * m * C, kk = rem / C, ch = rem - kk * C;
                uint32_t ld2[kNP / 2], mn2[kNP / 2];
#pragma unroll
                for (int u = 0; u < kNP / 2; ++u) {
                    ld2[u] = 0u;
                    mn2[u] = 0xFFFFFFFFu;
                }
                const uint32_t tg = (uint32_t)__cvta_generic_to_shared(s_tab) + (uint32_t)(gg * n * kNP * 2);
                for (int j = ch; j < n; j += C) {
                    const uint32_t pj = (uint32_t)__ldg(t.p + j * m + kk);
                    const uint32_t t2 = (uint32_t)__ldg(t.tails + j * m + kk) * 0x10001u;  // (t, t)
                    const uint4 s0 = lds128(tg + (uint32_t)j * 16u), s1 = lds128(tg + (uint32_t)(j + n) * 16u);
                    const uint32_t sel[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                    for (int u = 0; u < kNP / 2; ++u) {
                        ld2[u] += pj * sel[u];
                        mn2[u] = __vminu2(mn2[u], t2 | ~(sel[u] * 0xFFFFu));
                    }
                }
#pragma unroll
                for (int u = 0; u < kNP / 2; ++u) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int tt = gg * kNP + 2 * u + h;
                        if (tt >= tn) continue;
                        const int32_t ld = (int32_t)(h ? ld2[u] >> 16 : ld2[u] & 0xFFFFu);
                        const int32_t mn = (int32_t)(h ? mn2[u] >> 16 : mn2[u] & 0xFFFFu);
                        if (C == 1) {
                            s_Lc[tt * m + kk] = ld;
                            s_mt[tt * m + kk] = mn;
                        } else {
                            if (ld) atomicAdd(&s_Lc[tt * m + kk], ld);
                            if (mn != 0xFFFF) atomicMin(&s_mt[tt * m + kk], mn);
                        }
                    }
                }
            }
        }
        __syncthreads();
        for (int x = tid; x < tn * m; x += kK3Threads) {
            const int tt = x / m;
            int32_t lc;
            if (NW >= 4) {
                const int32_t mn = s_mt[x];
                lc = mn == 0xFFFF ? 0 : s_Lc[x] + mn;  // no unscheduled job: 0
            } else {  // n <= 64: a thread per (node, machine) walking the unscheduled jobs
                const int kk = x - tt * m;
                int32_t load = 0, mt = INT_MAX;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    uint32_t u = ~s_sched[tt * NW + w];
                    while (u) {
                        const int j = 32 * w + __ffs(u) - 1;
                        u &= u - 1;
                        load += __ldg(t.p + j * m + kk);
                        mt = min(mt, __ldg(t.tails + j * m + kk));
                    }
                }
                lc = mt == INT_MAX ? 0 : load + mt;
            }
            s_Lc[x] = lc;
            if (s_dep[tt] < n) atomicMax(&s_lb[tt], s_R[x] + lc);
        }
        __syncthreads();
        // ---- machine pairs: one sweep of the pair's row for the group's 16 nodes
        if (active) {
            uint32_t D2[kNP / 2], M2[kNP / 2];
#pragma unroll
            for (int u = 0; u < kNP / 2; ++u) {
                D2[u] = (uint32_t)bias;  // (D_b, D_a + bias) = (0, bias)
                M2[u] = 0x80008000u;     // (-32768, -32768)
            }
            const uint32_t* rp = rowq;
            uint32_t e = __ldg(rp);
            for (int i = 0; i < n; ++i) {
                rp += P;
                const uint32_t en = i + 1 < n ? __ldg(rp) : 0u;  // next position
                const uint32_t at = tab_sa + (e & 0xFFu) * 16u;
                const uint4 s0 = lds128(at), s1 = lds128(at + half_b);
                const uint32_t cb2 = prmt(e, 0x3232u);            // (c + c0, c + c0)
                const int32_t d = (int32_t)prmt(e, 0x9991u);      // int8 d, sign-extended
                const uint32_t sel[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                for (int u = 0; u < kNP / 2; ++u) {
                    const uint32_t ce2 = cb2 & (sel[u] * 0xFFFFu);
                    M2[u] = __viaddmax_s16x2(D2[u], ce2, M2[u]);
                    D2[u] += (uint32_t)d * sel[u];
                }
                e = en;
            }
#pragma unroll
            for (int u = 0; u < kNP / 2; ++u) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int tt = g * kNP + 2 * u + h;
                    const int32_t Mx = h ? ((int32_t)M2[u] >> 16) - c0
                                         : (int32_t)(int16_t)(M2[u] & 0xFFFFu) - bias - c0;
                    int32_t v = 0;
                    if (tt < tn && s_dep[tt] < n) {
                        const int32_t* R = s_R + tt * m;
                        v = s_Lc[tt * m + l] + max(R[l], R[k] + Mx);
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
        for (int x = tid; x < tn; x += kK3Threads)
            lb_out[base + x] = s_dep[x] >= n ? s_R[x * m + m - 1] : s_lb[x];  // leaf: bound.hpp:95
    }
}

template <int NW>
int k1v3_blocks(const DevTables& t, int device, size_t smem) {
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaFuncSetAttribute(k1v3_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);  // > 64 KB cap
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1v3_kernel<NW>, kK3Threads, smem);
    return sms * (per_sm < 1 ? 1 : per_sm);
}

}  // namespace

bool k1v3_config(const DevTables& t, int device, K1Config* out) {
    if (!t.rowk1 || !(t.safe16 & kSafeK1x2) || t.m > 20 || t.m < 2 || t.n > 256) return false;
    K1Config c;
    c.threads = kK3Threads;
    c.jm_in_smem = false;
    const int NW = t.n <= 32 ? 1 : (t.n <= 64 ? 2 : (t.n <= 128 ? 4 : 8));
    // as many pair groups as the 192 threads hold, while the tile's arrays stay <= 64 KB
    // (>= 3 CTAs per SM)
    int G = kK3Threads / t.P;
    while (G > 1 && k1v3_layout(t.n, t.m, kNP * G, NW).total > (64u << 10)) --G;
    c.tile = kNP * G;
    c.variant = 100 + NW;
    c.smem = k1v3_layout(t.n, t.m, c.tile, NW).total;
    switch (NW) {
        case 1: c.blocks = k1v3_blocks<1>(t, device, c.smem); break;
        case 2: c.blocks = k1v3_blocks<2>(t, device, c.smem); break;
        case 4: c.blocks = k1v3_blocks<4>(t, device, c.smem); break;
        default: c.blocks = k1v3_blocks<8>(t, device, c.smem); break;
    }
    *out = c;
    return true;
}

cudaError_t launch_k1v3(const DevTables& t, const K1Config& cfg, const uint64_t* masks, const int32_t* heads,
                        const int32_t* depth, int64_t count, int32_t* lb, cudaStream_t stream) {
    const int64_t ntiles = (count + cfg.tile - 1) / cfg.tile;
    const int blocks = (int)(ntiles < cfg.blocks ? ntiles : cfg.blocks);
#define K1V3(NW) \
    k1v3_kernel<NW><<<blocks, kK3Threads, cfg.smem, stream>>>(t, masks, heads, depth, count, lb, cfg.tile)
    switch (cfg.variant) {
        case 101: K1V3(1); break;
        case 102: K1V3(2); break;
        case 104: K1V3(4); break;
        default: K1V3(8); break;
    }
#undef K1V3
    return cudaGetLastError();
}

}  // namespace fbb
