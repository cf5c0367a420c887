// tables.cu -- instance constants staged on the device once per context.
//
// Replaces the per-node, per-pair work of the reference bound
// (bound.hpp:27-44, 79-90: unscheduled list, LagJob vector, std::stable_sort)
// with instance constants: the Johnson order of ALL n jobs for each machine
// pair, computed once.  Restricted to any unscheduled set U it is exactly the
// order stable_sort produces over U listed in ascending job index, because the
// comparator is a strict weak order on (group, key) and ties fall back to the
// input (= job index) order.
#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>

#include "fbb_internal.h"

namespace fbb {

int build_host_tables(const int32_t* p, int n, int m, HostTables* out, std::string* why) {
    if (n < 1 || m < 1) {
        *why = "instance dimensions must be positive";
        return FBB_E_ARG;
    }
    if (n > kMaxJobs || m > kMaxMachines) {
        *why = "instance larger than the device tables support (n <= 256, m <= 64)";
        return FBB_E_RANGE;
    }
    HostTables& h = *out;
    h.n = n;
    h.m = m;
    h.P = m * (m - 1) / 2;
    h.W = (n + 63) / 64;
    h.p.assign(p, p + (size_t)n * m);
    for (int32_t v : h.p)
        if (v < 0) {
            *why = "negative processing time";
            return FBB_E_ARG;
        }
    // instance.hpp:38-45
    h.tails.assign((size_t)n * m, 0);
    for (int j = 0; j < n; ++j) {
        int32_t acc = 0;
        for (int k = m - 1; k >= 0; --k) {
            h.tails[(size_t)j * m + k] = acc;
            acc += h.p[(size_t)j * m + k];
        }
    }
    h.pair_k.clear();
    h.pair_l.clear();
    for (int k = 0; k < m; ++k)
        for (int l = k + 1; l < m; ++l) {  // bound.hpp:97-98 pair order
            h.pair_k.push_back((int16_t)k);
            h.pair_l.push_back((int16_t)l);
        }
    const int P = h.P;
    h.jm.assign((size_t)n * std::max(P, 1), 0);
    h.jw.assign((size_t)n * std::max(P, 1) * 4, 0);
    std::vector<int> order(n);
    std::vector<int64_t> a(n), b(n), lag(n);
    h.packed = true;
    h.max_abs_d = 0;
    h.m_hi = 0;
    h.m_lo = 0;
    h.spos_max = 0;
    for (int q = 0; q < P; ++q) {
        int k = h.pair_k[q], l = h.pair_l[q];
        for (int j = 0; j < n; ++j) {
            a[j] = h.p[(size_t)j * m + k];
            b[j] = h.p[(size_t)j * m + l];
            lag[j] = (int64_t)h.tails[(size_t)j * m + k] - h.p[(size_t)j * m + l] - h.tails[(size_t)j * m + l];
        }
        std::iota(order.begin(), order.end(), 0);
        // bound.hpp:30-36 comparator; stable_sort over ascending job index
        auto in_first = [&](int i) { return a[i] + lag[i] < lag[i] + b[i]; };
        std::stable_sort(order.begin(), order.end(), [&](int i, int j) {
            bool fi = in_first(i), fj = in_first(j);
            if (fi != fj) return fi;
            if (fi) return a[i] + lag[i] < a[j] + lag[j];
            return lag[i] + b[i] > lag[j] + b[j];
        });
        int64_t spos = 0, sneg = 0, cmax = 0;
        for (int i = 0; i < n; ++i) {
            int j = order[i];
            int64_t d = a[j] - b[j];
            int64_t c = a[j] + lag[j];  // = sum_{k <= u < l} p[j][u] >= 0
            if (d < -256 || d > 255 || c < 0 || c >= (1 << 14)) h.packed = false;
            else h.jm[(size_t)i * P + q] = pack_entry(j, (int)d, (int)c);
            int32_t* w = &h.jw[((size_t)i * P + q) * 4];
            w[0] = j;
            w[1] = (int32_t)d;
            w[2] = (int32_t)c;
            h.max_abs_d = std::max<int64_t>(h.max_abs_d, d < 0 ? -d : d);
            (d > 0 ? spos : sneg) += d;
            cmax = std::max(cmax, c);
        }
        h.m_hi = std::max(h.m_hi, spos + cmax);
        h.spos_max = std::max(h.spos_max, spos);
        h.m_lo = std::min(h.m_lo, sneg);
    }
    if (!h.packed) std::fill(h.jm.begin(), h.jm.end(), 0u);
    h.lc_max = 0;
    int64_t load_max = 0, tail_max = 0;
    for (int l = 0; l < m; ++l) {
        int64_t load = 0, tmax = 0;
        for (int j = 0; j < n; ++j) {
            load += h.p[(size_t)j * m + l];
            tmax = std::max<int64_t>(tmax, h.tails[(size_t)j * m + l]);
        }
        h.lc_max = std::max(h.lc_max, load + tmax);
        load_max = std::max(load_max, load);
        tail_max = std::max(tail_max, tmax);
    }
    // 16-bit intermediates (see DevTables::safe16); every bound is exact in int32
    h.safe16 = h.packed ? kTablesPacked : 0;
    // K1 v3: low halves of D lifted by 1 - m_lo, candidates by 1 + spos_max (bound_v3.cu)
    // and the one-machine loads / tails as unsigned 16-bit halves
    if (h.packed && h.max_abs_d <= 127 && (1 - h.m_lo) + (1 + h.spos_max) + h.m_hi <= 32767 &&
        load_max <= 65535 && tail_max < 65535)
        h.safe16 |= kSafeK1x2;
    if (h.packed && h.m_hi <= 32767 && h.m_lo >= -32767) {
        h.safe16 |= kSafeM16;
        if (h.lc_max + h.m_hi <= 32767) {
            h.safe16 |= kSafeLcM16;
            if (h.m_hi <= 16383 && h.m_lo >= -16383) h.safe16 |= kSafeDual16;
        }
    }
    // every head / bound fits int32 comfortably; check the worst makespan
    int64_t total = 0;
    for (int32_t v : h.p) total += v;
    if (total > (int64_t)1 << 30) {
        *why = "total processing time too large for int32 arithmetic (sum of p > 2^30)";
        return FBB_E_RANGE;
    }
    return FBB_OK;
}

template <class T>
static cudaError_t upload(T** dst, const std::vector<T>& src) {
    size_t bytes = std::max<size_t>(src.size(), 1) * sizeof(T);
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) return e;
    if (!src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

int upload_tables(const HostTables& h, DevTables* d, std::string* why) {
    *d = DevTables{};
    d->n = h.n;
    d->m = h.m;
    d->P = h.P;
    d->W = h.W;
    cudaError_t e;
    if ((e = upload(&d->p, h.p)) != cudaSuccess || (e = upload(&d->tails, h.tails)) != cudaSuccess ||
        (e = upload(&d->jm, h.jm)) != cudaSuccess || (e = upload(&d->pair_k, h.pair_k)) != cudaSuccess ||
        (e = upload(&d->pair_l, h.pair_l)) != cudaSuccess) {
        *why = std::string("table upload: ") + cudaGetErrorString(e);
        return FBB_E_CUDA;
    }
    d->safe16 = h.safe16;
    if (!h.packed || !(h.safe16 & kSafeM16)) {  // some kernel runs the unpacked int32 form
        std::vector<int4> w(h.jw.size() / 4);
        std::memcpy(w.data(), h.jw.data(), w.size() * sizeof(int4));
        if ((e = upload(&d->jw, w)) != cudaSuccess) {
            *why = std::string("table upload: ") + cudaGetErrorString(e);
            return FBB_E_CUDA;
        }
    }
    if (h.packed && h.max_abs_d <= 127) {
        std::vector<uint32_t> rp(h.jm.size());
        for (size_t x = 0; x < h.jm.size(); ++x) {
            const uint32_t e = h.jm[x];
            const uint32_t j = (uint32_t)entry_job(e);
            rp[x] = (31u - (j & 31u)) | ((j >> 5) << 5) | ((uint32_t)entry_c(e) << 8) |
                    ((uint32_t)(entry_d(e) & 0xFF) << 24);
        }
        if ((e = upload(&d->rowpk, rp)) != cudaSuccess) {
            *why = std::string("table upload: ") + cudaGetErrorString(e);
            return FBB_E_CUDA;
        }
        for (size_t x = 0; x < h.jm.size(); ++x) {
            const uint32_t en = h.jm[x];
            rp[x] = (uint32_t)entry_job(en) | ((uint32_t)(entry_d(en) & 0xFF) << 8) |
                    ((uint32_t)entry_c(en) << 16);
        }
        if ((e = upload(&d->rowv3, rp)) != cudaSuccess) {
            *why = std::string("table upload: ") + cudaGetErrorString(e);
            return FBB_E_CUDA;
        }
        if (h.safe16 & kSafeK1x2) {
            d->k1_bias = (int32_t)(1 - h.m_lo);
            d->k1_c0 = (int32_t)(1 + h.spos_max);
            for (size_t x = 0; x < h.jm.size(); ++x) {
                const uint32_t en = h.jm[x];
                rp[x] = (uint32_t)entry_job(en) | ((uint32_t)(entry_d(en) & 0xFF) << 8) |
                        ((uint32_t)(entry_c(en) + d->k1_c0) << 16);
            }
            if ((e = upload(&d->rowk1, rp)) != cudaSuccess) {
                *why = std::string("table upload: ") + cudaGetErrorString(e);
                return FBB_E_CUDA;
            }
        }
    }
    return FBB_OK;
}

void free_tables(DevTables* d) {
    cudaFree(d->p);
    cudaFree(d->tails);
    cudaFree(d->jm);
    cudaFree(d->pair_k);
    cudaFree(d->pair_l);
    cudaFree(d->rowpk);
    cudaFree(d->rowv3);
    cudaFree(d->rowk1);
    cudaFree(d->rowk2);
    cudaFree(d->jw);
    *d = DevTables{};
}

}  // namespace fbb
