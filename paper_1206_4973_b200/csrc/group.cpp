// group.cpp -- fbb_group_*: the multi-device explorer inside one process (include/flowbb_b200.h).
//
// The reference splits every pool over k backends and merges the results in order
// (split_slices / evaluate_multi / merge_slices, backend.hpp:73-158); the paper runs that
// split over the GPUs of one host.  Here, as in the multi-process
// driver (parallel.py), the split is of the pending TREE: member i explores its own
// subtrees with the fused device round, and the members exchange only the incumbent
// (solve mode) and, when one runs dry, whole subtrees.  One persistent host thread per
// member runs its rounds (calls on different contexts are independent, see the header);
// the exchange runs on the calling thread between steps, so no member ever waits on a
// collective in the middle of a round.
#include <algorithm>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "flowbb_b200.h"

namespace {

struct Transfer {
    int donor, receiver;
    int64_t count;
};

// The deterministic rebalancing plan of parallel.py plan_transfers: receivers in ascending
// (pending, index) order below `low` take half the difference (<= cap) from the richest
// member with more than 2 * low that has not donated in this step.
std::vector<Transfer> plan_transfers(std::vector<int64_t> est, int64_t low, int64_t cap) {
    const int G = (int)est.size();
    std::vector<int> order(G);
    for (int i = 0; i < G; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        return est[a] != est[b] ? est[a] < est[b] : a < b;
    });
    std::vector<char> donated(G, 0);
    std::vector<Transfer> plan;
    for (int rcv : order) {
        if (est[rcv] >= low) break;
        int d = -1;
        for (int i = 0; i < G; ++i) {
            if (donated[i] || i == rcv || est[i] <= 2 * low) continue;
            if (d < 0 || est[i] > est[d]) d = i;  // ties: the lowest index
        }
        if (d < 0) break;
        const int64_t k = std::min<int64_t>(cap, (est[d] - est[rcv]) / 2);
        if (k <= 0) continue;
        plan.push_back({d, rcv, k});
        est[d] -= k;
        est[rcv] += k;
        donated[d] = 1;
    }
    return plan;
}

}  // namespace

struct fbb_group {
    std::vector<fbb_ctx*> ctx;
    int n = 0, m = 0;
    int frozen = 1;
    int status = FBB_OK, fail_member = -1;
    std::string msg;

    // worker pool: one persistent thread per member
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv_go, cv_done;
    int64_t generation = 0;
    int busy = 0;
    bool quit = false;
    int64_t job_target = 0;
    int job_rounds = 1;
    std::vector<int> job_rc;
    std::vector<std::vector<fbb_round_t>> job_rec;
    std::vector<int64_t> job_done;
    std::vector<double> dev_ms;  // per member, summed round device time of the current call

    int fail(int code, int member, const std::string& m_) {
        status = code;
        fail_member = member;
        msg = m_;
        return code;
    }
    int member_fail(int i, int rc) {
        char buf[512] = {0};
        int dev = -1;
        fbb_last_error(ctx[i], &dev, buf, sizeof buf);
        return fail(rc, i, "member " + std::to_string(i) + " (device " + std::to_string(dev) + "): " + buf);
    }

    void worker(int i) {
        int64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu);
            cv_go.wait(lk, [&] { return quit || generation != seen; });
            if (quit) return;
            seen = generation;
            const int64_t target = job_target;
            const int rounds = job_rounds;
            lk.unlock();
            int64_t done = 0;
            int rc = fbb_explorer_run(ctx[i], &target, 1, rounds, 0, job_rec[i].data(), &done);
            lk.lock();
            job_rc[i] = rc;
            job_done[i] = done;
            if (--busy == 0) cv_done.notify_all();
        }
    }

    // one step's rounds on every member, concurrently; returns the first failure
    int run_members(int64_t target, int rounds) {
        for (auto& v : job_rec)
            if ((int)v.size() < rounds) v.resize(rounds);
        {
            std::lock_guard<std::mutex> lk(mu);
            job_target = target;
            job_rounds = rounds;
            busy = (int)ctx.size();
            ++generation;
        }
        cv_go.notify_all();
        std::unique_lock<std::mutex> lk(mu);
        cv_done.wait(lk, [&] { return busy == 0; });
        for (size_t i = 0; i < ctx.size(); ++i)
            if (job_rc[i] != FBB_OK) return member_fail((int)i, job_rc[i]);
        return FBB_OK;
    }

    ~fbb_group() {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv_go.notify_all();
        for (auto& t : workers)
            if (t.joinable()) t.join();
        for (fbb_ctx* c : ctx) fbb_destroy(c);
    }
};

namespace {

struct MemberState {
    int32_t incumbent = INT32_MAX, found = 0;
    int64_t pending = 0, totals[4] = {0, 0, 0, 0};
};

int member_state(fbb_group* g, int i, MemberState* s) {
    int rc = fbb_explorer_state(g->ctx[i], &s->incumbent, &s->found, nullptr, &s->pending, s->totals);
    return rc == FBB_OK ? FBB_OK : g->member_fail(i, rc);
}

}  // namespace

extern "C" {

fbb_group* fbb_group_create(const int* devices, int G, const int32_t* p, int n, int m) {
    if (!devices || G < 1 || G > 64) return nullptr;
    fbb_group* g = new fbb_group();
    g->n = n;
    g->m = m;
    for (int i = 0; i < G; ++i) {
        fbb_ctx* c = fbb_create(devices[i], p, n, m);
        if (!c) {
            delete g;
            return nullptr;
        }
        g->ctx.push_back(c);
    }
    g->job_rc.assign(G, FBB_OK);
    g->job_rec.assign(G, std::vector<fbb_round_t>(1));
    g->job_done.assign(G, 0);
    g->dev_ms.assign(G, 0.0);
    for (int i = 0; i < G; ++i) g->workers.emplace_back([g, i] { g->worker(i); });
    return g;
}

void fbb_group_destroy(fbb_group* g) { delete g; }

int fbb_group_size(const fbb_group* g) { return g ? (int)g->ctx.size() : 0; }

fbb_ctx* fbb_group_context(fbb_group* g, int i) {
    if (!g || i < 0 || i >= (int)g->ctx.size()) return nullptr;
    return g->ctx[i];
}

int fbb_group_last_error(const fbb_group* g, int* member, char* msg, size_t cap) {
    if (!g) return FBB_E_ARG;
    if (member) *member = g->fail_member;
    if (msg && cap > 0) {
        std::strncpy(msg, g->msg.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    return g->status;
}

int fbb_group_reset(fbb_group* g, const uint8_t* prefix, const int32_t* depth, int64_t count,
                    int32_t ub, int frozen) {
    if (!g) return FBB_E_ARG;
    if (count < 0 || (count > 0 && (!prefix || !depth))) return g->fail(FBB_E_ARG, -1, "invalid nodes");
    const int G = (int)g->ctx.size();
    g->frozen = frozen ? 1 : 0;
    // split_slices (backend.hpp:73-84): ceil(count / G) per slice, the last one short
    const int64_t per = (count + G - 1) / G;
    for (int i = 0; i < G; ++i) {
        const int64_t off = std::min<int64_t>(count, per * i);
        const int64_t len = std::min<int64_t>(count - off, per);
        int rc = fbb_explorer_reset(g->ctx[i], len ? prefix + off * g->n : nullptr,
                                    len ? depth + off : nullptr, len, ub, frozen);
        if (rc != FBB_OK) return g->member_fail(i, rc);
    }
    return FBB_OK;
}

int fbb_group_start_solve(fbb_group* g, int32_t ub) {
    if (!g) return FBB_E_ARG;
    g->frozen = 0;
    fbb_round_t r0;
    int rc = fbb_explorer_start_solve(g->ctx[0], ub, &r0);
    if (rc != FBB_OK) return g->member_fail(0, rc);
    for (size_t i = 1; i < g->ctx.size(); ++i) {
        rc = fbb_explorer_reset(g->ctx[i], nullptr, nullptr, 0, r0.incumbent, 0);
        if (rc != FBB_OK) return g->member_fail((int)i, rc);
    }
    return FBB_OK;
}

int fbb_group_run(fbb_group* g, int64_t target, int64_t max_steps, int rounds_per_step,
                  int balance_every, int64_t budget, fbb_group_stats_t* stats) {
    if (!g) return FBB_E_ARG;
    if (target < 1 || rounds_per_step < 1) return g->fail(FBB_E_ARG, -1, "target and rounds_per_step must be >= 1");
    const int G = (int)g->ctx.size(), n = g->n;
    if (balance_every < 1) balance_every = 1;
    const auto t0 = std::chrono::steady_clock::now();
    double exch_ms = 0.0;
    int64_t steps = 0, rounds = 0, moved = 0;
    std::fill(g->dev_ms.begin(), g->dev_ms.end(), 0.0);
    std::vector<MemberState> st(G);
    std::vector<uint8_t> buf_pre;
    std::vector<int32_t> buf_dep;
    int rc;
    while (steps < max_steps) {
        rc = g->run_members(target, rounds_per_step);
        if (rc != FBB_OK) return rc;
        for (int i = 0; i < G; ++i) {
            rounds += g->job_done[i];
            for (int64_t r = 0; r < g->job_done[i]; ++r) g->dev_ms[i] += g->job_rec[i][r].round_ms;
        }
        ++steps;
        // ---- exchange (calling thread; the members are idle)
        const auto x0 = std::chrono::steady_clock::now();
        int64_t pend = 0, bounded = 0;
        int32_t inc = INT32_MAX;
        for (int i = 0; i < G; ++i) {
            if ((rc = member_state(g, i, &st[i])) != FBB_OK) return rc;
            pend += st[i].pending;
            bounded += st[i].totals[1];
            inc = std::min(inc, st[i].incumbent);
        }
        if (!g->frozen)  // the UB min-allreduce
            for (int i = 0; i < G; ++i)
                if (st[i].incumbent > inc && (rc = fbb_explorer_set_incumbent(g->ctx[i], inc)) != FBB_OK)
                    return g->member_fail(i, rc);
        bool stop = pend == 0 || (budget > 0 && bounded >= budget);
        if (!stop && G > 1 && steps % balance_every == 0) {
            std::vector<int64_t> est(G);
            for (int i = 0; i < G; ++i) est[i] = st[i].pending;
            const int64_t low = std::max<int64_t>(1, target / std::max(1, n));
            for (const Transfer& t : plan_transfers(est, low, 1 << 16)) {
                buf_pre.resize((size_t)t.count * n);
                buf_dep.resize((size_t)t.count);
                int64_t got = 0;
                if ((rc = fbb_explorer_take(g->ctx[t.donor], t.count, buf_pre.data(), buf_dep.data(), &got)) != FBB_OK)
                    return g->member_fail(t.donor, rc);
                if ((rc = fbb_explorer_push(g->ctx[t.receiver], buf_pre.data(), buf_dep.data(), got)) != FBB_OK)
                    return g->member_fail(t.receiver, rc);
                moved += got;
            }
        }
        exch_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - x0).count();
        if (stop) break;
    }
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->steps = steps;
        stats->rounds = rounds;
        int32_t inc = INT32_MAX;
        int32_t found = 0;
        for (int i = 0; i < G; ++i) {
            if ((rc = member_state(g, i, &st[i])) != FBB_OK) return rc;
            stats->branched += st[i].totals[0];
            stats->bounded += st[i].totals[1];
            stats->pruned += st[i].totals[2];
            stats->leaves += st[i].totals[3];
            stats->pending += st[i].pending;
            inc = std::min(inc, st[i].incumbent);
            found |= st[i].found;
        }
        stats->incumbent = inc;
        stats->found = found;
        stats->transfers = moved;
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        stats->device_ms_max = *std::max_element(g->dev_ms.begin(), g->dev_ms.end());
        stats->exchange_ms = exch_ms;
    }
    return FBB_OK;
}

int fbb_plan_transfers(const int64_t* pending, int G, int64_t low, int64_t cap, int64_t* plan,
                       int* count) {
    if (!pending || !plan || !count || G < 1) return FBB_E_ARG;
    const std::vector<Transfer> p = plan_transfers(std::vector<int64_t>(pending, pending + G), low, cap);
    for (size_t i = 0; i < p.size(); ++i) {
        plan[3 * i] = p[i].donor;
        plan[3 * i + 1] = p[i].receiver;
        plan[3 * i + 2] = p[i].count;
    }
    *count = (int)p.size();
    return FBB_OK;
}

int fbb_group_best(fbb_group* g, int32_t* value, int32_t* schedule) {
    if (!g) return FBB_E_ARG;
    int32_t best = INT32_MAX;
    int who = -1;
    for (size_t i = 0; i < g->ctx.size(); ++i) {
        int32_t v = INT32_MAX;
        int f = fbb_explorer_best(g->ctx[i], &v, nullptr);
        if (f < 0) return g->member_fail((int)i, f);
        if (f && v < best) {  // strict: the lowest member index wins ties
            best = v;
            who = (int)i;
        }
    }
    if (value) *value = best;
    if (who < 0) return 0;
    if (schedule) {
        int f = fbb_explorer_best(g->ctx[who], &best, schedule);
        if (f < 0) return g->member_fail(who, f);
    }
    return 1;
}

}  // extern "C"
