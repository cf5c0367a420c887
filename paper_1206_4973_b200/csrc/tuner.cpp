// tuner.cpp -- the paper's adaptive pool-size tuner (Algorithm 1,
// PAPER.md:235-279) with the reference's state-machine semantics
// (autotune.hpp:35-156): doubling of grain x units while <= max_batch,
// then geometric probes around the best size (below ascending, then above),
// then fixed.  A window of W observations closes with throughput =
// sum(nodes) / sum(seconds); strict improvement keeps the first best; the
// recorded batch is target(), not the observed pool size (autotune.hpp:76).
//
// B200 re-derivation (the descriptor, not the machine): grain = children per
// K2 tile, base_units = SMs x resident tiles per SM (occupancy API), max_batch
// = what HBM holds for a round (fbb_descriptor in capi.cu), so the doubling
// grid starts at one full wave of the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <set>
#include <string>
#include <vector>

#include "flowbb_b200.h"

struct fbb_tuner {
    int64_t grain, base_units, max_batch;
    int window, probes_per_side;
    int phase = 0;  // 0 doubling, 1 refining, 2 fixed
    int64_t units;
    int64_t iter = 0;
    int64_t window_nodes = 0;
    double window_time = 0.0;
    int64_t best_batch = 0;
    double best_throughput = -1.0;
    std::deque<int64_t> probes;
    std::set<int64_t> visited;
    fbb_tuner_trace_fn trace = nullptr;  // Tuner::set_trace (autotune.hpp)
    void* trace_user = nullptr;
    int window_index = 0;

    int64_t target() const {
        switch (phase) {
            case 0: return grain * units;
            case 1: return probes.front();
            default: return best_batch;
        }
    }

    int64_t scale(int64_t base, int step) const {  // autotune.hpp:134-140
        double factor = std::pow(2.0, (double)step / (2.0 * probes_per_side));
        int64_t raw = (int64_t)std::floor((double)base * factor);
        raw = std::clamp<int64_t>(raw, grain, max_batch);
        raw -= raw % grain;
        return std::max<int64_t>(raw, grain);
    }

    void build_probes() {  // autotune.hpp:123-132
        std::vector<int64_t> cand;
        for (int i = probes_per_side; i >= 1; --i) cand.push_back(scale(best_batch, -i));
        for (int i = 1; i <= probes_per_side; ++i) cand.push_back(scale(best_batch, i));
        for (int64_t c : cand)
            if (!visited.count(c) && std::find(probes.begin(), probes.end(), c) == probes.end())
                probes.push_back(c);
    }

    void advance(int64_t measured, double tp) {  // autotune.hpp:89-121
        const char* what = "";
        if (phase == 0) {
            if (grain * units * 2 <= max_batch) {
                units *= 2;
                what = "double to ";
            } else {
                build_probes();
                phase = probes.empty() ? 2 : 1;
                what = phase == 2 ? "fix at " : "refine at ";
            }
        } else if (phase == 1) {
            probes.pop_front();
            while (!probes.empty() && visited.count(probes.front())) probes.pop_front();
            if (probes.empty()) phase = 2;
            what = phase == 2 ? "fix at " : "refine at ";
        }
        if (trace) {  // the decision strings of the reference's trace
            const std::string decision = std::string(what) + std::to_string(target());
            trace(trace_user, window_index, measured, tp, decision.c_str());
        }
        ++window_index;
    }

    void observe(int64_t nodes, double seconds) {  // autotune.hpp:69-86
        if (phase == 2) return;
        window_nodes += nodes;
        window_time += seconds;
        if (++iter % window != 0) return;
        int64_t measured = target();
        double tp = (double)window_nodes / window_time;
        visited.insert(measured);
        if (tp > best_throughput) {
            best_throughput = tp;
            best_batch = measured;
        }
        window_nodes = 0;
        window_time = 0.0;
        advance(measured, tp);
    }
};

extern "C" {

fbb_tuner* fbb_tuner_create(int32_t grain, int32_t base_units, int64_t max_batch, int window,
                            int probes_per_side) {
    // autotune.hpp:41-49 argument checks
    if (window < 1 || probes_per_side < 0 || grain < 1 || base_units < 1 ||
        max_batch < (int64_t)grain * base_units)
        return nullptr;
    fbb_tuner* t = new fbb_tuner();
    t->grain = grain;
    t->base_units = base_units;
    t->max_batch = max_batch;
    t->window = window;
    t->probes_per_side = probes_per_side;
    t->units = base_units;
    return t;
}

void fbb_tuner_destroy(fbb_tuner* t) { delete t; }

int64_t fbb_tuner_target(const fbb_tuner* t) { return t ? t->target() : 0; }

int fbb_tuner_observe(fbb_tuner* t, int64_t nodes_bounded, double elapsed_seconds) {
    if (!t || !(elapsed_seconds > 0.0)) return FBB_E_ARG;
    t->observe(nodes_bounded, elapsed_seconds);
    return FBB_OK;
}

int fbb_tuner_phase(const fbb_tuner* t) { return t ? t->phase : -1; }
int64_t fbb_tuner_best_batch(const fbb_tuner* t) { return t ? t->best_batch : 0; }
double fbb_tuner_best_throughput(const fbb_tuner* t) { return t ? t->best_throughput : -1.0; }

int fbb_tuner_set_trace(fbb_tuner* t, fbb_tuner_trace_fn fn, void* user) {
    if (!t) return FBB_E_ARG;
    t->trace = fn;
    t->trace_user = user;
    return FBB_OK;
}

}  // extern "C"
