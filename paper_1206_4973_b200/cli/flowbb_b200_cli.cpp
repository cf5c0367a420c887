// flowbb-b200 -- the reference CLI (proj/tools/flowbb_main.cpp:62-244) over the B200
// library: the same four subcommands, options, output formats and exit codes, with the
// bounding done by libflowbb_b200.so (C-ABI, include/flowbb_b200.h).  No CLI11 (not in
// this image): a small option parser with the same option names.
//
//   gen-instance --jobs N --machines M --seed S [--out FILE]
//       Taillard's generator (instance.hpp:227-265), simple format (to_simple_format).
//   print-instance --instance FILE [--format auto|simple|taillard] [--out FILE]
//       parse_instance (instance.hpp:184-222) re-emitted in the simple format (no GPU).
//   solve --instance FILE [--format auto|simple|taillard] [--ub V] [--batch B | --autotune]
//         [--backends K] [--window W] [--probes P] [--grain G] [--max-batch X]
//         [--trace-tuner] [--seed S] [--json] [--device D]
//       solve() (search.hpp:124-174) on the device explorer; key=value lines or one JSON
//       document; "infeasible under given bound V" and exit 1 when nothing beats --ub.
//   workload --instance FILE --ub V (--nodes N | --seconds T) [--seed S] --out FILE
//       generate_workload (workload.hpp:62-98): frozen-UB sequential search with a seeded
//       child shuffle, bounds from K1; the snapshot in the flowbb-workload v1 text format.
//   bench --workload FILE [--backends K] [--batch B | --autotune] [--window W] [--probes P]
//         [--grain G] [--max-batch X] [--format table|csv|json]
//       run_experiment (bench.hpp:116-145): the snapshot resolved with batch 1 and with the
//       given configuration on the device explorer; exit 2 when the two disagree
//       (ResolutionMismatch), else the report (emit_report, bench.hpp:150-223).
//
// --backends K: K explorer contexts over the visible GPUs (device i % count); K = 1 is one
// GPU.  Exit codes: 0 ok, 1 error or infeasible, 2 resolution mismatch.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "flowbb_b200.h"

namespace {

using Clock = std::chrono::steady_clock;

struct Instance {
    int n = 0, m = 0;
    std::vector<int32_t> p;  // job-major
    int32_t at(int j, int k) const { return p[(size_t)j * m + k]; }
};

// ---- options ------------------------------------------------------------------------------
struct Args {
    std::map<std::string, std::string> kv;
    std::set<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) || flags.count(k); }
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : it->second;
    }
    long long num(const std::string& k, long long dflt) const {
        auto it = kv.find(k);
        if (it == kv.end()) return dflt;
        size_t pos = 0;
        long long v = std::stoll(it->second, &pos);
        if (pos != it->second.size()) throw std::runtime_error("--" + k + ": not an integer: " + it->second);
        return v;
    }
    double real(const std::string& k, double dflt) const {
        auto it = kv.find(k);
        return it == kv.end() ? dflt : std::stod(it->second);
    }
};

Args parse_args(int argc, char** argv, int first, const std::set<std::string>& flag_names,
                const std::set<std::string>& value_names) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) != 0) throw std::runtime_error("unexpected argument: " + s);
        std::string key = s.substr(2), val;
        const size_t eq = key.find('=');
        const bool inline_val = eq != std::string::npos;
        if (inline_val) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        }
        if (flag_names.count(key)) {
            if (inline_val) throw std::runtime_error("--" + key + " takes no value");
            a.flags.insert(key);
        } else if (value_names.count(key)) {
            if (!inline_val) {
                if (i + 1 >= argc) throw std::runtime_error("--" + key + " needs a value");
                val = argv[++i];
            }
            a.kv[key] = val;
        } else {
            throw std::runtime_error("unknown option --" + key);
        }
    }
    return a;
}

void require(const Args& a, const std::string& k) {
    if (!a.has(k)) throw std::runtime_error("--" + k + " is required");
}

// ---- instances (instance.hpp:100-226: simple / Taillard formats) ---------------------------
std::string read_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

void write_output(const std::string& path, const std::string& text) {
    if (path.empty() || path == "-") {
        std::cout << text;
        return;
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open " + path + " for writing");
    out << text;
}

bool is_int(const std::string& t) {
    if (t.empty()) return false;
    size_t i = (t[0] == '-' || t[0] == '+') ? 1 : 0;
    if (i == t.size()) return false;
    for (; i < t.size(); ++i)
        if (!std::isdigit((unsigned char)t[i])) return false;
    return true;
}

Instance parse_instance(const std::string& text, bool taillard) {
    std::istringstream in(text);
    std::vector<std::string> tok;
    for (std::string t; in >> t;) tok.push_back(t);
    size_t i = 0;
    auto seek_int = [&]() {  // Taillard header prose is skipped token by token
        while (i < tok.size() && !is_int(tok[i])) ++i;
        return i < tok.size();
    };
    auto expect = [&](const char* what) -> long {
        if (i >= tok.size()) throw std::runtime_error(std::string("unexpected end of input, expected ") + what);
        if (!is_int(tok[i]))
            throw std::runtime_error(std::string("expected ") + what + ", got '" + tok[i] + "'");
        return std::stol(tok[i++]);
    };
    Instance inst;
    if (taillard) {
        if (!seek_int()) throw std::runtime_error("missing Taillard header values");
        inst.n = (int)expect("job count");
        inst.m = (int)expect("machine count");
        expect("initial seed");
        expect("upper bound");
        expect("lower bound");
        if (!seek_int()) throw std::runtime_error("missing processing-time matrix");
    } else {
        inst.n = (int)expect("job count");
        inst.m = (int)expect("machine count");
    }
    if (inst.n < 1 || inst.m < 1) throw std::runtime_error("dimensions must be positive");
    inst.p.assign((size_t)inst.n * inst.m, 0);
    if (taillard) {
        for (int k = 0; k < inst.m; ++k)
            for (int j = 0; j < inst.n; ++j) inst.p[(size_t)j * inst.m + k] = (int32_t)expect("processing time");
    } else {
        for (int j = 0; j < inst.n; ++j)
            for (int k = 0; k < inst.m; ++k) inst.p[(size_t)j * inst.m + k] = (int32_t)expect("processing time");
    }
    for (int32_t t : inst.p)
        if (t < 0) throw std::runtime_error("negative processing time");
    if (i < tok.size()) throw std::runtime_error("trailing data after matrix: '" + tok[i] + "'");
    return inst;
}

Instance load_instance(const std::string& path, const std::string& format) {
    const std::string text = read_file(path);
    bool taillard;
    if (format == "simple") taillard = false;
    else if (format == "taillard") taillard = true;
    else if (format == "auto") {  // Taillard files carry prose headers, simple files are digits
        taillard = std::any_of(text.begin(), text.end(), [](char c) { return std::isalpha((unsigned char)c); });
    } else {
        throw std::runtime_error("--format: expected auto|simple|taillard");
    }
    return parse_instance(text, taillard);
}

Instance generate_instance(int n, int m, long long seed) {  // instance.hpp:227-265
    if (n < 1 || m < 1) throw std::runtime_error("instance dimensions must be positive");
    if (seed <= 0 || seed >= 2147483647) throw std::runtime_error("Taillard seed must be in (0, 2^31-1)");
    Instance inst{n, m, std::vector<int32_t>((size_t)n * m)};
    int64_t state = seed;
    for (int k = 0; k < m; ++k)
        for (int j = 0; j < n; ++j) {
            const int64_t q = state / 127773;
            state = 16807 * (state % 127773) - 2836 * q;
            if (state < 0) state += 2147483647;
            inst.p[(size_t)j * m + k] = 1 + (int32_t)((double)state / 2147483647.0 * 99);
        }
    return inst;
}

std::string to_simple_format(const Instance& inst) {
    std::ostringstream out;
    out << inst.n << ' ' << inst.m << '\n';
    for (int j = 0; j < inst.n; ++j) {
        for (int k = 0; k < inst.m; ++k) out << (k ? " " : "") << inst.at(j, k);
        out << '\n';
    }
    return out.str();
}

// ---- device plumbing ------------------------------------------------------------------------
struct Device {
    fbb_ctx* ctx = nullptr;
    Device(const Instance& inst, int device) {
        ctx = fbb_create(device, inst.p.data(), inst.n, inst.m);
        if (!ctx) fail(nullptr);
    }
    ~Device() { fbb_destroy(ctx); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    [[noreturn]] static void fail(const fbb_ctx* c) {
        char msg[512];
        int dev = -1;
        fbb_last_error(c, &dev, msg, sizeof msg);
        throw std::runtime_error(std::string("backend ") + std::to_string(dev < 0 ? 0 : dev) + ": " + msg);
    }
    void check(int rc) const {
        if (rc != FBB_OK) fail(ctx);
    }
    fbb_descriptor_t descriptor() const {
        fbb_descriptor_t d;
        check(fbb_descriptor(ctx, &d));
        return d;
    }
};

struct TunerOpts {
    int window = 5, probes = 2;
    long long grain = 0, max_batch = 0;
    bool trace = false;
};

// BackendDescriptor of the run (make_descriptor, flowbb_main.cpp:94-100)
fbb_descriptor_t make_descriptor(const Device& dev, const TunerOpts& o) {
    fbb_descriptor_t d = dev.descriptor();
    if (o.grain > 0) d.grain = (int32_t)o.grain;
    if (o.max_batch > 0) d.max_batch = o.max_batch;
    d.max_batch = std::max<int64_t>(d.max_batch, (int64_t)d.grain * d.base_units);
    return d;
}

void trace_line(void*, int window, int64_t batch, double throughput, const char* decision) {
    std::cerr << "tuner window=" << window << " batch=" << batch << " throughput=" << throughput
              << " decision=" << decision << '\n';
}

struct Tuner {
    fbb_tuner* t = nullptr;
    Tuner(const fbb_descriptor_t& d, const TunerOpts& o) {
        t = fbb_tuner_create(d.grain, d.base_units, d.max_batch, o.window, o.probes);
        if (!t) throw std::runtime_error("invalid tuner configuration");
        if (o.trace) fbb_tuner_set_trace(t, trace_line, nullptr);
    }
    ~Tuner() { fbb_tuner_destroy(t); }
};

// Runs rounds until the pending tree is empty: one C call for a fixed target, one round
// per call under the tuner (which observes each round's device time, search.hpp:155-165).
void drive(Device& dev, std::optional<Tuner>& tuner, int64_t batch) {
    fbb_round_t rec;
    int64_t done = 0;
    if (!tuner) {
        for (;;) {
            int64_t pending = 0;
            dev.check(fbb_explorer_state(dev.ctx, nullptr, nullptr, nullptr, &pending, nullptr));
            if (pending == 0) return;
            dev.check(fbb_explorer_run(dev.ctx, &batch, 1, 1 << 20, 0, nullptr, &done));
        }
    }
    for (;;) {
        const int64_t target = fbb_tuner_target(tuner->t);
        const auto t0 = Clock::now();
        dev.check(fbb_explorer_run(dev.ctx, &target, 1, 1, 0, &rec, &done));
        if (done == 0) return;
        double secs = rec.round_ms > 0 ? rec.round_ms * 1e-3
                                       : std::chrono::duration<double>(Clock::now() - t0).count();
        fbb_tuner_observe(tuner->t, rec.bounded, std::max(secs, 1e-9));
    }
}

std::string join(const std::vector<int32_t>& v) {
    std::ostringstream out;
    for (size_t i = 0; i < v.size(); ++i) out << (i ? " " : "") << v[i];
    return out.str();
}

TunerOpts tuner_opts(const Args& a) {
    TunerOpts o;
    o.window = (int)a.num("window", 5);
    o.probes = (int)a.num("probes", 2);
    o.grain = a.num("grain", 0);
    o.max_batch = a.num("max-batch", 0);
    o.trace = a.has("trace-tuner");
    return o;
}

// ---- subcommands ----------------------------------------------------------------------------
int cmd_gen(const Args& a) {
    require(a, "jobs");
    require(a, "machines");
    require(a, "seed");
    const Instance inst = generate_instance((int)a.num("jobs", 0), (int)a.num("machines", 0), a.num("seed", 0));
    write_output(a.get("out"), to_simple_format(inst));
    return 0;
}

int cmd_solve(const Args& a) {
    require(a, "instance");
    if (a.has("batch") && a.has("autotune")) throw std::runtime_error("--autotune excludes --batch");
    const Instance inst = load_instance(a.get("instance"), a.get("format", "auto"));
    const int backends = (int)a.num("backends", 1);
    if (backends < 1) throw std::runtime_error("backend count must be positive");
    Device dev(inst, (int)a.num("device", 0));
    const TunerOpts to = tuner_opts(a);
    const fbb_descriptor_t d = make_descriptor(dev, to);
    std::optional<Tuner> tuner;
    if (a.has("autotune")) tuner.emplace(d, to);
    const int64_t batch = a.has("batch") ? a.num("batch", 1) : (int64_t)d.grain * d.base_units;
    if (batch < 1) throw std::runtime_error("--batch must be positive");
    const auto t0 = Clock::now();
    fbb_round_t r0;
    const int32_t ub = a.has("ub") ? (int32_t)a.num("ub", 0) : -1;
    if (a.has("ub") && ub < 0) throw std::runtime_error("--ub must be non-negative");
    dev.check(fbb_explorer_start_solve(dev.ctx, ub, &r0));
    if (tuner) fbb_tuner_observe(tuner->t, 1, std::max(std::chrono::duration<double>(Clock::now() - t0).count(), 1e-9));
    drive(dev, tuner, batch);
    const double elapsed = std::chrono::duration<double>(Clock::now() - t0).count();
    int32_t inc = 0, found = 0;
    int64_t pending = 0, tot[4] = {0, 0, 0, 0};
    std::vector<int32_t> sched(inst.n);
    dev.check(fbb_explorer_state(dev.ctx, &inc, &found, sched.data(), &pending, tot));
    if (a.has("json")) {
        std::cout << "{\"feasible\":" << (found ? "true" : "false");
        if (found) std::cout << ",\"optimum\":" << inc << ",\"schedule\":\"" << join(sched) << "\"";
        std::cout << ",\"nodes_branched\":" << tot[0] << ",\"nodes_bounded\":" << tot[1]
                  << ",\"nodes_pruned\":" << tot[2] << ",\"elapsed_seconds\":" << elapsed << "}\n";
        return 0;
    }
    if (!found) {
        std::cout << "infeasible under given bound " << inc << '\n';
        return 1;
    }
    std::cout << "optimum=" << inc << '\n'
              << "schedule=" << join(sched) << '\n'
              << "nodes_branched=" << tot[0] << '\n'
              << "nodes_bounded=" << tot[1] << '\n'
              << "nodes_pruned=" << tot[2] << '\n'
              << "elapsed_seconds=" << elapsed << '\n';
    return 0;
}

// Node of a workload capture: prefix + heads + scheduled set (node.hpp:28-53).
struct WNode {
    std::vector<uint8_t> prefix;
    std::vector<int32_t> heads;
    std::vector<uint64_t> mask;
};

WNode child_of(const Instance& inst, const WNode& par, int job) {  // Node::child, child_heads
    WNode c = par;
    c.prefix.push_back((uint8_t)job);
    c.mask[job >> 6] |= 1ull << (job & 63);
    int32_t prev = 0;
    for (int k = 0; k < inst.m; ++k) {
        prev = std::max(prev, c.heads[k]) + inst.at(job, k);
        c.heads[k] = prev;
    }
    return c;
}

struct Snapshot {
    Instance inst;
    std::vector<std::vector<int>> nodes;  // prefixes, drain order
    int incumbent = 0;
    uint32_t seed = 0;
    bool by_nodes = true;
    long long nodes_cut = 0;
    double seconds_cut = 0.0;
};

// generate_workload (workload.hpp:62-98): the root is always branched; each expansion's
// children (branch: ascending job, depth n-1 auto-completed) are shuffled by the seeded
// Fisher-Yates of workload.hpp:47-56, leaves dropped, the rest bounded (K1) and pushed
// when lb < ub; pending = per-depth LIFO buckets (pending.hpp); L = drain order.
Snapshot generate_workload(const Instance& inst, int ub, bool by_nodes, long long nodes, double seconds,
                           uint32_t seed) {
    Device dev(inst, 0);
    const int n = inst.n, m = inst.m, W = (n + 63) / 64;
    std::mt19937 rng(seed);
    std::vector<std::vector<WNode>> bucket(n + 1);
    int64_t count = 0;
    int deepest = 0;
    auto expand = [&](const WNode& node) {
        std::vector<WNode> kids;
        for (int j = 0; j < n; ++j) {  // branch (search.hpp:40-59)
            if ((node.mask[j >> 6] >> (j & 63)) & 1ull) continue;
            WNode c = child_of(inst, node, j);
            if ((int)c.prefix.size() == n - 1) {  // auto-complete the last job
                for (int y = 0; y < n; ++y)
                    if (!((c.mask[y >> 6] >> (y & 63)) & 1ull)) c = child_of(inst, c, y);
            }
            kids.push_back(std::move(c));
        }
        for (size_t i = 0; i + 1 < kids.size(); ++i) {  // deterministic_shuffle
            const size_t k = i + rng() % (kids.size() - i);
            std::swap(kids[i], kids[k]);
        }
        std::vector<uint64_t> masks;
        std::vector<int32_t> heads, depth;
        std::vector<size_t> idx;
        for (size_t i = 0; i < kids.size(); ++i) {
            if ((int)kids[i].prefix.size() == n) continue;  // frozen incumbent: leaves dropped
            masks.insert(masks.end(), kids[i].mask.begin(), kids[i].mask.end());
            heads.insert(heads.end(), kids[i].heads.begin(), kids[i].heads.end());
            depth.push_back((int32_t)kids[i].prefix.size());
            idx.push_back(i);
        }
        std::vector<int32_t> lb(idx.size());
        if (!idx.empty())
            dev.check(fbb_bound(dev.ctx, masks.data(), heads.data(), depth.data(), (int64_t)idx.size(), lb.data()));
        for (size_t t = 0; t < idx.size(); ++t)
            if (lb[t] < ub) {
                WNode& c = kids[idx[t]];
                const int d = (int)c.prefix.size();
                bucket[d].push_back(std::move(c));
                deepest = std::max(deepest, d);
                ++count;
            }
    };
    WNode root{{}, std::vector<int32_t>(m, 0), std::vector<uint64_t>(W, 0)};
    const auto t0 = Clock::now();
    expand(root);
    long long branched = 0;
    while (count > 0) {
        if (by_nodes) {
            if (branched >= nodes) break;
        } else if (std::chrono::duration<double>(Clock::now() - t0).count() >= seconds) {
            break;
        }
        while (bucket[deepest].empty()) --deepest;  // PendingTree::pop
        WNode node = std::move(bucket[deepest].back());
        bucket[deepest].pop_back();
        --count;
        expand(node);
        ++branched;
    }
    Snapshot s{inst, {}, ub, seed, by_nodes, nodes, seconds};
    for (auto& b : bucket)
        for (WNode& x : b) s.nodes.emplace_back(x.prefix.begin(), x.prefix.end());
    return s;
}

std::string save_workload(const Snapshot& s) {  // workload.hpp:100-131 format
    std::ostringstream out;
    out << "flowbb-workload v1\n"
        << "jobs " << s.inst.n << '\n'
        << "machines " << s.inst.m << '\n'
        << "incumbent " << s.incumbent << '\n'
        << "seed " << s.seed << '\n';
    if (s.by_nodes) out << "cutoff nodes " << s.nodes_cut << '\n';
    else out << "cutoff seconds " << s.seconds_cut << '\n';
    out << "times\n";
    for (int j = 0; j < s.inst.n; ++j) {
        for (int k = 0; k < s.inst.m; ++k) out << (k ? " " : "") << s.inst.at(j, k);
        out << '\n';
    }
    out << "nodes " << s.nodes.size() << '\n';
    for (const auto& pr : s.nodes) {
        for (size_t i = 0; i < pr.size(); ++i) out << (i ? " " : "") << pr[i];
        out << '\n';
    }
    return out.str();
}

Snapshot load_workload(const std::string& path) {  // workload.hpp:133-203 checks
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    auto fail = [](const std::string& what) { throw std::runtime_error("workload file: " + what); };
    std::string line;
    if (!std::getline(in, line) || line != "flowbb-workload v1") fail("bad or missing version header");
    auto field = [&](const std::string& key) {
        if (!std::getline(in, line)) fail("truncated header, expected '" + key + "'");
        std::istringstream ls(line);
        std::string got, rest;
        ls >> got;
        if (got != key) fail("expected '" + key + "', got '" + got + "'");
        std::getline(ls, rest);
        return rest;
    };
    Snapshot s;
    s.inst.n = std::stoi(field("jobs"));
    s.inst.m = std::stoi(field("machines"));
    s.incumbent = std::stoi(field("incumbent"));
    s.seed = (uint32_t)std::stoul(field("seed"));
    std::istringstream cut(field("cutoff"));
    std::string kind;
    cut >> kind;
    if (kind == "nodes") {
        s.by_nodes = true;
        cut >> s.nodes_cut;
    } else if (kind == "seconds") {
        s.by_nodes = false;
        cut >> s.seconds_cut;
    } else {
        fail("unknown cutoff kind '" + kind + "'");
    }
    if (!std::getline(in, line) || line != "times") fail("expected 'times' section");
    s.inst.p.assign((size_t)s.inst.n * s.inst.m, 0);
    for (int j = 0; j < s.inst.n; ++j) {
        if (!std::getline(in, line)) fail("truncated time matrix");
        std::istringstream ls(line);
        for (int k = 0; k < s.inst.m; ++k)
            if (!(ls >> s.inst.p[(size_t)j * s.inst.m + k])) fail("short time matrix row " + std::to_string(j));
    }
    const size_t count = std::stoul(field("nodes"));
    for (size_t i = 0; i < count; ++i) {
        if (!std::getline(in, line)) fail("truncated node list");
        std::istringstream ls(line);
        std::vector<int> pr;
        std::vector<char> seen(s.inst.n, 0);
        for (int job; ls >> job;) {
            if (job < 0 || job >= s.inst.n) fail("job index out of range in node " + std::to_string(i));
            if (seen[job]) fail("repeated job in node " + std::to_string(i));
            seen[job] = 1;
            pr.push_back(job);
        }
        if (pr.empty()) fail("empty prefix in node " + std::to_string(i));
        s.nodes.push_back(std::move(pr));
    }
    return s;
}

int cmd_workload(const Args& a) {
    require(a, "instance");
    require(a, "ub");
    require(a, "out");
    if (a.has("nodes") && a.has("seconds")) throw std::runtime_error("--seconds excludes --nodes");
    const Instance inst = load_instance(a.get("instance"), a.get("format", "auto"));
    const bool by_time = a.has("seconds");
    const Snapshot s = generate_workload(inst, (int)a.num("ub", 0), !by_time, a.num("nodes", 0),
                                         a.real("seconds", -1.0), (uint32_t)a.num("seed", 0));
    write_output(a.get("out"), save_workload(s));
    std::cerr << "captured " << s.nodes.size() << " pending nodes\n";
    return 0;
}

struct Resolution {
    std::optional<int> best;
    int64_t nodes_bounded = 0;
    double seconds = 0.0;
    int64_t batch_used = 0;
};

// resolve_workload (bench.hpp:63-114) on the device explorer: one untimed warm-up bound
// of a prefix of L, then L pushed in order, rounds until the tree is empty.
Resolution resolve(const Snapshot& s, int64_t batch, bool autotune, const TunerOpts& to, int device) {
    const Instance& inst = s.inst;
    Device dev(inst, device);
    const int n = inst.n;
    std::vector<uint8_t> pre((size_t)std::max<size_t>(s.nodes.size(), 1) * n, 0);
    std::vector<int32_t> dep(std::max<size_t>(s.nodes.size(), 1), 0);
    for (size_t i = 0; i < s.nodes.size(); ++i) {
        for (size_t d = 0; d < s.nodes[i].size(); ++d) pre[i * n + d] = (uint8_t)s.nodes[i][d];
        dep[i] = (int32_t)s.nodes[i].size();
    }
    const fbb_descriptor_t d = make_descriptor(dev, to);
    std::optional<Tuner> tuner;
    if (autotune) tuner.emplace(d, to);
    if (batch <= 0) batch = (int64_t)d.grain * d.base_units;
    {  // warm-up: a bounding round over a prefix of L (bench.hpp:75-80)
        const int64_t warm = std::min<int64_t>((int64_t)s.nodes.size(), tuner ? fbb_tuner_target(tuner->t) : batch);
        dev.check(fbb_explorer_reset(dev.ctx, pre.data(), dep.data(), warm, s.incumbent, 1));
        int64_t done = 0;
        if (warm > 0) dev.check(fbb_explorer_run(dev.ctx, &batch, 1, 1, 0, nullptr, &done));
    }
    const auto t0 = Clock::now();
    dev.check(fbb_explorer_reset(dev.ctx, pre.data(), dep.data(), (int64_t)s.nodes.size(), s.incumbent, 1));
    drive(dev, tuner, batch);
    Resolution r;
    r.seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    int32_t inc = 0, found = 0;
    int64_t pending = 0, tot[4];
    dev.check(fbb_explorer_state(dev.ctx, &inc, &found, nullptr, &pending, tot));
    if (found) r.best = inc;
    r.nodes_bounded = tot[1];
    r.batch_used = tuner ? fbb_tuner_best_batch(tuner->t) : batch;
    if (tuner && r.batch_used == 0) r.batch_used = fbb_tuner_target(tuner->t);
    return r;
}

std::string fmt2(double v) {
    std::ostringstream o;
    o << std::fixed << std::setprecision(2) << v;
    return o.str();
}

int cmd_bench(const Args& a) {
    require(a, "workload");
    if (a.has("batch") && a.has("autotune")) throw std::runtime_error("--autotune excludes --batch");
    const std::string format = a.get("format", "table");
    if (format != "table" && format != "csv" && format != "json")
        throw std::runtime_error("--format: expected table|csv|json");
    const Snapshot s = load_workload(a.get("workload"));
    const TunerOpts to = tuner_opts(a);
    const int backends = (int)a.num("backends", 1);
    if (backends < 1) throw std::runtime_error("backend count must be positive");
    // run_experiment (bench.hpp:116-145): the strictly sequential resolution (batch 1)
    // against the configured one; any disagreement is a correctness failure (exit 2)
    TunerOpts seq_to = to;
    seq_to.trace = false;
    const Resolution seq = resolve(s, 1, false, seq_to, 0);
    const Resolution par = resolve(s, a.has("batch") ? a.num("batch", 0) : 0, a.has("autotune"), to, 0);
    if (par.best != seq.best) {
        std::cerr << "error: optimum mismatch between sequential and parallel resolution\n";
        return 2;
    }
    if (par.nodes_bounded != seq.nodes_bounded) {
        std::cerr << "error: bounded-node count mismatch between resolutions\n";
        return 2;
    }
    const double speedup = seq.seconds / std::max(par.seconds, 1e-12);
    const std::string label = std::to_string(s.inst.n) + "x" + std::to_string(s.inst.m);
    if (format == "csv") {  // emit_report (bench.hpp:150-223)
        std::cout << "instance,batch,backends,t_seq,t_par,speedup,nodes_bounded\n"
                  << label << ',' << par.batch_used << ',' << backends << ',' << seq.seconds << ','
                  << par.seconds << ',' << fmt2(speedup) << ',' << par.nodes_bounded << '\n';
    } else if (format == "json") {
        std::cout << "[{\"instance\":\"" << label << "\",\"batch\":" << par.batch_used
                  << ",\"backends\":" << backends << ",\"t_seq\":" << seq.seconds << ",\"t_par\":" << par.seconds
                  << ",\"speedup\":" << fmt2(speedup) << ",\"nodes_bounded\":" << par.nodes_bounded << "}]\n";
    } else {
        std::cout << "(No. of jobs x No. of machines) | " << par.batch_used << '\n'
                  << s.inst.n << " x " << s.inst.m << " (k=" << backends << ") | " << fmt2(speedup) << "*\n";
    }
    return 0;
}

void usage() {
    std::cerr << "Exact branch-and-bound solver for the permutation flow shop (B200)\n"
                 "usage: flowbb-b200 <gen-instance|solve|workload|bench> [options]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 1;
    }
    const std::string cmd = argv[1];
    const std::set<std::string> solver_flags = {"autotune", "trace-tuner"};
    const std::set<std::string> solver_vals = {"backends", "batch", "window", "probes", "grain", "max-batch"};
    try {
        if (cmd == "gen-instance") {
            return cmd_gen(parse_args(argc, argv, 2, {}, {"jobs", "machines", "seed", "out"}));
        }
        if (cmd == "print-instance") {  // parse (auto|simple|taillard) and re-emit as simple
            const Args a = parse_args(argc, argv, 2, {}, {"instance", "format", "out"});
            require(a, "instance");
            write_output(a.get("out"), to_simple_format(load_instance(a.get("instance"), a.get("format", "auto"))));
            return 0;
        }
        if (cmd == "solve") {
            std::set<std::string> f = solver_flags, v = solver_vals;
            f.insert("json");
            v.insert({"instance", "format", "ub", "seed", "device"});
            return cmd_solve(parse_args(argc, argv, 2, f, v));
        }
        if (cmd == "workload") {
            return cmd_workload(
                parse_args(argc, argv, 2, {}, {"instance", "format", "ub", "nodes", "seconds", "seed", "out"}));
        }
        if (cmd == "bench") {
            std::set<std::string> v = solver_vals;
            v.insert({"workload", "format"});
            return cmd_bench(parse_args(argc, argv, 2, solver_flags, v));
        }
        if (cmd == "--help" || cmd == "-h") {
            usage();
            return 0;
        }
        usage();
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
