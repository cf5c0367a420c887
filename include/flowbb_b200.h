/*
 * flowbb_b200.h -- C-ABI of the B200-native parallel-bounding hot path.
 *
 * This is the drop-in boundary for the reference flowbb (arXiv 1206.4973
 * reference implementation, proj/include/flowbb/).  Plain pointers and sizes
 * only; no C++ or torch types cross it.  The C++ wrapper that makes it a
 * reference `Backend` (duck-typed concept used by evaluate_multi<Backend>,
 * backend.hpp:105-138) is include/flowbb_b200/gpu_backend.hpp; the cgo / JNI /
 * ctypes bindings a maintainer would add are in INTEGRATION.md.
 *
 * Node batches are structure-of-arrays, position-aligned, caller-owned:
 *   masks   count x W uint64   (W = (n+63)/64), bit j set <=> job j scheduled
 *                              (replaces Node::scheduled, node.hpp:12-24,31)
 *   heads   count x m int32    per-machine completion times of the prefix
 *                              (Node::heads, node.hpp:32; instance.hpp:76-89)
 *   depth   count int32        prefix length (Node::depth(), node.hpp:35)
 *   prefix  count x n uint8    scheduled jobs in order (Node::prefix,
 *                              node.hpp:30); only the first depth[i] bytes are
 *                              read; required only by the explorer entry points
 *
 * Errors: every entry point returns FBB_OK (0) or a negative status; the
 * message and the failing device are available from fbb_last_error.  This is
 * the C form of BackendError{backend} (backend.hpp:19-25): the C++ wrapper
 * rethrows it as flowbb::BackendError(device, message).  There is no CPU
 * fallback: without a usable sm_100 device fbb_create fails.
 *
 * Threading: one context per device; calls on different contexts may run
 * concurrently from different host threads (the reference calls
 * CpuBackend::evaluate concurrently on disjoint slices, backend.hpp:116-122).
 * Calls on one context are serialised by the caller, as the reference's
 * control thread does (search.hpp:124-174).
 */
#ifndef FLOWBB_B200_H
#define FLOWBB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBB_OK 0
#define FBB_E_ARG -1      /* invalid argument (std::invalid_argument in the reference) */
#define FBB_E_CUDA -2     /* CUDA runtime / launch failure on the context's device */
#define FBB_E_RANGE -3    /* instance outside the packed device-table range */
#define FBB_E_NOMEM -4    /* device or pinned allocation failed */
#define FBB_E_STATE -5    /* call not valid in the context's current state */

typedef struct fbb_ctx fbb_ctx;

/* Capacity description; mirrors BackendDescriptor (backend.hpp:27-33).
 * grain      = children per K2 tile (the batch-size multiple),
 * base_units = SMs x resident tiles per SM (cudaOccupancy...),
 * max_batch  = largest admissible pool (bounded by HBM, not by threads). */
typedef struct {
    int32_t grain;
    int32_t base_units;
    int64_t max_batch;
} fbb_descriptor_t;

/* Per-round counters of the explorer entry points (search.hpp:21-26,75-79). */
typedef struct {
    int64_t target;    /* pool target given to the selection (fill_buffer) */
    int64_t branched;  /* parents expanded */
    int64_t bounded;   /* children bounded (= pool size) */
    int64_t inserted;  /* internal children pushed to pending */
    int64_t pruned;    /* internal children eliminated (lb >= incumbent) */
    int64_t leaves;    /* complete children */
    int32_t incumbent; /* incumbent after the round (frozen: best leaf < UB, else UB) */
    float k2_ms;       /* device time of the internal-children K2 launch (first CTA start ..
                          last CTA end on the device clock; CUDA events with FBB_PDL=0) */
    int64_t pending;   /* pending nodes after the round */
    float round_ms;    /* device time of the round, pool upload .. summary download */
    int32_t launches;  /* kernels this library launched for the round */
    float host_ms;     /* wall time of the round inside the library (steady clock) */
    float sync_ms;     /* part of host_ms spent waiting for the device */
    int64_t h2d_bytes; /* host -> device bytes of the round (host-resident explorer) */
    int64_t d2h_bytes; /* device -> host bytes of the round (host-resident explorer) */
    float place_ms;    /* place_kernel + summary time (CUDA events, FBB_PDL=0 only; else -1); device-planned
                          rounds: plan start .. first K2 CTA start (device clock) */
    int32_t reserved;
} fbb_round_t;

/* ---- context ----------------------------------------------------------------------------
 * Replaces Instance(n, m, times) (instance.hpp:30-46) + CpuBackend(descriptor)
 * (backend.hpp:50-59): uploads p (job-major, n x m int32, p[j*m+k]) and builds
 * the device tables (tails, per-machine-pair Johnson orders).  Returns NULL on
 * failure; fbb_last_error(NULL, ...) then reports why. */
fbb_ctx* fbb_create(int device, const int32_t* p_jobmajor, int n, int m);
void fbb_destroy(fbb_ctx* ctx);

/* Last error of ctx (or of the last failed fbb_create when ctx is NULL).
 * Copies up to cap-1 bytes of the message; returns the status code. */
int fbb_last_error(const fbb_ctx* ctx, int* device, char* msg, size_t cap);

/* BackendDescriptor of this device (backend.hpp:29-33, 61). */
int fbb_descriptor(fbb_ctx* ctx, fbb_descriptor_t* out);

/* ---- K1: bound-only (drop-in for CpuBackend::evaluate, backend.hpp:63-65,
 * i.e. evaluate_batch, bound.hpp:104-109).  Host buffers; lb_out[i] is
 * lower_bound(inst, node_i) (bound.hpp:94-101), position-aligned. */
int fbb_bound(fbb_ctx* ctx, const uint64_t* masks, const int32_t* heads, const int32_t* depth,
              int64_t count, int32_t* lb_out);

/* Same, device pointers, on `stream` (cudaStream_t, NULL = the context's own
 * stream); asynchronous. */
int fbb_bound_device(fbb_ctx* ctx, const uint64_t* d_masks, const int32_t* d_heads,
                     const int32_t* d_depth, int64_t count, int32_t* d_lb_out, void* stream);

/* Synthetic node pool on the device (bounding-stress workload): node i is the
 * reference test helper's random_node (tests/helpers.hpp:47-55) with a
 * counter-based generator -- depth uniform in [min_depth, max_depth], the first
 * `depth` picks of a Fisher-Yates shuffle (splitmix64 of seed ^ i*0xD1B54A32D192ED03),
 * heads folded with child_heads.  Device pointers (d_prefix may be NULL);
 * asynchronous on `stream` (NULL = the context's stream). */
int fbb_synth_pool(fbb_ctx* ctx, uint64_t seed, int64_t count, int32_t min_depth, int32_t max_depth,
                   uint64_t* d_masks, int32_t* d_heads, int32_t* d_depth, uint8_t* d_prefix,
                   void* stream);

/* ---- K2: fused expand + bound + prune + compact of one pool.
 * Replaces, for the given parents (in pop order), branch (search.hpp:40-59)
 * + evaluate + integrate (search.hpp:84-107) / the frozen prune
 * (bench.hpp:96-106):
 *   children of each parent in ascending job order, depth-(n-1) children
 *   auto-completed; every child bounded; leaves reduce to (value, first
 *   position) of the batch minimum; internal children survive iff
 *   lb < min(ub, batch leaf minimum) (solve, frozen == 0) or lb < ub
 *   (frozen != 0).  Survivors are returned stably compacted (batch order) in
 *   the same SoA layout (capacity: sum of children).  Host buffers.
 * leaf_best / leaf_pos: minimum leaf value < ub (INT32_MAX if none) and the
 * batch position of its first occurrence; when leaf_schedule != NULL and a
 * leaf improved, it receives the leaf's full permutation (n int32). */
int fbb_expand_bound_prune(fbb_ctx* ctx, const uint64_t* masks, const int32_t* heads,
                           const int32_t* depth, const uint8_t* prefix, int64_t nparents,
                           int32_t ub, int frozen, uint64_t* out_masks, int32_t* out_heads,
                           int32_t* out_depth, uint8_t* out_prefix, int32_t* out_lb,
                           int64_t* out_count, int32_t* leaf_best, int64_t* leaf_pos,
                           int32_t* leaf_schedule, fbb_round_t* counts);

/* ---- device-resident explorer (pending tree in HBM) -------------------
 * The pending tree (pending.hpp:13-56: per-depth buckets, deepest first, LIFO)
 * lives in device memory; every round is selection (fill_buffer,
 * search.hpp:64-73) + K2 + in-order push, with no host traffic but a few
 * counters.  Semantics are those of resolve_workload (bench.hpp:63-114, frozen
 * incumbent) or solve (search.hpp:124-174). */

/* Where the pending tree lives: device memory (0, default) or pinned host
 * memory (1: the paper's Type-1 split -- the host owns the tree; each round K2
 * reads its parents from the device-mapped host buckets over the host link and
 * the surviving children are written back into them).  Clears the pending
 * tree.  Same explorer semantics either way; the per-round h2d/d2h byte counts
 * are reported in fbb_round_t. */
int fbb_explorer_set_residency(fbb_ctx* ctx, int pending_on_host);

/* Reset the pending tree to the given nodes (pushed in order, like
 * bench.hpp:84) with incumbent `ub` (frozen or not). */
int fbb_explorer_reset(fbb_ctx* ctx, const uint8_t* prefix, const int32_t* depth, int64_t count,
                       int32_t ub, int frozen);

/* solve()'s first round (search.hpp:150-153): bound the root, integrate it.
 * Initial UB: ub >= 0, or the identity-permutation makespan when ub < 0
 * (search.hpp:131-137). */
int fbb_explorer_start_solve(fbb_ctx* ctx, int32_t ub, fbb_round_t* round0);

/* Runs up to max_rounds rounds with pool target targets[r] (the last value
 * repeats), stopping early when pending is empty or when the cumulative
 * bounded count reaches `budget` (> 0).  Fills rounds[0..*done). */
int fbb_explorer_run(fbb_ctx* ctx, const int64_t* targets, int ntargets, int64_t max_rounds,
                     int64_t budget, fbb_round_t* rounds, int64_t* done);

/* Incumbent value, schedule (n int32) when found, pending size, totals
 * (branched, bounded, pruned, leaves). */
int fbb_explorer_state(fbb_ctx* ctx, int32_t* incumbent, int32_t* found, int32_t* schedule,
                       int64_t* pending, int64_t* totals4);

/* Host-side copy of the pending tree, shallowest bucket first, insertion
 * order within a bucket (PendingTree::drain order, pending.hpp:41-50),
 * without modifying it.  prefix: cap x n bytes; returns the count in *count
 * (FBB_E_ARG with *count = size if cap is too small). */
int fbb_explorer_pending(fbb_ctx* ctx, uint8_t* prefix, int32_t* depth, int64_t cap,
                         int64_t* count);

/* ---- multi-device exploration (one context per GPU) ---------------------
 * Lower the pruning incumbent to `ub` when it improves it: the value of a leaf
 * found on another device, delivered by the caller's min-allreduce (solve mode
 * only; FBB_E_STATE when frozen). */
int fbb_explorer_set_incumbent(fbb_ctx* ctx, int32_t ub);

/* This context's own best leaf: returns 1 and its value (and, in solve mode,
 * its schedule, n int32) when one was found, else 0 with *value = INT32_MAX. */
int fbb_explorer_best(fbb_ctx* ctx, int32_t* value, int32_t* schedule);

/* Pool rebalancing: remove up to k pending nodes from the tops of the
 * shallowest non-empty buckets (the roots of the largest unexplored subtrees)
 * and return them (prefix rows of n bytes, depths); *taken = how many. */
int fbb_explorer_take(fbb_ctx* ctx, int64_t k, uint8_t* prefix, int32_t* depth, int64_t* taken);

/* Push nodes (given as prefixes) onto the pending tree, in order, without
 * resetting it (the receiving side of fbb_explorer_take). */
int fbb_explorer_push(fbb_ctx* ctx, const uint8_t* prefix, const int32_t* depth, int64_t count);

/* ---- device group: one process, G devices, the exchange inside the library ------------
 * The single-process form of the multi-GPU explorer (SURVEY 8(b) "fbb_group_create(devs[],
 * G)"; the paper's Type-1 split of one host over the GPUs of a box, with
 * the reference's BackendSet(k) over k devices, backend.hpp:142-158).  Each member is an
 * ordinary context (device ids may repeat) driven by its own host thread; every step runs
 * `rounds_per_step` explorer rounds on all members concurrently, then the library
 * exchanges, on the calling thread:
 *   - solve mode: the minimum incumbent over members becomes every member's pruning
 *     bound (the UB min-allreduce; fbb_explorer_set_incumbent),
 *   - every `balance_every` steps: a starving member (pending < target / n) receives
 *     half the difference (<= 65536 nodes) from the richest member, shallowest pending
 *     nodes first (fbb_explorer_take -> fbb_explorer_push), the same deterministic plan
 *     as the multi-process driver (paper_1206_4973_b200/parallel.py plan_transfers).
 * Frozen exploration is partition-invariant (bench.hpp:60-62): the summed counts to
 * exhaustion equal one context's. */
typedef struct fbb_group fbb_group;

typedef struct {
    int64_t steps;         /* exchange steps run by this call */
    int64_t rounds;        /* explorer rounds summed over members */
    int64_t branched, bounded, pruned, leaves;  /* totals over members since the reset */
    int64_t pending;       /* pending nodes over members after the call */
    int64_t transfers;     /* nodes moved between members by this call */
    int32_t incumbent;     /* group incumbent (frozen: best leaf < UB, else UB) */
    int32_t found;         /* a leaf below the initial UB was found */
    double seconds;        /* wall time of the call */
    double device_ms_max;  /* max over members of their summed round device time */
    double exchange_ms;    /* wall time spent in the exchanges (calling thread) */
} fbb_group_stats_t;

/* Creates one context per entry of devices[0..G) over the same instance (p job-major,
 * n x m).  NULL on failure (fbb_last_error(NULL, ...) says why). */
fbb_group* fbb_group_create(const int* devices, int G, const int32_t* p_jobmajor, int n, int m);
void fbb_group_destroy(fbb_group* g);
int fbb_group_size(const fbb_group* g);
/* Member i's context (owned by the group): its fbb_explorer_* counters stay per member. */
fbb_ctx* fbb_group_context(fbb_group* g, int i);
/* Last error of the group: the failing member's status, index and message. */
int fbb_group_last_error(const fbb_group* g, int* member, char* msg, size_t cap);
/* Resets every member: the nodes are split into G contiguous slices (split_slices,
 * backend.hpp:73-84), slice i pushed in order onto member i; incumbent `ub`. */
int fbb_group_reset(fbb_group* g, const uint8_t* prefix, const int32_t* depth, int64_t count,
                    int32_t ub, int frozen);
/* solve()'s root round (search.hpp:131-153) on member 0 (ub < 0: identity makespan);
 * the other members start empty with the same incumbent and are fed by rebalancing. */
int fbb_group_start_solve(fbb_group* g, int32_t ub);
/* Runs exchange steps with pool target `target` per member until every member's
 * pending tree is empty, max_steps steps ran, or the summed bounded count reached
 * `budget` (> 0).  stats may be NULL. */
int fbb_group_run(fbb_group* g, int64_t target, int64_t max_steps, int rounds_per_step,
                  int balance_every, int64_t budget, fbb_group_stats_t* stats);
/* The group's (and paper_1206_4973_b200/parallel.py's) deterministic rebalancing plan over
 * G pending sizes: receivers in ascending (pending, index) order below `low` take half the
 * difference (<= cap) from the richest member above 2*low that has not donated yet.
 * Writes up to G (donor, receiver, count) triples to plan (3*G int64) and their number to
 * *count.  Host-only: a multi-process C++ driver computes the same plan on every rank. */
int fbb_plan_transfers(const int64_t* pending, int G, int64_t low, int64_t cap, int64_t* plan,
                       int* count);

/* Group best leaf: min over members of (value, member index); returns 1 and its value
 * (and, in solve mode, its schedule) when found, else 0 with *value = INT32_MAX. */
int fbb_group_best(fbb_group* g, int32_t* value, int32_t* schedule);

/* ---- adaptive pool-size tuner (autotune.hpp:35-156), re-derived descriptor ----------- */
typedef struct fbb_tuner fbb_tuner;
fbb_tuner* fbb_tuner_create(int32_t grain, int32_t base_units, int64_t max_batch, int window,
                            int probes_per_side);
void fbb_tuner_destroy(fbb_tuner* t);
int64_t fbb_tuner_target(const fbb_tuner* t);
/* returns FBB_E_ARG on non-positive elapsed (std::invalid_argument) */
int fbb_tuner_observe(fbb_tuner* t, int64_t nodes_bounded, double elapsed_seconds);
int fbb_tuner_phase(const fbb_tuner* t); /* 0 doubling, 1 refining, 2 fixed */
int64_t fbb_tuner_best_batch(const fbb_tuner* t);
double fbb_tuner_best_throughput(const fbb_tuner* t);
/* Tuner::set_trace (autotune.hpp:112-113): called once per closed window with the
 * window index, the measured batch, its throughput and the decision text
 * ("double to B" | "refine at B" | "fix at B"); fn == NULL disables it. */
typedef void (*fbb_tuner_trace_fn)(void* user, int window, int64_t batch, double throughput,
                                   const char* decision);
int fbb_tuner_set_trace(fbb_tuner* t, fbb_tuner_trace_fn fn, void* user);

/* The kernel variants this context launches, as one line of text, e.g.
 * "K1=k1v2_kernel<8,4> K2=k2_v3_kernel<4,20> cmax=224 ppc_cap=16 blocks=444"
 * (measurement labels; copies up to cap-1 bytes). */
int fbb_kernels(fbb_ctx* ctx, char* buf, size_t cap);

/* Library build identification (sm arch, git-less version string). */
const char* fbb_version(void);

#ifdef __cplusplus
}
#endif

#endif
