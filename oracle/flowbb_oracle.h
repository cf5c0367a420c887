/*
 * flowbb_oracle.h -- CPU restatement of the reference flowbb hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product library (paper_1206_4973_b200/libflowbb_b200.so)
 * never links or calls anything here, and has no CPU fallback.
 *
 * Every function restates one reference function; the file:line it follows
 * is cited (paths relative to the reference's proj/include/flowbb/).
 * Parity of this restatement is pinned by
 *   - the reference's own known-answer tests (tests/test_*.cpp KATs, encoded
 *     in tests/test_oracle.py), and
 *   - golden vectors produced by the reference itself compiled in place
 *     (oracle/_ref, see oracle/Makefile and tests/golden/make_golden.py).
 *
 * Node representation (flat, structure-of-arrays, shared with the CUDA path):
 *   mask   : W = (n+63)/64 uint64 words per node, bit j set <=> job j scheduled
 *            (node.hpp:12-24 JobMask)
 *   heads  : m int32 per node, per-machine completion times of the prefix
 *            (instance.hpp:76-78 Heads)
 *   depth  : int32, prefix length (node.hpp:35)
 *   prefix : n int32 per node (only the first `depth` are meaningful)
 */
#ifndef FLOWBB_ORACLE_H
#define FLOWBB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* instance.hpp:238-265 -- Taillard generator, times U[1,99] machine-major.
 * Writes p job-major (p[j*m+k]).  Returns 0, or -1 on an invalid seed. */
int orc_generate_instance(int n, int m, int32_t seed, int32_t* p_out);

/* instance.hpp:38-45 -- tails[j*m+k] = sum_{u>k} p[j][u]. */
void orc_tails(int n, int m, const int32_t* p, int32_t* tails_out);

/* instance.hpp:81-89 */
void orc_child_heads(int n, int m, const int32_t* p, const int32_t* heads, int job,
                     int32_t* out);

/* instance.hpp:92-96 */
int32_t orc_makespan(int n, int m, const int32_t* p, const int32_t* perm, int len);

/* bound.hpp:27-44 -- stable Johnson order with lags + simulation. */
int32_t orc_johnson_two_machine(const int32_t* a, const int32_t* lag, const int32_t* b,
                                int count, int32_t release_a, int32_t release_b);

/* bound.hpp:61-74 */
int32_t orc_lb_one_machine(int n, int m, const int32_t* p, const uint64_t* mask,
                           const int32_t* heads);

/* bound.hpp:79-90 */
int32_t orc_lb_machine_pair(int n, int m, const int32_t* p, const uint64_t* mask,
                            const int32_t* heads, int k, int l);

/* bound.hpp:94-101 */
int32_t orc_lower_bound(int n, int m, const int32_t* p, const uint64_t* mask,
                        const int32_t* heads, int depth);

/* bound.hpp:104-109 -- position-aligned map of orc_lower_bound. */
void orc_evaluate_batch(int n, int m, const int32_t* p, int64_t count, const uint64_t* masks,
                        const int32_t* heads, const int32_t* depth, int32_t* lb_out);

/* Builds a node from a prefix by folding Node::child (node.hpp:44-52).
 * Writes mask (W words) and heads (m). */
void orc_node_from_prefix(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
                          uint64_t* mask_out, int32_t* heads_out);

/* search.hpp:40-59 -- children of one node, ascending job index, depth n-1
 * children auto-completed.  Writes up to n-depth children (prefix n ints,
 * mask W words, heads m ints, depth).  Returns the child count, -1 if the
 * node is complete (logic_error in the reference). */
int orc_branch(int n, int m, const int32_t* p, const int32_t* prefix, int depth,
               int32_t* child_prefix, uint64_t* child_mask, int32_t* child_heads,
               int32_t* child_depth);

/* Per-round trace record of the explorer restatements below. */
typedef struct {
    int64_t target;      /* pool target used by fill_buffer this round (0 for the root round) */
    int64_t branched;    /* parents popped by fill_buffer (search.hpp:69) */
    int64_t bounded;     /* batch size (search.hpp:158 / bench.hpp:95) */
    int64_t inserted;    /* internal children pushed */
    int64_t pruned;      /* internal children eliminated */
    int64_t leaves;      /* complete children */
    int32_t incumbent;   /* incumbent after the round (solve) / best-or-UB (resolve) */
    int32_t pad;
    int64_t pending;     /* pending size after integration */
} orc_round;

/* Result of a run. */
typedef struct {
    int64_t branched, bounded, pruned, leaves, rounds;
    int32_t optimum;     /* solve: incumbent value; resolve: best leaf < UB or -1 */
    int32_t found;       /* solve: schedule present; resolve: best present */
    int64_t pending;     /* pending size at exit (non-zero when a budget stopped the run) */
} orc_result;

/* search.hpp:124-174 solve(), restated call for call with
 *   - targets[r] (r = fill round index, last value repeats) replacing
 *     fixed_batch / tuner targets (search.hpp:144-147, 164),
 *   - an optional bounded-node budget (0 = none) checked after each round's
 *     integration; a budget stop leaves pending non-empty.
 * initial_ub < 0 selects the identity-permutation UB (search.hpp:131-137).
 * schedule_out (n ints) receives the incumbent schedule when found.
 * trace (max_trace entries, may be NULL) receives one record per round. */
int orc_solve(int n, int m, const int32_t* p, int32_t initial_ub, const int64_t* targets,
              int ntargets, int64_t budget, orc_result* res, int32_t* schedule_out,
              orc_round* trace, int64_t max_trace);

/* bench.hpp:63-114 resolve_workload(), frozen incumbent, restated with the
 * same targets/budget extensions.  The snapshot is nroots prefixes
 * (roots_prefix nroots x n ints, roots_depth). */
int orc_resolve(int n, int m, const int32_t* p, int32_t ub, int64_t nroots,
                const int32_t* roots_prefix, const int32_t* roots_depth, const int64_t* targets,
                int ntargets, int64_t budget, orc_result* res, orc_round* trace,
                int64_t max_trace);

#ifdef __cplusplus
}
#endif

#endif
