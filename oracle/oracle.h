/*
 * oracle.h -- plain fp64 CPU oracle of FastDOG's Alg. "Parallel Deferred
 * Min-Marginal Averaging" (arXiv 2111.10270).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the product path
 * (include/fastdog.h, paper_2111_10270_b200/csrc/); it declares its own
 * problem struct on purpose.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = SPEC.md.
 * Readings of ambiguous passages are the ones listed in DESIGN.md §3
 * (A1..A16, same labels as SURVEY.md §8(c)).
 *
 * Error codes: 0 ok, 1 invalid argument, 2 infeasible constraint,
 *              3 out of memory, 6 bad state, 7 rounding without consensus.
 */
#ifndef FASTDOG_ORACLE_H
#define FASTDOG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Binary program (BP) P:555-565 given as 0-1 ILP rows (Example ILP P:567-577).
 * Row j: sum_{p in [row_ptr[j], row_ptr[j+1])} col_coef[p] * x[col_var[p]]  rel[j]  rhs[j]
 * rel: -1 "<=", 0 "==", +1 ">=".  col_var strictly ascending within a row. */
typedef struct {
  int32_t n_vars;
  const double *cost;
  int32_t n_cons;
  const int64_t *row_ptr;
  const int32_t *col_var;
  const int32_t *col_coef;
  const int8_t *rel;
  const int64_t *rhs;
} oracle_problem;

typedef struct oracle_solver oracle_solver;

/* Compile every row to a quasi-reduced ordered BDD (compiler "A": top-down
 * partial-sum states, bottom-up (s0,s1)-signature merge), initialise
 * lambda = c_i/|J_i| (A9), mbar = 0, and cost_to_terminal.
 * clamp: value substituted for an infinite min-marginal difference (A5).
 * n_threads <= 0: OpenMP default. */
int oracle_create(const oracle_problem *p, double clamp, int n_threads, oracle_solver **out);
void oracle_destroy(oracle_solver *s);

/* One pass (forward = 1: ascending hops; forward = 0: backward,
 * P:647-648), including the deferred averaging before it and the swap
 * mbar <- m after it. */
int oracle_pass(oracle_solver *s, int forward, double omega);
/* n_iter x (forward pass, backward pass). */
int oracle_iterate(oracle_solver *s, int n_iter, double omega);
/* Non-deferred variant ([lange2021efficient]): variables visited
 * one at a time in ascending (forward) / descending (backward) global order;
 * all j in J_i compute m_ij, then lambda_i^j <- lambda_i^j - omega d_ij +
 * mean_k omega d_ik.  Needs delta_bar = 0 (fresh, finalized, or after another
 * _seq pass; else 6).  Leaves delta_bar = 0; the bound is sum_j E^j. */
int oracle_pass_seq(oracle_solver *s, int forward, double omega);
int oracle_iterate_seq(oracle_solver *s, int n_iter, double omega);
/* Lifted lower bound (A7) of the last completed pass, or sum_j E^j at init /
 * after finalize. */
int oracle_lower_bound(const oracle_solver *s, double *out);
/* Raw sum_j E^j(lambda^j) + sum_free min(c_i,0) at the current lambda. */
int oracle_dual_energy(const oracle_solver *s, double *out);
/* Final correction P:650-652: lambda += delta_bar (per slot), delta_bar = 0,
 * recompute cost_to_terminal. */
int oracle_finalize(oracle_solver *s);
/* Averaged final correction (P:673 prose; A11 alternative). */
int oracle_finalize_avg(oracle_solver *s);

/* Slots in canonical order (j ascending, hop ascending). */
int oracle_num_slots(const oracle_solver *s, int64_t *out);
int oracle_get_lambda(const oracle_solver *s, double *out, int64_t len);
/* delta_bar = omega * clamp(mbar1 - mbar0) of the last pass (A10). */
int oracle_get_deferred(const oracle_solver *s, double *out, int64_t len);
/* m0, m1 recorded during the last pass (+inf where infeasible). */
int oracle_min_marginals(const oracle_solver *s, double *m0, double *m1, int64_t len);
/* Overwrite lambda (canonical order); delta_bar is kept.  Recomputes both
 * distance directions from the definition; the bound
 * becomes sum_j E^j(lambda) + sum min(delta_bar, 0) + free term (A7). */
int oracle_set_lambda(oracle_solver *s, const double *lambda, int64_t len);

/* BDD inspection (for the path-set / closed-form pins). */
int oracle_bdd_size(const oracle_solver *s, int32_t j, int32_t *k, int32_t *n_nodes);
/* vars[k], hop_start[k+1], lo[n_nodes], hi[n_nodes]; successor codes:
 * >= 0 node index within the BDD, -1 = bottom, -2 = top. */
int oracle_bdd_get(const oracle_solver *s, int32_t j, int32_t *vars, int32_t *hop_start,
                   int32_t *lo, int32_t *hi);
int oracle_total_nodes(const oracle_solver *s, int64_t *out);

/* Alg. "Perturbation Primal Rounding", reading of DESIGN.md §3:
 * signs of the min-marginals recorded in the last pass; r ~ U[-delta, delta]
 * from the counter-based generator splitmix64(seed, round, i).
 * oracle_primal_step: one classification (+ perturbation if any variable's
 * subproblems disagree); *conflicts = number of such variables; x = labeling.
 * oracle_round_primal: the full loop with `inner` Alg.-1 iterations per round;
 * returns 7 when max_rounds perturbation rounds did not reach consensus. */
int oracle_primal_step(oracle_solver *s, int32_t round, double delta, uint64_t seed, int64_t *conflicts,
                       uint8_t *x);
int oracle_round_primal(oracle_solver *s, double delta0, double alpha, int32_t inner, int32_t max_rounds,
                        uint64_t seed, double omega, uint8_t *x, int32_t *rounds);
int oracle_num_threads(const oracle_solver *s);

/* Lifted representation: switch a fresh solver (no pass yet, else
 * 6) to two costs per slot, lambda^{j,0} = 0 and lambda^{j,1} = c_i/|J_i|
 * (P:622), updated by reading A8 (P:53-56 with max(., 0)).  Afterwards
 * oracle_pass runs lifted passes, oracle_lower_bound is the plain sum of the
 * per-BDD shortest paths (+ free term), oracle_get_lambda returns lambda^1 -
 * lambda^0, oracle_finalize adds max(+-delta_bar, 0) to the two
 * sides; pass_seq, set_lambda, dual_energy, finalize_avg and the primal
 * rounding return 6. */
int oracle_set_lifted(oracle_solver *s);
int oracle_get_lifted(const oracle_solver *s, double *lam0, double *lam1, int64_t len);

#ifdef __cplusplus
}
#endif
#endif
