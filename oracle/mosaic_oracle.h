/* mosaic_oracle.h — CPU restatement of the reference planner hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the CHECKER, never by the product path.
 *
 * Every function restates the reference algorithm operation for operation (same fp64
 * operation order, compiled with -ffp-contract=off) and cites the file:line it
 * follows under /root/reference/proj/include/mosaic/.  Parity of this restatement is
 * pinned against golden outputs of the real reference (tests/golden, generated from
 * oracle/_ref by tests/golden/make_golden.py) in tests/test_oracle_restatement.py.
 */
#ifndef MOSAIC_ORACLE_H
#define MOSAIC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mo_problem mo_problem;

/* spec: "cfg1".."cfg5" | "random:SEED:N:G" | "preset:NAME:COUNT:G"; levels 0 = default.
 * Optional model overrides (NaN / negative = keep): e1,e2,e3, include_self (0/1),
 * additive (0/1), memory capacity. */
mo_problem* mo_synth(const char* spec, int levels);
void mo_set_model(mo_problem* p, double e1, double e2, double e3, int include_self,
                  int additive, double memory_capacity);
void mo_set_solve_flags(mo_problem* p, int enable_prune, int enable_cache);
void mo_free(mo_problem* p);
int mo_num_modules(const mo_problem* p);

/* candidate_options rows of module m; returns the count (arrays may be NULL to query). */
int mo_options(mo_problem* p, int m, int* d, int* u, double* base, double* bw, double* fp);

/* Stage result: status 0 ok, 1 infeasible (nullopt), 2 module without option.
 * ent: per entry (module, d, units, n_gpus), gpus flattened in entry order. */
typedef struct {
    int status;
    double stage_time;
    int n_entries;
    int ent[64 * 4];
    int gpus[64 * 1024];
    long long probes;
} mo_stage;

void mo_stage_eval(mo_problem* p, uint64_t mask, mo_stage* out);  /* stage_eval */
void mo_exact(mo_problem* p, uint64_t mask, mo_stage* out);       /* ExactStageSolver */
void mo_feasible(mo_problem* p, uint64_t mask, double tau, mo_stage* out);

/* stage_time of one allocation given as mo_stage-style entries */
double mo_stage_time(mo_problem* p, int n_entries, const int* ent, const int* gpus);

typedef struct {
    int status; /* 0 ok, 1 infeasible, 2 module without option, 4 too large */
    int n_stages;
    uint64_t masks[64];
    double times[64];
    double iteration_time;
    long long stage_eval_calls, feasibility_calls, partitions;
} mo_plan;

void mo_solve(mo_problem* p, mo_plan* out);        /* GAHC, solver.hpp:157-289 */
void mo_brute_force(mo_problem* p, mo_plan* out);  /* oracle.hpp:206-255 */
/* allocation of stage s of the last plan */
void mo_plan_stage(mo_problem* p, int s, mo_stage* out);

/* n draws of std::normal_distribution<double>(0, 1) over std::mt19937_64(seed), libstdc++
 * algorithm (Marsaglia polar over generate_canonical<double, 53>) as simulate() uses them
 * (simulator.hpp:75-76, 89-91); the device replay kernel (sim.cu) restates the same. */
void mo_normals(uint64_t seed, int n, double* out);

#ifdef __cplusplus
}
#endif
#endif
