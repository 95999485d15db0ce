/* Host-side native library of the B200 PBDR training path (libsplat_host.so).
 *
 * C ABI (plain pointers and sizes), no CUDA: the offline and online
 * scheduling algorithms of the reference that run on the host between GPU
 * steps, re-implemented in C++ so they scale to the BASELINE configs.
 *
 * Status codes follow include/splat_b200.h (0 OK, 1 ParameterError). */
#ifndef SPLAT_HOST_H
#define SPLAT_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_HOST_OK 0
#define BS_HOST_ERR_PARAMETER 1

/* One run of the multilevel k-way partitioner -- replaces Multilevel.run of
 * /root/reference/pkg/src/splatsched/partition.py:104-434 (called by
 * partition_graph, partition.py:398-434, once per seed run).  Graph: n
 * vertices with balance weights, n_edges undirected edges (eu[e], ev[e],
 * ew[e]); parts >= 2; eps = balance slack.  pcg_state: numpy PCG64 state of
 * np.random.default_rng(SeedSequence([seed, run])) as
 * {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}.  Output:
 * labels int64[n], identical to the reference's for integer weights. */
int32_t bs_partition_multilevel(int64_t n, const double* balance, int64_t n_edges, const int64_t* eu,
                                const int64_t* ev, const double* ew, int32_t parts, double eps,
                                const uint64_t* pcg_state, int64_t* labels);

/* Steepest-ascent pairwise-swap local search of the online image placement
 * -- replaces local_search of /root/reference/pkg/src/splatsched/placement.py:182-281
 * (called by place / hierarchical_place, placement.py:301-361).  A: int64
 * [B][N] access matrix (row-major), W: int64[B] initial assignment, updated
 * in place; coefficients beta/gamma/delta and p (>= 1, or inf) of
 * CostCoefficients; max_sweeps; wall_time in seconds (< 0: none).
 * simd_pow: the address of numpy's float64 SIMD power kernel on this CPU
 * (numpy's exported __svml_pow8), or NULL for libm pow -- the elementwise
 * powers then match np.power bit for bit, so the swap sequence and the
 * relaxed-value history are the numpy restatement's.  history: double
 * [max_sweeps + 1], *n_history = entries written (relaxed_history). */
int32_t bs_local_search(int64_t B, int32_t N, const int64_t* A, int64_t* W, double beta, double gamma,
                        double delta, double p, int32_t max_sweeps, double wall_time, const void* simd_pow,
                        int32_t n_threads, double* history, int64_t* n_history);

/* out[i] = x[i] ** y with the power kernel bs_local_search uses (simd_pow as
 * above, NULL = libm); the caller checks it against np.power. */
int32_t bs_array_pow(const double* x, double y, double* out, int64_t n, const void* simd_pow);

#ifdef __cplusplus
}
#endif

#endif /* SPLAT_HOST_H */
