/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the QSU/QR/EVC hot path.
 *
 * A plain-C restatement of the reference dist-sim numeric loops
 * (/root/reference/proj/src/dist_sim.cpp), used by tests/ and bench.py's
 * cpu_baseline leg as the checker.  The product never links or calls it.
 *
 * Layout convention (same as the reference's DistributedState::sub):
 * `sub` holds p sub-vectors of 2^nl complex amplitudes, PE-major,
 * interleaved (re, im) doubles: amplitude (pe, off) is
 * sub[2*((pe << nl) + off) + {0,1}].
 *
 * Parity pin: tests/test_oracle.py checks every function below against the
 * compiled reference (oracle/_ref) and the committed golden vectors in
 * tests/golden/.
 */
#ifndef QRT_ORACLE_H
#define QRT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* apply_gate_narrow (dist_sim.cpp:163-201): pos[j] = position of targets[j]
 * (matrix bit j <-> targets[j]); u is the row-major 2^k x 2^k payload. */
void orc_apply_gate(double* sub, int p, int nl, int k, const int* pos, const double* u);

/* perform_qr (dist_sim.cpp:203-240): dest[p] = after.pos_of[before.qubit_at[p]].
 * scratch has the same size as sub.  Returns the relocated count. */
uint64_t orc_perform_qr(double* sub, double* scratch, int p, int nl, int n, const int* dest);

/* mask_term (dist_sim.cpp:60-81).  Returns 0, or -1 for a global X/Y letter
 * (NotDiagonalizable). */
typedef struct {
    uint64_t x, y, z, global_z;
    int y_count;
} orc_masked_term;
int orc_mask_term(const char* letters, int n, const int* pos_of, int nl, orc_masked_term* out);

/* local_pauli_expectation (dist_sim.cpp:84-93) on one sub-vector of len amps. */
void orc_local_pauli(const double* v, uint64_t len, const orc_masked_term* m, double* out2);

/* The per-tile accumulation of expectation() (dist_sim.cpp:289-295):
 * partial[pe] += sum_i coeff_i * pe_sign(pe, gz_i) * local_pauli(sub[pe], m_i). */
void orc_expectation_tile(const double* sub, int p, int nl, int n_terms, const orc_masked_term* m,
                          const double* coeffs, double* partial);

/* flatten (dist_sim.cpp:142-161): qubit_at[position] -> canonical order. */
void orc_flatten(const double* sub, int p, int nl, int n, const int* qubit_at, double* out);

#ifdef __cplusplus
}
#endif
#endif
