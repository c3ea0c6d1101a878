/*
 * TEST INFRASTRUCTURE ONLY — see qrt_oracle.h.  Each function restates one
 * loop of /root/reference/proj/src/dist_sim.cpp (line numbers cited) in
 * plain C, with the same evaluation order for the complex arithmetic so the
 * results agree bit-for-bit with the compiled reference on x86-64 (no FMA
 * contraction at the default -O2 baseline ISA).
 */
#include "qrt_oracle.h"

#include <stdlib.h>
#include <string.h>

static int popc64(uint64_t v) { return __builtin_popcountll(v); }

/* insert_zero_bits (dist_sim.cpp:43-49): spread value over the positions
 * not in sorted[0..k). */
static uint64_t spread(uint64_t value, const int* sorted, int k) {
    for (int j = 0; j < k; ++j) {
        int p = sorted[j];
        uint64_t low = value & ((1ULL << p) - 1ULL);
        value = ((value >> p) << (p + 1)) | low;
    }
    return value;
}

void orc_apply_gate(double* sub, int p, int nl, int k, const int* pos, const double* u) {
    int sorted[64];
    for (int j = 0; j < k; ++j) sorted[j] = pos[j];
    for (int a = 1; a < k; ++a) /* insertion sort: dist_sim.cpp:175-176 */
        for (int b = a; b > 0 && sorted[b - 1] > sorted[b]; --b) {
            int t = sorted[b];
            sorted[b] = sorted[b - 1];
            sorted[b - 1] = t;
        }
    const int dim = 1 << k;
    const uint64_t groups = 1ULL << (nl - k);
    double* in = (double*)malloc(sizeof(double) * 2 * (size_t)dim);
    uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)dim);
    for (int pe = 0; pe < p; ++pe) {
        double* v = sub + 2 * ((uint64_t)pe << nl);
        for (uint64_t g = 0; g < groups; ++g) { /* :185-199 */
            uint64_t base = spread(g, sorted, k);
            for (int m = 0; m < dim; ++m) {
                uint64_t i = base;
                for (int j = 0; j < k; ++j)
                    if ((m >> j) & 1) i |= 1ULL << pos[j];
                idx[m] = i;
                in[2 * m] = v[2 * i];
                in[2 * m + 1] = v[2 * i + 1];
            }
            for (int r = 0; r < dim; ++r) {
                double ar = 0.0, ai = 0.0;
                for (int c = 0; c < dim; ++c) {
                    double a = u[2 * ((size_t)r * dim + c)], b = u[2 * ((size_t)r * dim + c) + 1];
                    double x = in[2 * c], y = in[2 * c + 1];
                    double pr = a * x - b * y;
                    double pi = a * y + b * x;
                    ar += pr;
                    ai += pi;
                }
                v[2 * idx[r]] = ar;
                v[2 * idx[r] + 1] = ai;
            }
        }
    }
    free(in);
    free(idx);
}

uint64_t orc_perform_qr(double* sub, double* scratch, int p, int nl, int n, const int* dest) {
    (void)p;
    uint64_t stay = 0;
    int from[64], to[64], nm = 0;
    for (int q = 0; q < n; ++q) { /* :213-222 */
        if (dest[q] == q)
            stay |= 1ULL << q;
        else {
            from[nm] = q;
            to[nm] = dest[q];
            ++nm;
        }
    }
    uint64_t relocated = 0;
    const uint64_t total = 1ULL << n;
    for (uint64_t i = 0; i < total; ++i) { /* :228-233 */
        uint64_t j = i & stay;
        for (int t = 0; t < nm; ++t) j |= ((i >> from[t]) & 1ULL) << to[t];
        if ((j >> nl) != (i >> nl)) ++relocated;
        scratch[2 * j] = sub[2 * i];
        scratch[2 * j + 1] = sub[2 * i + 1];
    }
    memcpy(sub, scratch, sizeof(double) * 2 * total);
    return relocated;
}

int orc_mask_term(const char* letters, int n, const int* pos_of, int nl, orc_masked_term* m) {
    memset(m, 0, sizeof *m);
    for (int q = 0; q < n; ++q) {
        char c = letters[q];
        if (c == 'I') continue;
        int pos = pos_of[q];
        if (pos < nl) {
            if (c == 'X') m->x |= 1ULL << pos;
            if (c == 'Y') {
                m->y |= 1ULL << pos;
                ++m->y_count;
            }
            if (c == 'Z') m->z |= 1ULL << pos;
        } else {
            if (c != 'Z') return -1; /* NotDiagonalizable, :74-76 */
            m->global_z |= 1ULL << (pos - nl);
        }
    }
    return 0;
}

void orc_local_pauli(const double* v, uint64_t len, const orc_masked_term* m, double* out2) {
    const uint64_t xy = m->x | m->y;
    const uint64_t sign_mask = m->z | m->y;
    double ar = 0.0, ai = 0.0;
    for (uint64_t i = 0; i < len; ++i) { /* :88-91 */
        double sgn = (popc64(i & sign_mask) & 1) ? -1.0 : 1.0;
        /* (sgn * conj(v[i^xy])) * v[i] */
        double a = sgn * v[2 * (i ^ xy)], b = sgn * -v[2 * (i ^ xy) + 1];
        double c = v[2 * i], d = v[2 * i + 1];
        ar += a * c - b * d;
        ai += a * d + b * c;
    }
    /* ipow(y_count) * acc (:15-22, :92) as a full complex product, keeping
     * the signed-zero behaviour of std::complex multiplication. */
    double ir, ii;
    switch (m->y_count & 3) {
        case 0: ir = 1.0; ii = 0.0; break;
        case 1: ir = 0.0; ii = 1.0; break;
        case 2: ir = -1.0; ii = 0.0; break;
        default: ir = 0.0; ii = -1.0; break;
    }
    out2[0] = ir * ar - ii * ai;
    out2[1] = ir * ai + ii * ar;
}

void orc_expectation_tile(const double* sub, int p, int nl, int n_terms, const orc_masked_term* m,
                          const double* coeffs, double* partial) {
    for (int pe = 0; pe < p; ++pe) { /* :289-295 */
        double ar = 0.0, ai = 0.0;
        const double* v = sub + 2 * ((uint64_t)pe << nl);
        for (int t = 0; t < n_terms; ++t) {
            double sgn = (popc64((uint64_t)pe & m[t].global_z) & 1) ? -1.0 : 1.0;
            double loc[2];
            orc_local_pauli(v, 1ULL << nl, &m[t], loc);
            /* coeffs[i] * pe_sign * local : (c * s) * loc */
            double cr = coeffs[2 * t] * sgn, ci = coeffs[2 * t + 1] * sgn;
            ar += cr * loc[0] - ci * loc[1];
            ai += cr * loc[1] + ci * loc[0];
        }
        partial[2 * pe] += ar;
        partial[2 * pe + 1] += ai;
    }
}

void orc_flatten(const double* sub, int p, int nl, int n, const int* qubit_at, double* out) {
    (void)n;
    for (int pe = 0; pe < p; ++pe) /* :147-159 */
        for (uint64_t off = 0; off < (1ULL << nl); ++off) {
            uint64_t idx = ((uint64_t)pe << nl) | off;
            uint64_t b = 0, rest = idx;
            while (rest) {
                int pos = __builtin_ctzll(rest);
                b |= 1ULL << qubit_at[pos];
                rest &= rest - 1;
            }
            out[2 * b] = sub[2 * idx];
            out[2 * b + 1] = sub[2 * idx + 1];
        }
}
