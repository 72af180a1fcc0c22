/*
 * oracle/sv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU state-vector simulator in complex128.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  It shares NO code, header, table or constant
 * with the CUDA path (paper_2008_00216_b200/) and the product never calls it.
 *
 * What it computes (SURVEY.md 8(c) "Definition"):
 *     psi_out = U_G ... U_2 U_1 e_{x0}
 * where U_g is gate g's 2^q x 2^q matrix on its qubits and identity elsewhere
 * ("pad each gate with an identity matrix ... and multiply", PAPER.md L230-233,
 * Sec. 3 "Baseline Simulation Algorithms"), evaluated without padding, gate by
 * gate, exactly in input order ("Fast Schroedinger
 * simulation": the 2^{n-q} disjoint sets of 2^q amplitudes sharing a set id
 * are updated in place).  No reordering, no fusion, no relabelling, no special
 * case for diagonal or permutation gates.
 *
 * Conventions (DESIGN.md readings):
 *   A1  qubit q <-> bit q of the amplitude index (LSB), as in the paper's
 *       bitmask figures.
 *   A2  for a 2-qubit gate (q0, q1) the local matrix index is 2*b(q0)+b(q1):
 *       the first-listed qubit is the MSB (CNOT matrix).
 *   Gate matrices: Appendix A of SURVEY.md; paper sources cited per gate.
 *
 * Parity pins (tests/test_oracle.py, all -m "not gpu"): gate identities,
 * a numpy Kronecker brute force for n<=8, closed forms (uniform H^n|0>, GHZ,
 * QFT of a basis state), norm preservation and the mirror test.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

/* oracle-private gate codes (the product defines its own, independently) */
enum { OG_H = 0, OG_X, OG_Y, OG_Z, OG_S, OG_T, OG_SX, OG_SY, OG_SW,
       OG_CZ, OG_CNOT, OG_SWAP, OG_CPHASE, OG_FSIM, OG_U1, OG_U2, OG_NKINDS };

typedef struct {
    int32_t kind;
    int32_t adjoint;      /* nonzero: apply the conjugate transpose */
    int32_t q0, q1;       /* q1 = -1 for 1-qubit gates                */
    double theta, phi;    /* CPHASE(phi); FSIM(theta, phi)             */
    const double *m;      /* U1: 2x2, U2: 4x4, row-major (re, im)       */
} og_gate;

int oracle_nqubits_of(int kind) {
    return (kind >= OG_CZ && kind != OG_U1) ? 2 : 1;
}

/* Writes the gate's matrix (dim x dim, row-major) into U; returns dim or -1. */
int oracle_gate_matrix(int kind, int adjoint, double theta, double phi,
                       const double *m, double *out /* 2*dim*dim */) {
    cplx U[16];
    int d = oracle_nqubits_of(kind) == 2 ? 4 : 2;
    const double r2 = M_SQRT1_2;
    for (int i = 0; i < 16; ++i) U[i] = 0;
    switch (kind) {
    case OG_H:
        U[0] = r2; U[1] = r2; U[2] = r2; U[3] = -r2; break;
    case OG_X:  /* NOT */
        U[1] = 1; U[2] = 1; break;
    case OG_Y:  /* Pauli Y */
        U[1] = -I; U[2] = I; break;
    case OG_Z:
        U[0] = 1; U[3] = -1; break;
    case OG_S:  /* P = Z^{1/2} */
        U[0] = 1; U[3] = I; break;
    case OG_T:
        U[0] = 1; U[3] = r2 + r2 * I; break;
    case OG_SX: /* X^{1/2} */
        U[0] = 0.5 + 0.5 * I; U[1] = 0.5 - 0.5 * I;
        U[2] = 0.5 - 0.5 * I; U[3] = 0.5 + 0.5 * I; break;
    case OG_SY: /* Y^{1/2}, PAPER.md L170 (reading A3) */
        U[0] = 0.5 + 0.5 * I; U[1] = 0.5 + 0.5 * I;
        U[2] = -0.5 - 0.5 * I; U[3] = 0.5 + 0.5 * I; break;
    case OG_SW: /* W^{1/2} = T X^{1/2} T^dagger (reading A4) */
        U[0] = 0.5 + 0.5 * I; U[1] = -r2 * I;
        U[2] = r2;            U[3] = 0.5 + 0.5 * I; break;
    case OG_CZ:
        U[0] = 1; U[5] = 1; U[10] = 1; U[15] = -1; break;
    case OG_CNOT: /* first qubit = control */
        U[0] = 1; U[5] = 1; U[11] = 1; U[14] = 1; break;
    case OG_SWAP: /* exchanges |01> and |10> (hushed) */
        U[0] = 1; U[6] = 1; U[9] = 1; U[15] = 1; break;
    case OG_CPHASE: /* diag(1,1,1,e^{i phi}) (reading A6) */
        U[0] = 1; U[5] = 1; U[10] = 1; U[15] = cexp(I * phi); break;
    case OG_FSIM: /* reading A5 */
        U[0] = 1;
        U[5] = cos(theta); U[6] = -I * sin(theta);
        U[9] = -I * sin(theta); U[10] = cos(theta);
        U[15] = cexp(-I * phi); break;
    case OG_U1: case OG_U2:
        for (int i = 0; i < d * d; ++i) U[i] = m[2 * i] + m[2 * i + 1] * I;
        break;
    default:
        return -1;
    }
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            cplx z = adjoint ? conj(U[c * d + r]) : U[r * d + c];
            out[2 * (r * d + c)] = creal(z);
            out[2 * (r * d + c) + 1] = cimag(z);
        }
    return d;
}

/* Apply one gate in place: PAPER.md L236-241 ("set id" iteration).  AMP is the amplitude
 * storage type: complex128 (the oracle proper), or complex64 with every gate computed in
 * complex128 from the stored amplitudes and rounded once when stored (reading A19:
 * the only way the 2^34-amplitude c4 state fits the GPU box's host memory).  One definition,
 * instantiated per storage type so each loop is compiled for its own loads and stores. */
typedef float complex cplx32;
#define DEFINE_APPLY_GATE(NAME, AMP)                                                            \
static int NAME(int n, AMP *psi, const og_gate *g) {                                            \
    int q = oracle_nqubits_of(g->kind);                                                         \
    int tq[2] = {g->q0, g->q1};                                                                 \
    double Ud[32];                                                                              \
    if (oracle_gate_matrix(g->kind, g->adjoint, g->theta, g->phi, g->m, Ud) < 0) return -1;     \
    for (int i = 0; i < q; ++i)                                                                 \
        if (tq[i] < 0 || tq[i] >= n) return -2;                                                 \
    if (q == 2 && tq[0] == tq[1]) return -3;                                                    \
    int d = 1 << q;                                                                             \
    cplx U[16];                                                                                 \
    for (int i = 0; i < d * d; ++i) U[i] = Ud[2 * i] + Ud[2 * i + 1] * I;                       \
    /* sorted target positions for zero-bit insertion */                                        \
    int sorted[2] = {tq[0], tq[1]};                                                             \
    if (q == 2 && sorted[0] > sorted[1]) { int t = sorted[0]; sorted[0] = sorted[1]; sorted[1] = t; } \
    const int64_t nsets = (int64_t)1 << (n - q);                                                \
    _Pragma("omp parallel for schedule(static)")                                                \
    for (int64_t s = 0; s < nsets; ++s) {                                                       \
        uint64_t base = (uint64_t)s;                                                            \
        for (int i = 0; i < q; ++i) {       /* insert a 0 bit at sorted[i] */                   \
            uint64_t lo = base & ((1ull << sorted[i]) - 1);                                     \
            base = ((base >> sorted[i]) << (sorted[i] + 1)) | lo;                               \
        }                                                                                       \
        uint64_t idx[4];                                                                        \
        cplx v[4];                                                                              \
        for (int l = 0; l < d; ++l) {                                                           \
            uint64_t j = base;                                                                  \
            for (int i = 0; i < q; ++i)      /* first-listed qubit = MSB of l */                \
                j |= (uint64_t)((l >> (q - 1 - i)) & 1) << tq[i];                               \
            idx[l] = j;                                                                         \
            v[l] = (cplx)psi[j];                                                                \
        }                                                                                       \
        for (int r = 0; r < d; ++r) {                                                           \
            cplx acc = 0;                                                                       \
            for (int c = 0; c < d; ++c) acc += U[r * d + c] * v[c];                             \
            psi[idx[r]] = (AMP)acc;                                                             \
        }                                                                                       \
    }                                                                                           \
    return 0;                                                                                   \
}
DEFINE_APPLY_GATE(apply_gate, cplx)
DEFINE_APPLY_GATE(apply_gate_c64store, cplx32)

/* psi <- U_G...U_1 psi.  Returns 0, or -(1+i) on a bad gate i. */
int oracle_apply(int n, double *psi_ri, const og_gate *gates, int64_t ng, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t i = 0; i < ng; ++i)
        if (apply_gate(n, (cplx *)psi_ri, &gates[i]) != 0) return (int)(-(1 + i));
    return 0;
}

/* Reading A19: psi (2*2^n floats, complex64 storage) <- e_{x0}, then every gate computed in
 * complex128 from the stored amplitudes and rounded to complex64 when stored. */
int oracle_run_c64store(int n, uint64_t x0, float *psi_ri, const og_gate *gates, int64_t ng, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const uint64_t N = 1ull << n;
    if (x0 >= N) return -1000000;
    memset(psi_ri, 0, sizeof(float) * 2 * N);
    psi_ri[2 * x0] = 1.0f;
    for (int64_t i = 0; i < ng; ++i)
        if (apply_gate_c64store(n, (cplx32 *)psi_ri, &gates[i]) != 0) return (int)(-(1 + i));
    return 0;
}

/* psi <- e_{x0}; then apply.  psi_ri has 2*2^n doubles. */
int oracle_run(int n, uint64_t x0, double *psi_ri, const og_gate *gates, int64_t ng, int nthreads) {
    const uint64_t N = 1ull << n;
    if (x0 >= N) return -1000000;
    memset(psi_ri, 0, sizeof(double) * 2 * N);
    psi_ri[2 * x0] = 1.0;
    return oracle_apply(n, psi_ri, gates, ng, nthreads);
}

/* sum |psi_j|^2 in double, fixed sequential order. */
double oracle_norm(int n, const double *psi_ri) {
    const uint64_t N = 1ull << n;
    double s = 0;
    for (uint64_t j = 0; j < N; ++j) s += psi_ri[2 * j] * psi_ri[2 * j] + psi_ri[2 * j + 1] * psi_ri[2 * j + 1];
    return s;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
