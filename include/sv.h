/*
 * include/sv.h -- C ABI of the B200-native fused-gate state-vector engine.
 *
 * The boundary named by BASELINE.json north_star, item (1):
 *   sv_create(n, dtype) / sv_apply_circuit(gate list) / sv_get_amplitudes / sv_norm
 * plus the lifecycle/inspection calls of SURVEY.md 8(b).  Plain C types only:
 * no torch types cross this boundary.  PyTorch (through the thin Python
 * binding paper_2008_00216_b200/) only supplies device memory, the CUDA
 * stream and process groups.
 *
 * Method:
 *   * a circuit on n qubits acts on the 2^n complex amplitudes alpha_j of a
 *     state vector (Sec. 2); gates are applied in place to the
 *     2^{n-q} disjoint sets of 2^q amplitudes (Sec. 3);
 *   * gates are clustered after commutation-aware reordering (Sec. 4.5,
 *     L609-637), diagonal gates are aggregated per amplitude (Sec. 4.3,
 *     L416-541) and the state is stored in 32-bit float (Sec. 4.1).
 *
 * Conventions:
 *   A1 qubit q <-> bit q of the amplitude index j (LSB first).
 *   A2 for 2-qubit gates (q0, q1) the gate's local index is 2*b(q0) + b(q1):
 *      q0 is the MSB, i.e. the CNOT control.
 *   Amplitudes are interleaved (re, im): complex64 = 2 x float (8 B),
 *   complex128 = 2 x double (16 B).
 *
 * Ownership: the library owns the device state unless a buffer is given to
 * sv_wrap (then the caller's buffer must outlive the state).  Gate arrays and
 * matrices are caller-owned and only read during the call.  Output arrays are
 * caller-owned host memory.
 *
 * Errors: every call returns sv_status; sv_last_error() gives a thread-local
 * message naming the offending gate index where relevant.  Validation of a
 * gate list is all-or-nothing before any launch (SPEC.md L59-83 conventions).
 * A CUDA (or NCCL) failure in the middle of a circuit leaves the state
 * POISONED: every later call except sv_destroy returns SV_ERR_STATE.
 * One sv_state must not be used from two threads at once.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SV_OK = 0,
    SV_ERR_INVALID_ARG = 1,   /* bad qubit / kind / matrix / index / n        */
    SV_ERR_OUT_OF_MEMORY = 2, /* device or pinned-host allocation failed      */
    SV_ERR_CUDA = 3,          /* CUDA runtime error (state poisoned)          */
    SV_ERR_NCCL = 4,          /* NCCL error (state poisoned)                  */
    SV_ERR_UNSUPPORTED = 5,   /* feature not available (e.g. no NCCL loaded)  */
    SV_ERR_STATE = 6          /* state poisoned by an earlier failure         */
} sv_status;

typedef enum { SV_C64 = 0, SV_C128 = 1 } sv_dtype;

/* Gate kinds.  Matrices in DESIGN.md "Gate table":
 *   SV_H, SV_X (NOT), SV_Z, SV_CNOT, SV_CZ
 *   SV_S (= P = Z^1/2), SV_SX (X^1/2), SV_SY (Y^1/2, the L170 matrix), SV_T
 *                                               PAPER.md L165-171
 *   SV_SW  W^1/2 = T X^1/2 T^dagger            (reading A4)
 *   SV_Y   Pauli Y
 *   SV_SWAP                                     PAPER.md L1224-1228 (hushed)
 *   SV_CPHASE(phi) = diag(1,1,1,e^{i phi})      (reading A6; R_k: phi=2pi/2^k)
 *   SV_FSIM(theta, phi)                         (reading A5)
 *   SV_U1 / SV_U2  user 2x2 / 4x4 unitary, row-major (re, im) doubles in `m`
 */
typedef enum {
    SV_H = 0, SV_X, SV_Y, SV_Z, SV_S, SV_T, SV_SX, SV_SY, SV_SW,
    SV_CZ, SV_CNOT, SV_SWAP, SV_CPHASE, SV_FSIM, SV_U1, SV_U2,
    SV_NUM_KINDS
} sv_gate_kind;

#define SV_GATE_ADJOINT 0x1u /* apply the conjugate transpose of the gate */

typedef struct {
    int32_t kind;        /* sv_gate_kind                                  */
    uint32_t flags;      /* SV_GATE_ADJOINT                               */
    int32_t q0, q1;      /* qubits; q1 = -1 for one-qubit gates           */
    double theta, phi;   /* SV_CPHASE uses phi; SV_FSIM uses theta, phi   */
    const double *m;     /* SV_U1: 8 doubles, SV_U2: 32 doubles; else NULL */
} sv_gate;

/* Planner / executor options (NULL = defaults). */
#define SV_OPT_PROFILE      0x01u /* per-pass CUDA-event timing into sv_stats  */
#define SV_OPT_NO_RELABEL   0x02u /* apply SWAP/X/fSim(pi/2) as data movement  */
#define SV_OPT_NO_REORDER   0x04u /* no commutation-aware reordering (Sec 4.5) */
#define SV_OPT_ONE_GATE     0x08u /* one pass per gate (no fusion at all)      */
#define SV_OPT_NO_DIAG_FOLD 0x10u /* never fold diagonal gates into matrices   */
#define SV_OPT_NO_GROUPS    0x20u /* one shared-memory round trip per op (no register-resident gate groups) */
/* 0x40u reserved (was an experimental warp-per-tile kernel; ignored)                                     */
#define SV_OPT_NO_VARIANTS  0x80u /* do not merge 2-qubit sub-op chains into per-tile variant matrices      */
#define SV_OPT_NO_TC        0x100u /* complex64 gate groups on the CUDA-core FMA path only (no tcgen05 pass) */
#define SV_OPT_NO_SINK      0x400u /* keep diagonal terms over in-tile non-register bits in place (no sinking
                                        to the end of a gate group's program; tensor-core planning) */
#define SV_OPT_TMA          0x800u /* tensor-core passes: tiles staged with TMA tensor copies (SWIZZLE_128B
                                        layout) instead of 16-B cp.async (measured slower on c2/c4: opt-in) */
#define SV_OPT_NO_PLAN_CACHE 0x200u /* plan from scratch: do not reuse the plan of an identical earlier call
                                        (same gates, frame and options; the last 4 are kept per state) */
typedef struct {
    int32_t kmax;        /* max qubits of one fused dense block (1..4; register bits of a gate group); 0 = 4 */
    int32_t tile_bits;   /* max tile bits |S| of a fused pass; 0 = default              */
    int32_t low_bits;    /* min contiguous low bits in every tile; 0 = default            */
    int32_t budget;      /* per-pass compute budget, FMA-equivalents per amplitude; 0 = default */
    uint32_t flags;      /* SV_OPT_*                                                    */
} sv_options;

typedef struct sv_state sv_state;

/* Allocate a 2^n state on the current CUDA device (library-owned), |0...0>,
 * identity frame, default stream.  Errors: INVALID_ARG (n < 1, n > 40),
 * OUT_OF_MEMORY. */
sv_status sv_create(int n, sv_dtype dt, sv_state **out);

/* Wrap a caller-owned device buffer of >= 2^n amplitudes (e.g. a torch
 * tensor; 256-B aligned) and run on `cuda_stream` (a cudaStream_t, may be
 * NULL for the legacy default stream).  The buffer is initialised to |0..0>. */
sv_status sv_wrap(int n, sv_dtype dt, void *dev_buf, size_t bytes, void *cuda_stream,
                  sv_state **out);

/* Multi-GPU: rank r of world = 2^g ranks holds the 2^{n-g}
 * amplitudes whose top g physical index bits equal r.  `nccl_unique_id` is a
 * 128-byte ncclUniqueId created on rank 0 and broadcast by the caller (e.g.
 * torch.distributed).  `dev_buf` may be NULL (library allocates).  All calls
 * on a distributed state are collective: every rank passes identical
 * arguments.  Errors: UNSUPPORTED if NCCL cannot be loaded. */
sv_status sv_create_dist(int n, sv_dtype dt, const void *nccl_unique_id, int rank, int world,
                         void *dev_buf, size_t bytes, void *cuda_stream, sv_state **out);

/* Single-GPU emulation of a 2^g-rank partition ("virtual shards", SURVEY.md
 * 4 tier T2): the same planner and global-qubit remaps, with the all-to-all
 * done as device-to-device copies on one GPU. */
sv_status sv_create_virtual(int n, sv_dtype dt, int g, sv_state **out);

/* |x>: amplitude 1 at index x, 0 elsewhere; resets the frame.  x < 2^n. */
sv_status sv_set_basis(sv_state *s, uint64_t x);

/* Uniform superposition H^{(x)n}|0> = 2^{-n/2} sum_j |j> (PAPER.md L640
 * footnote, L1058-1060: the initial Hadamard layer as an initialisation). */
sv_status sv_set_uniform(sv_state *s);

/* psi <- U_G ... U_1 psi (gates in list order).  Validates the whole list
 * first (INVALID_ARG names the gate index; nothing is launched), plans
 * (relabel frame, Sec. 4.5 reordering, fusion, diagonal clustering, global
 * remaps), runs all passes on the state's stream and returns after the
 * stream completes. */
sv_status sv_apply_circuit(sv_state *s, const sv_gate *gates, size_t ng, const sv_options *opt);

/* Amplitudes at logical indices: idx[k] if idx != NULL, else first + k, for
 * k < count.  out receives 2*count doubles (re, im); complex64 values are
 * widened exactly.  Index >= 2^n -> INVALID_ARG. */
sv_status sv_get_amplitudes(sv_state *s, const uint64_t *idx, uint64_t first, size_t count,
                            double *out);

/* Raw readout in the state's own dtype (8 or 16 B per amplitude) of logical
 * indices [first, first+count) into host memory `out` (pinned or pageable). */
sv_status sv_read_state(sv_state *s, uint64_t first, uint64_t count, void *out);

/* sum_j |alpha_j|^2 in double with a fixed-shape reduction tree
 * (deterministic). */
sv_status sv_norm(sv_state *s, double *out);

/* Measurement sampling ("Simulating
 * measurements is then straightforward"; SPEC S:L286-292 sample_measurement).
 *   out[s] (s < shots) = logical basis index j drawn with probability |a_j|^2 / sum |a|^2.
 * Definition, in LOGICAL index order (independent of the internal frame and of the
 * partition): u_s = (splitmix64 output s+1 for `seed`, >> 11) * 2^-53 (counter-based,
 * so the result is deterministic given seed); the sample is the first logical index j
 * at which the cumulative sum of |a_0|^2 + ... + |a_j|^2 exceeds u_s * total.
 * Evaluation: fp64 |a|^2 read through the frame; 4096-index chunks of 32 lanes x 128
 * consecutive indices; chunk masses as a fixed warp tree, prefix-summed on the host in
 * order; per shot the lane and then the index inside the lane by sequential scans (a
 * rounding miss at a boundary falls back to the last index with mass).  The result can
 * differ from the exact definition only where u_s * total lies within summation rounding
 * of a cumulative-sum boundary.
 * out: caller host memory of `shots` uint64.  shots == 0 is a no-op.
 * Errors: SV_ERR_INVALID_ARG (NULL out with shots > 0, total mass <= 0 or not finite).
 * Distributed: collective (per-rank partial sums are all-reduced); every rank returns
 * all samples. */
sv_status sv_sample(sv_state *s, uint64_t seed, size_t shots, uint64_t *out);

typedef struct {
    double plan_ms;        /* host planning time of the last sv_apply_circuit      */
    double run_ms;         /* device time of all passes (events on the stream)     */
    int32_t n_pass[8];     /* by kind: fused-tile, tile-low, tile-high, diag, cnot,
                              remap, init, other                                   */
    double pass_ms[8];     /* filled when SV_OPT_PROFILE                           */
    double alg_bytes;      /* algorithmic HBM bytes of all passes      */
    double remap_bytes;    /* bytes sent per rank in remaps                        */
    int32_t n_ops[4];      /* ops inside fused passes: dense, diag, cnot, -        */
    int32_t n_kernels;     /* kernels launched by the last call                    */
    double h2d_bytes;      /* host->device bytes copied by the last call (plan)    */
    double alg_flops;      /* algorithmic flops of the fused tile passes */
    double tc_flops;       /* tensor-core flops issued by the tcgen05 group passes
                              (3xTF32: 3 real 32x32 products per 16-amplitude vector and
                              operator step = 384 flop per amplitude per step)     */
    int32_t n_tc_pass;     /* group passes that ran on the tensor-core kernel       */
    int32_t n_tc_steps;    /* their operator (MMA) steps                            */
} sv_stats;
sv_status sv_last_run_stats(const sv_state *s, sv_stats *out);

/* Current frame: perm[q] = physical bit holding logical qubit q, and the
 * X-flip mask over physical bits (stored index = P(j) xor xmask). */
sv_status sv_get_frame(const sv_state *s, int32_t *perm, uint64_t *xmask);

/* Host-only: the plan sv_apply_circuit would run, from an identity frame on
 * a 2^n state with n_global global qubits, as JSON (passes, ops, matrices,
 * diagonal forms, remaps, final frame).  Used by the CPU plan-interpreter
 * tests; needs no GPU.  If cap is too small, *needed gets the size. */
sv_status sv_plan_json(int n, int n_global, sv_dtype dt, const sv_gate *gates, size_t ng,
                       const sv_options *opt, char *buf, size_t cap, size_t *needed);

/* Host-only: the encoded device plan blob (pass_format.h) the kernels would
 * read, for the CPU blob-emulator tests; pass_off[i] = byte offset of pass i
 * (at most max_passes entries written; *npasses = total). */
sv_status sv_plan_blob(int n, int n_global, sv_dtype dt, const sv_gate *gates, size_t ng,
                       const sv_options *opt, uint8_t *buf, size_t cap, size_t *needed,
                       uint32_t *pass_off, size_t max_passes, size_t *npasses);

/* Host-only: the all-to-all schedule of one global<->local qubit swap
 * (SURVEY.md 8(e)): for rank `rank` of 2^g, swapping global bits `gbits`
 * (mask over [0,g)) with local physical bits `lbits` (ascending, same count
 * m), chunk c (the m-bit value of lbits) goes to peer[c]; peer[c] == rank
 * means the chunk stays.  Used by the world_size-2 gloo tests. */
sv_status sv_remap_peers(int g, int rank, uint32_t gbits, int m, int32_t *peer);

sv_status sv_destroy(sv_state *s);
const char *sv_last_error(void);
const char *sv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SV_H_ */
