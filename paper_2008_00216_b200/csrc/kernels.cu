// kernels.cu -- hand-written sm_100a kernels of the state-vector hot path.
//
//   k_tile_pass      SURVEY.md 8(a) a5/a6: one HBM pass applies a fused
//                    sequence of dense k-qubit ops, diagonal-phase ops and
//                    in-tile CNOTs to every tile.  Tiles (2^h runs of 2^L
//                    contiguous amplitudes) are staged into shared memory by
//                    TMA bulk copies (cp.async.bulk + mbarrier) in a 3-stage
//                    ring on persistent CTAs, and written back by bulk stores.
//                    Paper analog: "apply all applicable gates to a resident
//                    cache line".
//   k_diag_pass      a8: standalone diagonal cluster, one read pass, writes
//                    only amplitudes whose phase != 1.
//   k_cnot_pass      a9: CNOT as a pure permutation, touches only the half of
//                    the state with control = 1.
//   k_norm_*         a10: fp64 fixed-shape reduction.
//   k_init_*, k_gather  a11.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <cstring>
#include <algorithm>

#include "pass_format.h"

namespace stv {

template <typename R> struct C2T;
template <> struct C2T<float> { using T = float2; };
template <> struct C2T<double> { using T = double2; };

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA bulk copies (sm_90+/sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(0x100000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, uint32_t sleep_ns = 0) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
        if (sleep_ns) __nanosleep(sleep_ns);   // back off: spinning steals issue slots from the consumers
    }
}
__device__ __forceinline__ void tma_load_1d(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_1d(void *dst, const void *src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
    uint64_t r = 0;
    for (uint64_t m = mask; m; m &= m - 1) {
        if (x & 1) r |= m & (0 - m);
        x >>= 1;
    }
    return r;
}

// ---------------------------------------------------------------------------
// complex helpers and the phase application (multiply-free for quarter turns)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 cfma(float2 m, float2 x, float2 acc) {
    acc.x = fmaf(m.x, x.x, acc.x);
    acc.x = fmaf(-m.y, x.y, acc.x);
    acc.y = fmaf(m.x, x.y, acc.y);
    acc.y = fmaf(m.y, x.x, acc.y);
    return acc;
}
__device__ __forceinline__ double2 cfma(double2 m, double2 x, double2 acc) {
    acc.x = fma(m.x, x.x, acc.x);
    acc.x = fma(-m.y, x.y, acc.x);
    acc.y = fma(m.x, x.y, acc.y);
    acc.y = fma(m.y, x.x, acc.y);
    return acc;
}

__device__ __forceinline__ void phase_cs(uint64_t ph, float &c, float &s) {
    // angle in [-pi, pi): hardware sin/cos (abs. error ~2^-21.4 on this range),
    // far inside the complex64 bars (|delta| <= 2e-6, F >= 1-1e-5)
    const float x = (float)(int32_t)(uint32_t)(ph >> 32) * 1.4629180792671596e-09f;  // 2 pi / 2^32
    __sincosf(x, &s, &c);
}
__device__ __forceinline__ void phase_cs(uint64_t ph, double &c, double &s) {
    const double x = (double)(int64_t)ph * 1.0842021724855044340074528008699e-19;  // 2^-63
    sincospi(x, &s, &c);
}

// amplitude *= exp(2 pi i ph / 2^64).  Quarter turns (+-1, +-i) use sign
// flips and (re, im) swaps only -- no floating-point multiply (PAPER.md
// L365-369, Sec. 4.1); other phases cost one complex multiply (reading A9).
template <typename C>
__device__ __forceinline__ C apply_phase(C a, uint64_t ph) {
    if (ph == 0) return a;
    if ((ph & ((1ull << 62) - 1)) == 0) {
        const uint32_t q = (uint32_t)(ph >> 62);
        C b;
        if (q == 2) { b.x = -a.x; b.y = -a.y; }
        else if (q == 1) { b.x = -a.y; b.y = a.x; }
        else { b.x = a.y; b.y = -a.x; }
        return b;
    }
    decltype(a.x) c, s;
    phase_cs(ph, c, s);
    C b;
    b.x = a.x * c - a.y * s;
    b.y = a.x * s + a.y * c;
    return b;
}

// ---------------------------------------------------------------------------
// diagonal-phase evaluation over a tile (shared by k_tile_pass and k_diag_pass)
//
// Tile-local index of the amplitudes a thread owns:
//   i = (r << (V + 8)) | (tid << V) | e,   e < 2^V, V = 1 (c64) / 0 (c128)
// so every thread touches 16 contiguous bytes per r.  The phase splits into
//   per-tile constant ct + per-thread part (thread bits) + per-amplitude part
// (e and r bits): the per-amplitude part is a precomputed quadratic table qf
// over the <= 6 "free" bits plus a sum of <= 6 linear terms (the GPU form of
// the paper's incremental Gray-code update).
// ---------------------------------------------------------------------------
struct DiagScratch {
    uint64_t ct;
    uint64_t pad;
    uint64_t linp[STV_MAX_TILE_BITS + 2];
    uint64_t qf[64];
};

// per-tile prep: linp[q] = lin[q] + sum of cross terms whose outside bit is set
// in full_base; ct = cst + outside linear + outside quadratic terms;
// qf[c] = in-tile pair terms among the free bits of combo c.
template <int V>
__device__ void diag_prep(const StvDiag *__restrict__ D, int S, uint64_t full_base, DiagScratch *sc) {
    const int tid = threadIdx.x;
    const uint8_t *rec = (const uint8_t *)D;
    if (tid < S) {
        uint64_t l = D->lin[tid];
        const StvTerm *cr = (const StvTerm *)(rec + D->cross_off);
        const int b = D->cross_start[tid], e = D->cross_start[tid + 1];
        for (int k = b; k < e; ++k)
            if ((full_base >> cr[k].b) & 1) l += cr[k].ang;
        sc->linp[tid] = l;
    }
    if (tid >= 32 && tid < 64) {
        const int lane = tid - 32;
        uint64_t acc = 0;
        const StvTerm *ol = (const StvTerm *)(rec + D->olin_off);
        for (int k = lane; k < D->n_olin; k += 32)
            if ((full_base >> ol[k].a) & 1) acc += ol[k].ang;
        const StvTerm *oq = (const StvTerm *)(rec + D->oquad_off);
        for (int k = lane; k < D->n_oquad; k += 32)
            if (((full_base >> oq[k].a) & 1) && ((full_base >> oq[k].b) & 1)) acc += oq[k].ang;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) sc->ct = D->cst + acc;
    }
    // free bits: F = [0, V) U [V+8, S)
    const int nr = S > V + 8 ? S - V - 8 : 0;
    const int nF = V + nr;
    if (tid >= 64 && tid < 64 + (1 << nF)) {
        const int c = tid - 64;
        int fpos[6];
        int m = 0;
        for (int f = 0; f < V; ++f) fpos[m++] = f;
        for (int f = 0; f < nr; ++f) fpos[m++] = V + 8 + f;
        uint64_t acc = 0;
        for (int a = 0; a < nF; ++a)
            if ((c >> a) & 1)
                for (int b = a + 1; b < nF; ++b)
                    if ((c >> b) & 1) acc += D->A[fpos[a]][fpos[b]];
        sc->qf[c] = acc;
    }
}

// per-thread constant and the linear coefficients of the free bits
template <int V>
__device__ __forceinline__ void diag_thread(const StvDiag *__restrict__ D, int S, const DiagScratch *sc,
                                            uint64_t &bt, uint64_t *lf, int &nF) {
    const int tid = threadIdx.x;
    const int tb_hi = min(S, V + 8);
    const int nr = S > V + 8 ? S - V - 8 : 0;
    nF = V + nr;
    bt = sc->ct;
    for (int q = V; q < tb_hi; ++q) {
        if (!((tid >> (q - V)) & 1)) continue;
        bt += sc->linp[q];
        for (int p = V; p < q; ++p)
            if ((tid >> (p - V)) & 1) bt += D->A[p][q];
    }
    for (int f = 0; f < nF; ++f) {
        const int fp = f < V ? f : V + 8 + (f - V);
        uint64_t l = sc->linp[fp];
        for (int q = V; q < tb_hi; ++q)
            if ((tid >> (q - V)) & 1) l += D->A[q][fp];
        lf[f] = l;
    }
}

// ---------------------------------------------------------------------------
// named barrier among the consumer warps (the producer warp never joins)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(STV_THREADS) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// dense k-qubit op on a shared-memory tile (register-resident 2^k vector).
// K <= 2: the whole matrix lives in registers for the op; K >= 3: rows are
// streamed from shared memory as 16-byte pairs of entries.
// ---------------------------------------------------------------------------
template <int K, typename C>
__device__ __forceinline__ uint32_t dense_base(uint32_t v, const int *tp) {
    uint32_t base = v;
#pragma unroll
    for (int b = 0; b < K; ++b) {
        const uint32_t lo = base & ((1u << tp[b]) - 1);
        base = ((base >> tp[b]) << (tp[b] + 1)) | lo;
    }
    return base;
}

template <int K>
__device__ __forceinline__ uint32_t dense_off(int l, const int *tp) {
    uint32_t o = 0;
#pragma unroll
    for (int b = 0; b < K; ++b)
        if ((l >> b) & 1) o |= 1u << tp[b];
    return o;
}

template <int K, typename C>
__device__ void dense_op_reg(C *__restrict__ tile, int S, const int *tp, const C *__restrict__ M, int ctid) {
    constexpr int D = 1 << K;
    C m[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) m[i] = M[i];
    uint32_t off[D];
#pragma unroll
    for (int l = 0; l < D; ++l) off[l] = dense_off<K>(l, tp);
    const uint32_t nvec = 1u << (S - K);
    if (sizeof(C) == 8 && tp[0] == 0) {
        // target on tile bit 0 (complex64): amplitude pairs (l, l|1) are one 16-B word
        for (uint32_t v = ctid; v < nvec; v += STV_THREADS) {
            const uint32_t base = dense_base<K, C>(v, tp);
            C x[D];
#pragma unroll
            for (int l = 0; l < D; l += 2) {
                const float4 q = *(const float4 *)&tile[base | off[l]];
                x[l].x = q.x; x[l].y = q.y; x[l + 1].x = q.z; x[l + 1].y = q.w;
            }
#pragma unroll
            for (int r = 0; r < D; r += 2) {
                C a0, a1;
                a0.x = a0.y = a1.x = a1.y = 0;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    a0 = cfma(m[r * D + c], x[c], a0);
                    a1 = cfma(m[(r + 1) * D + c], x[c], a1);
                }
                *(float4 *)&tile[base | off[r]] = make_float4(a0.x, a0.y, a1.x, a1.y);
            }
        }
        return;
    }
    for (uint32_t v = ctid; v < nvec; v += STV_THREADS) {
        const uint32_t base = dense_base<K, C>(v, tp);
        C x[D];
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = tile[base | off[l]];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            C acc;
            acc.x = 0;
            acc.y = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) acc = cfma(m[r * D + c], x[c], acc);
            tile[base | off[r]] = acc;
        }
    }
}

// K >= 3: matrix rows streamed from shared memory (broadcast), two rows per
// step with split accumulators -> four independent FMA chains per thread
template <int K, typename C>
__device__ void dense_op_smem(C *__restrict__ tile, int S, const int *tp, const C *__restrict__ M, int ctid) {
    constexpr int D = 1 << K;
    const uint32_t nvec = 1u << (S - K);
    uint32_t off[D];
#pragma unroll
    for (int l = 0; l < D; ++l) off[l] = dense_off<K>(l, tp);
    for (uint32_t v = ctid; v < nvec; v += STV_THREADS) {
        const uint32_t base = dense_base<K, C>(v, tp);
        C x[D];
#pragma unroll
        for (int l = 0; l < D; ++l) x[l] = tile[base | off[l]];
#pragma unroll 1
        for (int r = 0; r < D; r += 2) {
            C p0, p1, q0, q1;
            p0.x = p0.y = p1.x = p1.y = q0.x = q0.y = q1.x = q1.y = 0;
            const C *M0 = M + r * D;
            const C *M1 = M0 + D;
#pragma unroll
            for (int c = 0; c < D; c += 2) {
                p0 = cfma(M0[c], x[c], p0);
                p1 = cfma(M0[c + 1], x[c + 1], p1);
                q0 = cfma(M1[c], x[c], q0);
                q1 = cfma(M1[c + 1], x[c + 1], q1);
            }
            p0.x += p1.x; p0.y += p1.y;
            q0.x += q1.x; q0.y += q1.y;
            uint32_t o0 = 0, o1 = 0;     // off[r], off[r+1] without dynamic register indexing
#pragma unroll
            for (int b = 0; b < K; ++b) {
                if ((r >> b) & 1) o0 |= off[1 << b];
                if (((r + 1) >> b) & 1) o1 |= off[1 << b];
            }
            tile[base | o0] = p0;
            tile[base | o1] = q0;
        }
    }
}

template <typename C>
__device__ void cnot_op(C *__restrict__ tile, int S, int t, int c_loc, int ctid) {
    const uint32_t npair = 1u << (S - 1);
    for (uint32_t v = ctid; v < npair; v += STV_THREADS) {
        const uint32_t lo = v & ((1u << t) - 1);
        const uint32_t i0 = ((v >> t) << (t + 1)) | lo;
        if (c_loc >= 0 && !((i0 >> c_loc) & 1)) continue;
        const uint32_t i1 = i0 | (1u << t);
        C a = tile[i0];
        tile[i0] = tile[i1];
        tile[i1] = a;
    }
}

template <int V, typename C>
__device__ void diag_op_tile(C *__restrict__ tile, int S, const StvDiag *__restrict__ D, const DiagScratch *sc) {
    uint64_t bt, lf[6];
    int nF;
    diag_thread<V>(D, S, sc, bt, lf, nF);
    const uint32_t tsz = 1u << S;
    const int nr = 1 << (nF - V);                 // r combos; each covers 2^V amplitudes (16 B)
    for (int r = 0; r < nr; ++r) {
        const uint32_t i = ((uint32_t)r << (V + 8)) | ((uint32_t)threadIdx.x << V);
        if (i >= tsz) continue;
        uint64_t ph = bt + sc->qf[r << V];
#pragma unroll
        for (int f = V; f < 6; ++f)
            if (f < nF && ((r >> (f - V)) & 1)) ph += lf[f];
        if (V == 1) {
            const uint64_t ph1 = ph + lf[0] + sc->qf[(r << 1) | 1] - sc->qf[r << 1];
            if (ph == 0 && ph1 == 0) continue;
            float4 *p = (float4 *)&tile[i];
            const float4 q = *p;
            float2 a = make_float2(q.x, q.y), b = make_float2(q.z, q.w);
            a = apply_phase(a, ph);
            b = apply_phase(b, ph1);
            *p = make_float4(a.x, a.y, b.x, b.y);
        } else {
            if (ph == 0) continue;
            tile[i] = apply_phase(tile[i], ph);
        }
    }
}

// ---------------------------------------------------------------------------
// the fused tile pass: warp-specialised.
//   producer warps (kProdWarps): gather the tile's 2^h runs of 2^L amplitudes
//     into a kStages shared-memory ring -- 16-B cp.async (LDGSTS) per thread
//     for runs < 8 KB, one TMA bulk copy per run for longer runs (a 1-D bulk
//     copy costs ~160 SM cycles, measured: profiles/r01_tma_runlen.md);
//     completion is tracked by the stage's `full` mbarrier.
//   consumer warps (8): apply the pass's op sequence to the resident tile,
//     write it back with 16-B stores and release the stage (`empty`).
// ---------------------------------------------------------------------------
constexpr int kStages = 3;
constexpr int kHdrBytes = 1024;    // barriers, tile bases, DiagScratch
constexpr int kTileThreads = STV_THREADS;

__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// x + y in the "expanded" domain of mask (carries jump over the gaps):
// pdep(a + b, m) == masked_add(pdep(a, m), pdep(b, m), m)
__device__ __forceinline__ uint64_t masked_add(uint64_t x, uint64_t y, uint64_t m) {
    return ((x | ~m) + y) & m;
}

// Move one tile between global memory and a shared-memory stage with NT
// threads (index t): 16-B chunks, run-aware addressing.
template <bool kLoad, int NT>
__device__ __forceinline__ void tile_copy16(uint8_t *gstate, uint8_t *stile, uint64_t base, uint64_t hmask,
                                            uint32_t run_bytes, uint32_t nruns, uint32_t esz, int t) {
    const uint32_t cpr = run_bytes >> 4;             // 16-B chunks per run (power of two)
    if (cpr >= (uint32_t)NT) {
        const uint64_t d1 = hmask & (0 - hmask);     // pdep(1, hmask)
        uint64_t roff = 0;
        for (uint32_t r = 0; r < nruns; ++r) {
            uint8_t *g = gstate + (base | roff) * esz;
            uint8_t *sm = stile + (size_t)r * run_bytes;
            for (uint32_t w = t; w < cpr; w += NT) {
                if (kLoad) cp_async16(sm + (size_t)w * 16, g + (size_t)w * 16);
                else *(uint4 *)(g + (size_t)w * 16) = *(const uint4 *)(sm + (size_t)w * 16);
            }
            roff = masked_add(roff, d1, hmask);
        }
    } else {
        const uint32_t lc = 31 - __clz(cpr);
        const uint32_t total = nruns * cpr;
        const uint64_t dstep = pdep64((uint32_t)NT >> lc, hmask);
        uint64_t roff = pdep64((uint32_t)t >> lc, hmask);
        const uint32_t within = ((uint32_t)t & (cpr - 1)) * 16;
        for (uint32_t c = t; c < total; c += NT) {
            uint8_t *g = gstate + (base | roff) * esz + within;
            uint8_t *sm = stile + (size_t)c * 16;
            if (kLoad) cp_async16(sm, g);
            else *(uint4 *)g = *(const uint4 *)sm;
            roff = masked_add(roff, dstep, hmask);
        }
    }
}

template <typename R>
__global__ void __launch_bounds__(kTileThreads, sizeof(R) == 4 ? 2 : 1)
k_tile_pass(typename C2T<R>::T *__restrict__ state, const uint8_t *__restrict__ blob, uint32_t pass_off,
            uint32_t ntiles, int dbg_flags) {
    using C = typename C2T<R>::T;
    constexpr int V = sizeof(C) == 8 ? 1 : 0;
    extern __shared__ __align__(1024) uint8_t smem[];
    const StvPass *G = (const StvPass *)(blob + pass_off);
    const uint32_t rec_bytes = G->rec_bytes;           // whole pass record, staged in smem
    const uint32_t rec_pad = (rec_bytes + 127u) & ~127u;
    const StvPass *P = (const StvPass *)(smem + kHdrBytes);
    {
        const uint4 *src = (const uint4 *)G;
        uint4 *dst = (uint4 *)(smem + kHdrBytes);
        for (uint32_t k = threadIdx.x; k < rec_bytes / 16; k += blockDim.x) dst[k] = src[k];
    }
    const int S = G->S, L = G->L, h = G->h;
    const uint64_t out_mask = G->out_mask, rank_bits = G->rank_bits;
    const int nops = (dbg_flags & 1) ? 0 : G->nops;   // bit 0: data movement only (microbenchmark)
    const StvOp *ops = (const StvOp *)((const uint8_t *)P + G->ops_off);

    uint64_t *full = (uint64_t *)smem;                 // [3] (TMA path only)
    DiagScratch *sc = (DiagScratch *)(smem + 128);
    const uint8_t *mat = (const uint8_t *)P + G->mat_off;
    const int ntab = G->ntab;
    C *tables = (C *)(smem + kHdrBytes + rec_pad);
    const uint32_t tab_pad = ((uint32_t)ntab * 16 * sizeof(C) + 127u) & ~127u;
    C *tiles = (C *)(smem + kHdrBytes + rec_pad + tab_pad);
    const uint32_t esz = sizeof(C);
    const uint32_t tile_elems = 1u << S;
    const uint32_t run_bytes = (1u << L) * esz;
    const uint32_t nruns = 1u << h;
    const uint32_t tile_bytes = tile_elems * esz;
    const int tid = threadIdx.x;
    // one contiguous run per tile: a single TMA bulk copy (1-D bulk copies cost
    // ~160 SM cycles each, so strided tiles use 16-B cp.async instead)
    const bool use_tma = (h == 0) && tile_bytes <= (1u << 20) - 1;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    __syncthreads();

    const uint32_t first = blockIdx.x, stride = gridDim.x;
    const uint32_t my_tiles = first < ntiles ? (ntiles - first + stride - 1) / stride : 0;
    uint64_t hmask = 0;
    for (int r = 0; r < h; ++r) hmask |= 1ull << G->hpos[r];
    uint8_t *gstate = (uint8_t *)state;
    const uint64_t tstep = pdep64(stride, out_mask);
    uint64_t load_tb = pdep64(first, out_mask);        // base of the next tile to load
    uint32_t loaded = 0;

    auto issue = [&](int s) {                            // all threads: tile `loaded` -> stage s
        uint8_t *stile = (uint8_t *)(tiles + (size_t)s * tile_elems);
        if (loaded < my_tiles) {
            if (use_tma) {
                if (tid == 0) {
                    mbar_arrive_expect_tx(&full[s], tile_bytes);
                    tma_load_1d(stile, gstate + load_tb * esz, tile_bytes, &full[s]);
                }
            } else {
                tile_copy16<true, STV_THREADS>(gstate, stile, load_tb, hmask, run_bytes, nruns, esz, tid);
            }
        }
        cp_async_commit();
        load_tb = masked_add(load_tb, tstep, out_mask);
        ++loaded;
    };
    issue(0);
    issue(1);
    uint64_t base = pdep64(first, out_mask);
    uint32_t tphase = 0;                                 // TMA mbarrier parity per stage ring pass
    for (uint32_t j = 0; j < my_tiles; ++j) {
        const int s = (int)(j % kStages);
        cp_async_wait1();                                // this thread's copies of tile j landed
        if (use_tma) mbar_wait(&full[s], tphase);
        __syncthreads();                                 // everyone's copies visible; stage (j+2)%3 free
        issue((int)((j + 2) % kStages));
        C *tile = tiles + (size_t)s * tile_elems;
        const uint64_t full_base = base | rank_bits;
        for (int o = 0; o < nops; ++o) {
            const StvOp &op = ops[o];
            const int type = op.type;
            if (type == OP_DENSE) {
                int tp[STV_MAX_K];
#pragma unroll
                for (int b = 0; b < STV_MAX_K; ++b) tp[b] = op.tpos[b];
                const C *M = (const C *)(mat + op.mat_off);
                switch (op.k) {
                case 1: dense_op_reg<1, C>(tile, S, tp, M, tid); break;
                case 2: dense_op_reg<2, C>(tile, S, tp, M, tid); break;
                case 3: dense_op_smem<3, C>(tile, S, tp, M, tid); break;
                case 4: dense_op_smem<4, C>(tile, S, tp, M, tid); break;
                }
            } else if (type == OP_CNOT) {
                const bool on = op.c_phys < 0 || ((full_base >> op.c_phys) & 1);
                if (on) cnot_op<C>(tile, S, op.t_loc, op.c_loc, tid);
            } else {
                const StvDiag *D = (const StvDiag *)((const uint8_t *)P + op.diag_off);
                diag_prep<V>(D, S, full_base, sc);
                __syncthreads();
                diag_op_tile<V, C>(tile, S, D, sc);
            }
            __syncthreads();
        }
        tile_copy16<false, STV_THREADS>(gstate, (uint8_t *)tile, base, hmask, run_bytes, nruns, esz, tid);
        if (use_tma) fence_proxy_async();                // generic smem accesses before the next TMA write
        base = masked_add(base, tstep, out_mask);
        if (s == kStages - 1) tphase ^= 1;
    }
    cp_async_wait0();
}

// ---------------------------------------------------------------------------
// k_group_pass: the fused tile pass for gate-group plans (the default; SURVEY.md
// 8(a) a5/a6 + NEXT #1).  Tiles are staged in a 3-stage shared-memory ring by
// 16-B cp.async gathers into the swizzled layout of pass_format.h; per tile the
// group diagonal tables are built, then every group is one shared-memory round
// trip: each thread gathers one 16-amplitude vector (bank-conflict-free by the
// encoder's vector-bit order), runs the sub-op program in registers (U1 / U2
// matrices, CNOT register swaps, diagonal table factors) and scatters it back.
// Paper analog: all clustered gates applied to a resident cache line, gates
// kept in factored form.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t swz_hash_d(uint32_t x) {
    return (uint32_t)(__popc(x & kSwzM0) & 1) | ((uint32_t)(__popc(x & kSwzM1) & 1) << 1) |
           ((uint32_t)(__popc(x & kSwzM2) & 1) << 2);
}

// Move one tile between global memory and its swizzled shared-memory stage:
// thread t moves chunks c = t + NT*k (16 B each) to / from slot
// c ^ H(c >> 3) = c ^ H(t >> 3) ^ H(NT*k >> 3)  (NT = 256: disjoint bits).
template <bool kLoad, int NT>
__device__ __forceinline__ void tile_copy_swz(uint8_t *gstate, uint8_t *stile, uint64_t base, uint64_t hmask,
                                              uint32_t run_bytes, uint32_t nruns, uint32_t esz, int t,
                                              uint32_t hash_t) {
    static_assert(NT >= 8 && (NT & (NT - 1)) == 0, "chunk split assumes a power-of-two thread count");
    const uint32_t cpr = run_bytes >> 4;             // 16-B chunks per run (power of two)
    if (cpr >= (uint32_t)NT) {
        const uint64_t d1 = hmask & (0 - hmask);
        uint64_t roff = 0;
        for (uint32_t r = 0; r < nruns; ++r) {
            uint8_t *g = gstate + (base | roff) * esz;
            for (uint32_t w = t; w < cpr; w += NT) {
                const uint32_t c = r * cpr + w;
                const uint32_t slot = c ^ hash_t ^ swz_hash_d((c - (uint32_t)t) >> 3);
                uint8_t *sm = stile + (size_t)slot * 16;
                if (kLoad) cp_async16(sm, g + (size_t)w * 16);
                else *(uint4 *)(g + (size_t)w * 16) = *(const uint4 *)sm;
            }
            roff = masked_add(roff, d1, hmask);
        }
    } else {
        const uint32_t lc = 31 - __clz(cpr);
        const uint32_t total = nruns * cpr;
        const uint64_t dstep = pdep64((uint32_t)NT >> lc, hmask);
        uint64_t roff = pdep64((uint32_t)t >> lc, hmask);
        const uint32_t within = ((uint32_t)t & (cpr - 1)) * 16;
        for (uint32_t c = t; c < total; c += NT) {
            uint8_t *g = gstate + (base | roff) * esz + within;
            const uint32_t slot = c ^ hash_t ^ swz_hash_d((c - (uint32_t)t) >> 3);
            uint8_t *sm = stile + (size_t)slot * 16;
            if (kLoad) cp_async16(sm, g);
            else *(uint4 *)g = *(const uint4 *)sm;
            roff = masked_add(roff, dstep, hmask);
        }
    }
}

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}

// exp(2 pi i ph / 2^64): complex128 in double precision; complex64 from the top
// 32 bits of the turn count in single precision (argument quantum 2^-31 turn,
// |error| < 2e-7 rad, far inside the complex64 bars)
template <typename C>
__device__ __forceinline__ C unit_phase(uint64_t ph) {
    C r;
    if constexpr (sizeof(C) == 8) {
        float s, c;
        sincospif((float)(int32_t)(uint32_t)(ph >> 32) * 4.656612873077393e-10f, &s, &c);   // 2^-31
        r.x = c;
        r.y = s;
    } else {
        double s, c;
        sincospi((double)(int64_t)ph * 1.0842021724855044340074528008699e-19, &s, &c);   // 2^-63
        r.x = c;
        r.y = s;
    }
    return r;
}

template <int A, typename C>
__device__ __forceinline__ void g_u1(C (&x)[16], const C *__restrict__ M) {
    const C m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3];
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & (1 << A)) continue;
        const C p = x[l], q = x[l | (1 << A)];
        C u, w;
        u.x = 0; u.y = 0; w.x = 0; w.y = 0;
        u = cfma(m0, p, u); u = cfma(m1, q, u);
        w = cfma(m2, p, w); w = cfma(m3, q, w);
        x[l] = u;
        x[l | (1 << A)] = w;
    }
}

template <int A, int B, typename C>
__device__ __forceinline__ void g_u2(C (&x)[16], const C *__restrict__ M) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        C v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        C o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            C acc;
            acc.x = 0; acc.y = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) acc = cfma(M[r * 4 + c], v[c], acc);
            o[r] = acc;
        }
        x[l] = o[0];
        x[l | (1 << A)] = o[1];
        x[l | (1 << B)] = o[2];
        x[l | (1 << A) | (1 << B)] = o[3];
    }
}

// CNOT as predicated register swaps: target TB, in-register control CB (or -1)
template <int CB, int TB, typename C>
__device__ __forceinline__ void g_cnot(C (&x)[16], bool on) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & (1 << TB)) continue;
        if (CB >= 0 && !(l & (1 << (CB < 0 ? 0 : CB)))) continue;
        const C a = x[l], b = x[l | (1 << TB)];
        x[l] = on ? b : a;
        x[l | (1 << TB)] = on ? a : b;
    }
}

// ---- complex64 with packed FP32 (FFMA2, sm_100): with m = (m_re, m_im),
//   acc += m x  is  acc = FFMA2(x, m_re.bcast, acc); acc = FFMA2(-x.swapped.lo, m_im.bcast, acc)
// i.e. (x_re, x_im) m_re + (-x_im, x_re) m_im: two instructions, the swap and
// the one-lane negation are operand modifiers (.LO_HI.NP).
__device__ __forceinline__ float2 cmac2(float2 m, float2 x, float2 acc) {
    acc = __ffma2_rn(x, make_float2(m.x, m.x), acc);
    return __ffma2_rn(make_float2(-x.y, x.x), make_float2(m.y, m.y), acc);
}
__device__ __forceinline__ float2 cmul1(float2 m, float2 x) {
    return __ffma2_rn(make_float2(-x.y, x.x), make_float2(m.y, m.y), __fmul2_rn(x, make_float2(m.x, m.x)));
}

// one complex64 matrix entry as a single 64-bit uniform load (LDCU.64)
__device__ __forceinline__ float2 ld_c64(const float2 *p) {
    const unsigned long long w = *(const unsigned long long *)p;
    return make_float2(__uint_as_float((unsigned)w), __uint_as_float((unsigned)(w >> 32)));
}

template <int A>
__device__ __forceinline__ void g_u1p(float2 (&x)[16], const float2 *__restrict__ M) {
    float2 m[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) m[e] = ld_c64(M + e);
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & (1 << A)) continue;
        const float2 p = x[l], q = x[l | (1 << A)];
        x[l] = cmac2(m[1], q, cmul1(m[0], p));
        x[l | (1 << A)] = cmac2(m[3], q, cmul1(m[2], p));
    }
}

template <int A, int B>
__device__ __forceinline__ void g_u2p(float2 (&x)[16], const float2 (&m)[16]) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        const float2 v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        float2 o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            float2 acc = cmul1(m[r * 4], v[0]);
#pragma unroll
            for (int c = 1; c < 4; ++c) acc = cmac2(m[r * 4 + c], v[c], acc);
            o[r] = acc;
        }
        x[l] = o[0];
        x[l | (1 << A)] = o[1];
        x[l | (1 << B)] = o[2];
        x[l | (1 << A) | (1 << B)] = o[3];
    }
}

// table entry of a unit phase: (re, im) in the state's precision
template <typename C> struct TabEnt { using T = C; };

// The pass record of a group pass travels as a __grid_constant__ kernel
// parameter: every field, sub-op and matrix is read with uniform constant-bank
// loads (LDCU) into uniform registers, FFMA2 takes the matrix entries straight
// from them, and sub-op dispatch is a uniform branch.  Only the per-lane static
// phase tables are read from the device copy of the blob (global, L1-cached).
struct __align__(16) RecParam {
    uint8_t b[STV_REC_PARAM_BYTES];
};

// Group diagonal tables.  Half tables (every term on one register bit) have only
// per-tile CONSTANT terms: their entries are static and built once per CTA
// (prologue); per tile only the scalar exp(i cst) is refreshed (scal[t], applied
// with the table).  Full tables carry per-index-bit per-tile coefficients and are
// rebuilt per tile: lane b < 7 reduces the terms on index bit b, lane 31 the
// constant; one warp per table.
template <typename C, int NT>
__device__ __forceinline__ void build_tables(const StvPass *__restrict__ P, const uint8_t *__restrict__ grec,
                                             uint64_t fb, typename TabEnt<C>::T *__restrict__ tables,
                                             C *__restrict__ scal, int ctid, bool prologue) {
    const StvDTab *tabs = (const StvDTab *)((const uint8_t *)P + P->tab_off);
    const int ntab = P->ntab;
    const int lane = ctid & 31, warp = ctid >> 5;
    if (prologue) {   // static entries: half tables, and full tables without per-tile terms
        for (int t = warp; t < ntab; t += NT / 32) {
            const StvDTab &d = tabs[t];
            if (!d.half && d.nterm) continue;
            const uint64_t *stat = (const uint64_t *)(grec + d.stat_off);
            const int lb4 = d.half ? 3 : 4, stride = d.half ? STV_TAB_STRIDE_H : STV_TAB_STRIDE;
            for (int e = lane; e < ((1 << lb4) << d.m); e += 32)
                tables[d.ent_off + (uint32_t)(e >> lb4) * stride + (e & ((1 << lb4) - 1))] =
                    unit_phase<C>(__ldg(stat + e));
        }
        return;
    }
    // per tile: work items (a half table's scalar, or 32 entries of a full table with
    // per-tile terms) dealt round-robin to the warps, so one large table does not
    // serialise the build behind one warp
    int item = 0;
    for (int t = 0; t < ntab; ++t) {
        const StvDTab &d = tabs[t];
        const int nterm = d.nterm;
        if (!nterm) continue;
        const StvTerm *tm = (const StvTerm *)((const uint8_t *)P + d.term_off);
        if (d.half) {
            if ((item++ & (NT / 32 - 1)) != warp) continue;
            if constexpr (sizeof(C) == 8) {   // complex64: 32-bit turns, one REDUX (see below)
                const StvTerm *gtm = (const StvTerm *)(grec + d.term_off);
                uint32_t acc = 0;
                for (int i = lane; i < nterm; i += 32) {
                    const int qa = __ldg(&gtm[i].a), qb = __ldg(&gtm[i].b);
                    bool on = (fb >> qb) & 1;
                    if (qa <= -2) on = on && ((fb >> (-2 - qa)) & 1);
                    if (on) acc += (uint32_t)((__ldg((const unsigned long long *)&gtm[i].ang) + 0x80000000ull) >> 32);
                }
                acc = __reduce_add_sync(0xffffffffu, acc);
                if (lane == 0) scal[t] = unit_phase<C>((uint64_t)acc << 32);
                continue;
            }
            uint64_t lam = 0;                              // constant terms only
            for (int i = lane; i < nterm; i += 32) {
                const StvTerm q = tm[i];
                if (!((fb >> q.b) & 1)) continue;
                if (q.a <= -2 && !((fb >> (-2 - q.a)) & 1)) continue;
                lam += q.ang;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) lam += __shfl_xor_sync(0xffffffffu, lam, o);
            if (lane == 0) scal[t] = unit_phase<C>(lam);
            continue;
        }
        const int ne = 16 << d.m, nit = (ne + 31) >> 5;
        const int mine = (warp - item) & (NT / 32 - 1);    // first chunk of this table dealt to this warp
        item += nit;
        if (mine >= nit) continue;
        const uint64_t *stat = (const uint64_t *)(grec + d.stat_off);
        if constexpr (sizeof(C) == 8) {
            // complex64 uses the top 32 bits of a phase (unit_phase): the per-tile coefficients
            // are summed in 32-bit turns (each term rounded to 2^-32 turn, far inside the
            // complex64 bars), the terms spread over the lanes (device copy of the record) and
            // reduced per index bit with one REDUX each, instead of every lane scanning all terms
            const StvTerm *gtm = (const StvTerm *)(grec + d.term_off);
            uint32_t acc[7] = {0, 0, 0, 0, 0, 0, 0}, accc = 0;
            for (int i = lane; i < nterm; i += 32) {
                const int qa = __ldg(&gtm[i].a), qb = __ldg(&gtm[i].b);
                const uint64_t qang = __ldg((const unsigned long long *)&gtm[i].ang);
                bool on = (fb >> qb) & 1;
                if (qa <= -2) on = on && ((fb >> (-2 - qa)) & 1);
                const uint32_t v = on ? (uint32_t)((qang + 0x80000000ull) >> 32) : 0u;
#pragma unroll
                for (int b = 0; b < 7; ++b) acc[b] += qa == b ? v : 0u;
                accc += qa < 0 ? v : 0u;
            }
            uint32_t lb[7];
#pragma unroll
            for (int b = 0; b < 7; ++b) lb[b] = __reduce_add_sync(0xffffffffu, acc[b]);
            const uint32_t cst = __reduce_add_sync(0xffffffffu, accc);
            for (int e = (mine << 5) | lane; e < ne; e += NT) {
                uint32_t ph = (uint32_t)((__ldg(stat + e) + 0x80000000ull) >> 32) + cst;
#pragma unroll
                for (int b = 0; b < 7; ++b)
                    if ((e >> b) & 1) ph += lb[b];
                tables[d.ent_off + (uint32_t)(e >> 4) * STV_TAB_STRIDE + (e & 15)] = unit_phase<C>((uint64_t)ph << 32);
            }
            continue;
        }
        // lane b < 4 + m sums the terms on index bit b, lane 31 the constant
        uint64_t lam = 0;
        for (int i = 0; i < nterm; ++i) {
            const StvTerm q = tm[i];
            const int who = q.a >= 0 ? q.a : 31;
            if (who != lane || !((fb >> q.b) & 1)) continue;
            if (q.a <= -2 && !((fb >> (-2 - q.a)) & 1)) continue;
            lam += q.ang;
        }
        const uint64_t cst = __shfl_sync(0xffffffffu, lam, 31);
        uint64_t lb[7];
#pragma unroll
        for (int b = 0; b < 7; ++b) lb[b] = __shfl_sync(0xffffffffu, lam, b);
        for (int e = (mine << 5) | lane; e < ne; e += NT) {
            uint64_t ph = __ldg(stat + e) + cst;
#pragma unroll
            for (int b = 0; b < 7; ++b)
                if ((e >> b) & 1) ph += lb[b];
            tables[d.ent_off + (uint32_t)(e >> 4) * STV_TAB_STRIDE + (e & 15)] = unit_phase<C>(ph);
        }
    }
}

// real-matrix U1 / U2: every output is a real combination of complex inputs -- one
// FMUL2 + FFMA2s with broadcast real coefficients per output (half the work of a
// complex matrix)
template <typename C, typename R>
__device__ __forceinline__ C rmul(R m, C x) {
    if constexpr (sizeof(C) == 8) return __fmul2_rn(x, make_float2(m, m));
    else { C r; r.x = m * x.x; r.y = m * x.y; return r; }
}
template <typename C, typename R>
__device__ __forceinline__ C rmac(R m, C x, C acc) {
    if constexpr (sizeof(C) == 8) return __ffma2_rn(x, make_float2(m, m), acc);
    else { acc.x = fma(m, x.x, acc.x); acc.y = fma(m, x.y, acc.y); return acc; }
}
template <int A, typename C, typename R>
__device__ __forceinline__ void g_u1r(C (&x)[16], const R *__restrict__ M) {
    const R m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3];
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & (1 << A)) continue;
        const C p = x[l], q = x[l | (1 << A)];
        x[l] = rmac(m1, q, rmul<C, R>(m0, p));
        x[l | (1 << A)] = rmac(m3, q, rmul<C, R>(m2, p));
    }
}
template <int A, int B, typename C, typename R>
__device__ __forceinline__ void g_u2r(C (&x)[16], const R (&m)[16]) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        const C v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        C o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            C acc = rmul<C, R>(m[r * 4], v[0]);
#pragma unroll
            for (int c = 1; c < 4; ++c) acc = rmac(m[r * 4 + c], v[c], acc);
            o[r] = acc;
        }
        x[l] = o[0];
        x[l | (1 << A)] = o[1];
        x[l | (1 << B)] = o[2];
        x[l | (1 << A) | (1 << B)] = o[3];
    }
}

// two U2 on complementary pairs (A1,B1) then (A2,B2): written as two passes over the
// quads so the compiler sees both programs at once
template <int A1, int B1, int A2, int B2, typename C>
__device__ __forceinline__ void g_u2x2(C (&x)[16], const C (&ma)[16], const C (&mb)[16]) {
    if constexpr (sizeof(C) == 8) {
        g_u2p<A1, B1>(*(float2(*)[16]) & x, *(const float2(*)[16]) & ma);
        g_u2p<A2, B2>(*(float2(*)[16]) & x, *(const float2(*)[16]) & mb);
    } else {
        g_u2<A1, B1>(x, ma);
        g_u2<A2, B2>(x, mb);
    }
}

// half-table diagonal: amplitudes with local bit J set times row[l without bit J]
template <int J, typename C>
__device__ __forceinline__ void g_diagh(C (&x)[16], const C *__restrict__ row, bool with_scalar, C sc) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (!(l & (1 << J))) continue;
        const int c = ((l >> (J + 1)) << J) | (l & ((1 << J) - 1));
        C f = row[c];
        if constexpr (sizeof(C) == 8) {   // packed: FMUL2 + FFMA2 per complex product
            if (with_scalar) *(float2 *)&f = cmul1(*(const float2 *)&sc, *(const float2 *)&f);
            *(float2 *)&x[l] = cmul1(*(const float2 *)&f, *(float2 *)&x[l]);
        } else {
            if (with_scalar) f = cmul(f, sc);
            x[l] = cmul(x[l], f);
        }
    }
}

// Run a group's sub-op program on NV register vectors (same program; matrix
// entries come from uniform registers).
template <typename C, int NV>
__device__ __forceinline__ void run_subs(C (&x)[NV][16], const uint32_t (&braw)[NV], const StvSub *__restrict__ subs,
                                         int nsub, const uint8_t *__restrict__ mat, const StvDTab *__restrict__ tabs,
                                         const typename TabEnt<C>::T *__restrict__ tables, uint64_t full_base,
                                         uint32_t tord, uint64_t rank_bits, const C *__restrict__ scal) {
    constexpr bool kPacked = sizeof(C) == 8;
    using R = decltype(x[0][0].x);
    auto vsel = [&](uint32_t w) {   // 3 x 5-bit selectors: bits of the tile ordinal (31: always 0)
        return ((tord >> (w & 31u)) & 1u) | (((tord >> ((w >> 5) & 31u)) & 1u) << 1) |
               (((tord >> ((w >> 10) & 31u)) & 1u) << 2);
    };
    for (int k = 0; k < nsub; ++k) {
        const uint2 ca = *(const uint2 *)&subs[k];         // code, arg: one LDCU.64
        int code = (int)(ca.x & 0xffu);
        const C *M = (const C *)(mat + ca.y);
        // a per-tile variant op runs the plain U2 case on the variant's matrix
        if ((unsigned)(code - SUBC_U2V) < 6u) {
            M += vsel(ca.x >> 8) * 16;
            code -= SUBC_U2V - SUBC_U2;
        }
        // one flat switch over the dense sub-op codes (a single indirect uniform branch)
        switch (code) {
#define STV_U2(p, a, b)                                                                     \
    case SUBC_U2 + (p): {                                                                   \
        C m[16];                                                                            \
        if constexpr (kPacked) {                                                            \
            _Pragma("unroll") for (int e = 0; e < 16; ++e)                                  \
                *(float2 *)&m[e] = ld_c64((const float2 *)M + e);                           \
            _Pragma("unroll") for (int i = 0; i < NV; ++i)                                  \
                g_u2p<(a), (b)>(*(float2(*)[16]) & x[i], *(const float2(*)[16]) & m);      \
        } else {                                                                            \
            _Pragma("unroll") for (int e = 0; e < 16; ++e) m[e] = M[e];                     \
            _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u2<(a), (b)>(x[i], m);         \
        }                                                                                   \
        break;                                                                              \
    }
        STV_U2(0, 0, 1) STV_U2(1, 0, 2) STV_U2(2, 0, 3) STV_U2(3, 1, 2) STV_U2(4, 1, 3) STV_U2(5, 2, 3)
#undef STV_U2
#define STV_UX2(p, a1, b1, a2, b2)                                                               \
    case SUBC_U2X2 + (p): {   /* two U2 on complementary pairs */                                \
        const C *MA = (const C *)(mat + ca.y) + vsel(ca.x >> 8) * 16;                            \
        const C *MB = (const C *)(mat + subs[k].ctl) + vsel(subs[k].pad) * 16;                   \
        C m[16];   /* one matrix live at a time (the pair of them exceeds the uniform registers) */ \
        if constexpr (kPacked) {                                                                 \
            _Pragma("unroll") for (int e = 0; e < 16; ++e) *(float2 *)&m[e] = ld_c64((const float2 *)MA + e); \
            _Pragma("unroll") for (int i = 0; i < NV; ++i)                                       \
                g_u2p<a1, b1>(*(float2(*)[16]) & x[i], *(const float2(*)[16]) & m);             \
            asm volatile("" ::: "memory");                                                       \
            _Pragma("unroll") for (int e = 0; e < 16; ++e) *(float2 *)&m[e] = ld_c64((const float2 *)MB + e); \
            _Pragma("unroll") for (int i = 0; i < NV; ++i)                                       \
                g_u2p<a2, b2>(*(float2(*)[16]) & x[i], *(const float2(*)[16]) & m);             \
        } else {                                                                                 \
            _Pragma("unroll") for (int e = 0; e < 16; ++e) m[e] = MA[e];                         \
            _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u2<a1, b1>(x[i], m);                \
            _Pragma("unroll") for (int e = 0; e < 16; ++e) m[e] = MB[e];                         \
            _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u2<a2, b2>(x[i], m);                \
        }                                                                                        \
        break;                                                                                   \
    }
        STV_UX2(0, 0, 1, 2, 3) STV_UX2(1, 0, 2, 1, 3) STV_UX2(2, 0, 3, 1, 2)
#undef STV_UX2
#define STV_U1(a)                                                                           \
    case SUBC_U1 + (a): {                                                                   \
        if constexpr (kPacked) {                                                            \
            _Pragma("unroll") for (int i = 0; i < NV; ++i)                                  \
                g_u1p<(a)>(*(float2(*)[16]) & x[i], (const float2 *)M);                     \
        } else {                                                                            \
            _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u1<(a)>(x[i], M);               \
        }                                                                                   \
        break;                                                                              \
    }
        STV_U1(0) STV_U1(1) STV_U1(2) STV_U1(3)
#undef STV_U1
#define STV_CX(c, t)                                                                             \
    case SUBC_CNOT + 4 * ((c) + 1) + (t): {                                                      \
        const uint32_t ctl = subs[k].ctl, raw = ctl & 0xffffu, ph = ctl >> 16;                   \
        const bool pon = ph == 0 || ((full_base >> (ph - 1)) & 1);                               \
        _Pragma("unroll") for (int i = 0; i < NV; ++i)                                           \
            g_cnot<(c), (t)>(x[i], pon && (raw == 0 || (braw[i] & raw) != 0));                   \
        break;                                                                                   \
    }
        STV_CX(-1, 0) STV_CX(-1, 1) STV_CX(-1, 2) STV_CX(-1, 3)
        STV_CX(0, 1) STV_CX(0, 2) STV_CX(0, 3)
        STV_CX(1, 0) STV_CX(1, 2) STV_CX(1, 3)
        STV_CX(2, 0) STV_CX(2, 1) STV_CX(2, 3)
        STV_CX(3, 0) STV_CX(3, 1) STV_CX(3, 2)
#undef STV_CX
        case SUBC_DIAG: {   // per-tile table row of each vector's V-bits
            const StvDTab &d = tabs[ca.y];
            const uint32_t v0 = d.vraw[0], v1 = d.vraw[1], v2 = d.vraw[2];
            const uint32_t eo = d.ent_off;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const uint32_t r = ((braw[i] & v0) ? 1u : 0u) | ((braw[i] & v1) ? 2u : 0u) | ((braw[i] & v2) ? 4u : 0u);
                const typename TabEnt<C>::T *row = tables + eo + r * STV_TAB_STRIDE;
                if constexpr (kPacked) {
                    float2(&xv)[16] = *(float2(*)[16]) & x[i];
#pragma unroll
                    for (int l = 0; l < 16; ++l) xv[l] = cmul1(row[l], xv[l]);
                } else {
#pragma unroll
                    for (int l = 0; l < 16; ++l) x[i][l] = cmul(x[i][l], row[l]);
                }
            }
            break;
        }
#define STV_DH(j)                                                                                \
    case SUBC_DIAGH + (j): {   /* half table on local bit j */                                   \
        const StvDTab &d = tabs[ca.y];                                                           \
        const uint32_t eo = d.ent_off;                                                           \
        _Pragma("unroll") for (int i = 0; i < NV; ++i) {                                         \
            uint32_t r = (braw[i] & d.vraw[0]) ? 1u : 0u;   /* m <= 1: the common case */        \
            if (d.m > 1) {                                                                       \
                _Pragma("unroll") for (int q = 1; q < STV_MAX_VBITS_H; ++q)                      \
                    r |= ((braw[i] & d.vraw[q]) ? 1u : 0u) << q;                                 \
            }                                                                                    \
            const typename TabEnt<C>::T *row = tables + eo + r * STV_TAB_STRIDE_H;               \
            const bool ws = d.nterm != 0;                                                        \
            const C sc = ws ? scal[ca.y] : C();                                                  \
            g_diagh<(j)>(x[i], row, ws, sc);                                                     \
        }                                                                                        \
        break;                                                                                   \
    }
        STV_DH(0) STV_DH(1) STV_DH(2) STV_DH(3)
#undef STV_DH
#define STV_U1R(a)                                                                               \
    case SUBC_U1R + (a): {                                                                       \
        const R *MRl = (const R *)(mat + ca.y);                                                  \
        _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u1r<(a)>(x[i], MRl);                    \
        break;                                                                                   \
    }
        STV_U1R(0) STV_U1R(1) STV_U1R(2) STV_U1R(3)
#undef STV_U1R
#define STV_U2R(p, a, b)                                                                         \
    case SUBC_U2R + (p): {                                                                       \
        const R *MRl = (const R *)(mat + ca.y);                                                  \
        R m[16];                                                                                 \
        _Pragma("unroll") for (int e = 0; e < 16; ++e) m[e] = MRl[e];                            \
        _Pragma("unroll") for (int i = 0; i < NV; ++i) g_u2r<(a), (b)>(x[i], m);                 \
        break;                                                                                   \
    }
        STV_U2R(0, 0, 1) STV_U2R(1, 0, 2) STV_U2R(2, 0, 3) STV_U2R(3, 1, 2) STV_U2R(4, 1, 3) STV_U2R(5, 2, 3)
#undef STV_U2R
        default: break;
        }
    }
}

// One group on the resident tile: thread ctid owns vectors v = ctid + NT*(i + NV*k).
template <typename C, int NT, int NV>
__device__ __forceinline__ void group_vec_op(C *__restrict__ tile, const StvGroup &g, const StvPass *__restrict__ P,
                                             const uint8_t *__restrict__ mat,
                                             const typename TabEnt<C>::T *__restrict__ tables, uint64_t full_base,
                                             uint32_t tord, const uint8_t *__restrict__ grec,
                                             const C *__restrict__ scal, int ctid) {
    constexpr int TB = NT == 128 ? 7 : 8;   // log2(NT)
    static_assert((1 << TB) == NT, "NT must be 128 or 256");
    const int nvb = g.nvb;
    uint32_t braw0, bsw0;
    if (NT == 256 && grec) {   // precomputed per-thread bases of the first 8 vector bits (global tail)
        const uint32_t w = __ldg((const uint32_t *)(grec + g.vtab_off) + ctid);
        bsw0 = w & 0xffffu;
        braw0 = w >> 16;
    } else {
        braw0 = 0;
        bsw0 = 0;
#pragma unroll
        for (int b = 0; b < TB; ++b) {
            const uint2 vb = *(const uint2 *)g.vbit[b];
            if (b < nvb && ((ctid >> b) & 1)) {
                braw0 |= vb.x;
                bsw0 ^= vb.y;
            }
        }
    }
    uint32_t so[16];
#pragma unroll
    for (int l = 0; l < 16; l += 2) {
        const uint2 w = *(const uint2 *)&g.sw_off[l];
        so[l] = w.x;
        so[l + 1] = w.y;
    }
    const StvSub *subs = (const StvSub *)((const uint8_t *)P + g.sub_off);
    const StvDTab *tabs = (const StvDTab *)((const uint8_t *)P + P->tab_off);
    const int nsub = g.nsub;
    const bool pair16 = sizeof(C) == 8 && g.pair16;
    const uint32_t nvec = 1u << nvb;
    for (uint32_t v0 = ctid; v0 < nvec; v0 += NT * NV) {
        uint32_t braw[NV], bsw[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint32_t v = v0 + NT * i;
            braw[i] = braw0;
            bsw[i] = bsw0;
            for (int b = TB; b < nvb; ++b)
                if ((v >> b) & 1) {
                    braw[i] |= g.vbit[b][0];
                    bsw[i] ^= g.vbit[b][1];
                }
        }
        // predicated X flips folded into the gather / scatter addresses (pass_format.h)
        uint32_t bsw_g[NV], bsw_s[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            bsw_g[i] = bsw[i];
            bsw_s[i] = bsw[i];
        }
        if (g.nflip_g | g.nflip_s) {
            auto flip_delta = [&](int from, int cnt, uint32_t br) {
                uint32_t dlt = 0;
                for (int q = 0; q < cnt; ++q) {
                    const uint32_t f = g.flip[from + q];
                    const uint32_t a = f >> 17;
                    const bool on = (f & (1u << 16)) ? ((full_base >> a) & 1) != 0 : (br & a) != 0;
                    if (on) dlt ^= f & 0xffffu;
                }
                return dlt;
            };
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                bsw_g[i] ^= flip_delta(0, g.nflip_g, braw[i]);
                bsw_s[i] ^= flip_delta(STV_MAX_FLIPS, g.nflip_s, braw[i]);
            }
        }
        C x[NV][16];
        const bool live1 = NV == 1 || v0 + NT < nvec;   // tiny tiles: the second vector may not exist
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (i > 0 && !live1) {
#pragma unroll
                for (int l = 0; l < 16; ++l) { x[i][l].x = 0; x[i][l].y = 0; }
                continue;
            }
            if (pair16) {
#pragma unroll
                for (int l = 0; l < 16; l += 2) {
                    const float4 q = *(const float4 *)&tile[bsw_g[i] ^ so[l]];
                    x[i][l].x = q.x; x[i][l].y = q.y; x[i][l + 1].x = q.z; x[i][l + 1].y = q.w;
                }
            } else {
#pragma unroll
                for (int l = 0; l < 16; ++l) x[i][l] = tile[bsw_g[i] ^ so[l]];
            }
        }
        run_subs<C, NV>(x, braw, subs, nsub, mat, tabs, tables, full_base, tord, P->rank_bits, scal);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (i > 0 && !live1) continue;
            if (pair16) {
#pragma unroll
                for (int l = 0; l < 16; l += 2)
                    *(float4 *)&tile[bsw_s[i] ^ so[l]] = make_float4(x[i][l].x, x[i][l].y, x[i][l + 1].x, x[i][l + 1].y);
            } else {
#pragma unroll
                for (int l = 0; l < 16; ++l) tile[bsw_s[i] ^ so[l]] = x[i][l];
            }
        }
    }
}

constexpr int kGStagesDefault = 2;  // double-buffered tiles (prefetch distance 1)

// Tile copy state that does not change from tile to tile (computed once per CTA).
struct CopyPlan {
    uint64_t roff0, dstep, d1;
    uint32_t cpr, total, within;
    bool long_runs;
};

template <int NT>
__device__ __forceinline__ CopyPlan make_copy_plan(uint64_t hmask, uint32_t run_bytes, uint32_t nruns, int t) {
    CopyPlan c;
    c.cpr = run_bytes >> 4;
    c.long_runs = c.cpr >= (uint32_t)NT;
    c.d1 = hmask & (0 - hmask);
    c.total = nruns * c.cpr;
    const uint32_t lc = 31 - __clz(c.cpr);
    c.dstep = c.long_runs ? 0 : pdep64((uint32_t)NT >> lc, hmask);
    c.roff0 = c.long_runs ? 0 : pdep64((uint32_t)t >> lc, hmask);
    c.within = c.long_runs ? 0 : ((uint32_t)t & (c.cpr - 1)) * 16;
    return c;
}

// Swizzled tile copy (see tile_copy_swz) with per-CTA precomputed addressing;
// hk[k] = H((NT * k) >> 3) for the k-th chunk of this thread.
template <bool kLoad, int NT>
__device__ __forceinline__ void tile_copy_fast(uint8_t *gstate, uint8_t *stile, uint64_t base, uint64_t hmask,
                                               const CopyPlan &cp, uint32_t nruns, uint32_t esz, int t,
                                               uint32_t hash_t, const uint8_t *hk) {
    if (cp.long_runs) {
        uint64_t roff = 0;
        for (uint32_t r = 0; r < nruns; ++r) {
            uint8_t *g = gstate + (base | roff) * esz;
            for (uint32_t w = t; w < cp.cpr; w += NT) {
                const uint32_t c = r * cp.cpr + w;
                const uint32_t slot = c ^ hash_t ^ hk[(c - (uint32_t)t) / NT];
                uint8_t *sm = stile + (size_t)slot * 16;
                if (kLoad) cp_async16(sm, g + (size_t)w * 16);
                else *(uint4 *)(g + (size_t)w * 16) = *(const uint4 *)sm;
            }
            roff = masked_add(roff, cp.d1, hmask);
        }
    } else if ((hmask >> 32) == 0) {
        // all tile bits below 2^32: 32-bit offset arithmetic from the tile's base pointer
        uint8_t *tb = gstate + base * esz + cp.within;
        const uint32_t m32 = (uint32_t)hmask, step = (uint32_t)cp.dstep;
        uint32_t roff = (uint32_t)cp.roff0;
        uint32_t k = 0;
        for (uint32_t c = t; c < cp.total; c += NT, ++k) {
            uint8_t *g = tb + (size_t)roff * esz;
            const uint32_t slot = c ^ hash_t ^ hk[k];
            uint8_t *sm = stile + slot * 16u;
            if (kLoad) cp_async16(sm, g);
            else *(uint4 *)g = *(const uint4 *)sm;
            roff = ((roff | ~m32) + step) & m32;
        }
    } else {
        uint64_t roff = cp.roff0;
        uint32_t k = 0;
        for (uint32_t c = t; c < cp.total; c += NT, ++k) {
            uint8_t *g = gstate + (base | roff) * esz + cp.within;
            const uint32_t slot = c ^ hash_t ^ hk[k];
            uint8_t *sm = stile + (size_t)slot * 16;
            if (kLoad) cp_async16(sm, g);
            else *(uint4 *)g = *(const uint4 *)sm;
            roff = masked_add(roff, cp.dstep, hmask);
        }
    }
}

template <typename R, int NT, int NV, int kGStages, int kMinB>
__global__ void __launch_bounds__(NT, kMinB)
k_group_pass(typename C2T<R>::T *__restrict__ state, const uint8_t *__restrict__ blob, uint32_t pass_off,
             uint32_t ntiles, int dbg_flags, const __grid_constant__ RecParam rec) {
    using C = typename C2T<R>::T;
    extern __shared__ __align__(1024) uint8_t smem[];
    const StvPass *P = (const StvPass *)rec.b;
    const uint8_t *grec = blob + pass_off;
    const int S = P->S, L = P->L, h = P->h;
    const uint64_t out_mask = P->out_mask, rank_bits = P->rank_bits;
    const int nops = (dbg_flags & 1) ? 0 : P->nops;   // bit 0: data movement only (microbenchmark)
    const int ntab = P->ntab;
    const StvGroup *groups = (const StvGroup *)(rec.b + P->ops_off);
    const uint8_t *mat = rec.b + P->mat_off;
    const uint32_t esz = sizeof(C);
    const uint32_t tab_pad = (P->tab_entries * esz + 127u) & ~127u;
    uint8_t *hk = smem;                                                    // 1024 B: chunk hashes
    C *scal = (C *)(smem + 1024);                                          // 512 B: half-table scalars
    typename TabEnt<C>::T *tables = (typename TabEnt<C>::T *)(smem + 1536);
    C *tiles = (C *)(smem + 1536 + tab_pad);
    const uint32_t tile_elems = 1u << S;
    const uint32_t run_bytes = (1u << L) * esz;
    const uint32_t nruns = 1u << h;
    const int tid = threadIdx.x;
    const uint32_t hash_t = swz_hash_d((uint32_t)tid >> 3);
    for (int k = tid; k < 1024; k += NT) hk[k] = (uint8_t)swz_hash_d(((uint32_t)NT * (uint32_t)k) >> 3);
    uint64_t hmask = 0;
    for (int r = 0; r < h; ++r) hmask |= 1ull << P->hpos[r];
    const CopyPlan cp = make_copy_plan<NT>(hmask, run_bytes, nruns, tid);
    if (ntab && nops) build_tables<C, NT>(P, grec, 0, tables, scal, tid, true);   // static table entries
    __syncthreads();

    const uint32_t first = blockIdx.x, stride = gridDim.x;
    const uint32_t my_tiles = first < ntiles ? (ntiles - first + stride - 1) / stride : 0;
    uint8_t *gstate = (uint8_t *)state;
    const uint64_t tstep = pdep64(stride, out_mask);
    uint64_t load_tb = pdep64(first, out_mask);
    uint32_t loaded = 0;
    auto issue = [&](int s) {
        uint8_t *stile = (uint8_t *)(tiles + (size_t)s * tile_elems);
        if (loaded < my_tiles && !(dbg_flags & 2))   // bit 1: compute only (microbenchmark)
            tile_copy_fast<true, NT>(gstate, stile, load_tb, hmask, cp, nruns, esz, tid, hash_t, hk);
        cp_async_commit();
        load_tb = masked_add(load_tb, tstep, out_mask);
        ++loaded;
    };
    for (int s = 0; s < kGStages - 1; ++s) issue(s);
    uint64_t base = pdep64(first, out_mask);
    for (uint32_t j = 0; j < my_tiles; ++j) {
        const int s = (int)(j % kGStages);
        if constexpr (kGStages == 1) {                   // no ring: other CTAs on the SM overlap the copy
            if (j) __syncthreads();                      // previous tile's write-back reads are done
            issue(0);
            cp_async_wait0();
            __syncthreads();
        } else {
            cp_async_wait_n<kGStages - 2>();
            __syncthreads();                             // tile j visible; stage (j-1)%kGStages free
            issue((int)((j + kGStages - 1) % kGStages));
        }
        C *tile = tiles + (size_t)s * tile_elems;
        const uint64_t full_base = base | rank_bits;
        if (ntab && nops) {
            build_tables<C, NT>(P, grec, full_base, tables, scal, tid, false);
            __syncthreads();
        }
        for (int o = 0; o < nops; ++o) {
            group_vec_op<C, NT, NV>(tile, groups[o], P, mat, tables, full_base, first + j * stride, grec, scal, tid);
            __syncthreads();
        }
        if (!(dbg_flags & 2))
            tile_copy_fast<false, NT>(gstate, (uint8_t *)tile, base, hmask, cp, nruns, esz, tid, hash_t, hk);
        base = masked_add(base, tstep, out_mask);
    }
    cp_async_wait0();
}

#include "tc_pass.cuh"

// ---------------------------------------------------------------------------
// standalone diagonal pass (streaming; skip-write)
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(STV_THREADS)
k_diag_pass(typename C2T<R>::T *__restrict__ state, const uint8_t *__restrict__ blob, uint32_t pass_off,
            uint64_t nchunks) {
    using C = typename C2T<R>::T;
    constexpr int V = sizeof(C) == 8 ? 1 : 0;
    __shared__ DiagScratch sc;
    const StvPass *P = (const StvPass *)(blob + pass_off);
    const StvDiag *D = (const StvDiag *)((const uint8_t *)P + P->diag_off);
    const int S = P->S;
    const uint64_t rank_bits = P->rank_bits;
    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const uint64_t base = ch << S;
        __syncthreads();
        diag_prep<V>(D, S, base | rank_bits, &sc);
        __syncthreads();
        uint64_t bt, lf[6];
        int nF;
        diag_thread<V>(D, S, &sc, bt, lf, nF);
        const int nr = nF - V;
        const uint32_t tsz = 1u << S;
        for (int r = 0; r < (1 << nr); ++r) {
            const uint32_t i0 = ((uint32_t)r << (V + 8)) | ((uint32_t)threadIdx.x << V);
            if (i0 >= tsz) continue;
            if (V == 1) {
                float4 *p = (float4 *)(state + base + i0);
                float4 v = *p;
                uint64_t ph0 = bt + sc.qf[r << 1], ph1 = bt + sc.qf[(r << 1) | 1] + lf[0];
#pragma unroll
                for (int f = 1; f < 6; ++f)
                    if (f < nF && (((r << 1) >> f) & 1)) { ph0 += lf[f]; ph1 += lf[f]; }
                if (ph0 == 0 && ph1 == 0) continue;
                float2 a = make_float2(v.x, v.y), b = make_float2(v.z, v.w);
                a = apply_phase(a, ph0);
                b = apply_phase(b, ph1);
                *p = make_float4(a.x, a.y, b.x, b.y);
            } else {
                C *p = state + base + i0;
                uint64_t ph = bt + sc.qf[r];
#pragma unroll
                for (int f = 0; f < 6; ++f)
                    if (f < nF && ((r >> f) & 1)) ph += lf[f];
                if (ph == 0) continue;
                *p = apply_phase(*p, ph);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// standalone CNOT(c, t): swap alpha_i <-> alpha_{i ^ 2^t} where bit c = 1;
// c < 0: unconditional X on t (control resolved per rank)
// ---------------------------------------------------------------------------
template <typename C>
__global__ void __launch_bounds__(STV_THREADS)
k_cnot_pass(C *__restrict__ state, int c, int t, uint64_t nitems) {
    const int lo_b = c >= 0 ? min(c, t) : t, hi_b = c >= 0 ? max(c, t) : -1;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nitems;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = ((v >> lo_b) << (lo_b + 1)) | (v & ((1ull << lo_b) - 1));
        if (hi_b >= 0) i = ((i >> hi_b) << (hi_b + 1)) | (i & ((1ull << hi_b) - 1));
        if (c >= 0) i |= 1ull << c;
        const uint64_t j = i | (1ull << t);
        C a = state[i];
        state[i] = state[j];
        state[j] = a;
    }
}

// swap physical index bits a and b (a != b): exchanges alpha_{..1_a..0_b..} <-> alpha_{..0_a..1_b..}
// ---------------------------------------------------------------------------
// norm: fp64 partials over a fixed grid, fixed-shape trees (deterministic)
// ---------------------------------------------------------------------------
template <typename C>
__global__ void __launch_bounds__(STV_THREADS) k_norm_partial(const C *__restrict__ state, uint64_t N, double *part) {
    __shared__ double red[STV_THREADS / 32];
    const uint64_t per = (N + gridDim.x - 1) / gridDim.x;
    const uint64_t b = blockIdx.x * per, e = min(N, b + per);
    double acc = 0;
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const C a = state[i];
        acc += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < STV_THREADS / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(STV_THREADS) k_norm_final(const double *part, int np, double *out) {
    __shared__ double red[STV_THREADS];
    double acc = 0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = STV_THREADS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// ---------------------------------------------------------------------------
// measurement sampling (NEXT #3), over LOGICAL index order (include/sv.h):
// logical chunk c = indices [4096 c, 4096 (c+1)); lane i of a warp owns the 128
// consecutive logical indices 4096 c + 128 i + k.  Every |a_j|^2 is read through
// the frame (physical p = P(j) xor xmask; P moves logical bit q to physical bit
// perm[q]); amplitudes another rank owns count 0 (distributed: the per-rank
// arrays are summed).  Lane sums are sequential over k in every kernel, so the
// chunk masses, the per-shot lane sums and the in-lane scan add the same values
// in the same order.
// ---------------------------------------------------------------------------
constexpr int kSampChunk = 4096;
static int num_sms();

struct SampMap {
    uint64_t plo[128];     // P(k) for the low 7 logical bits (k < 128)
    int32_t perm[64];      // logical qubit -> physical bit
    uint64_t xmask;
    uint64_t N;            // 2^n logical amplitudes
    uint64_t lmask;        // local physical bits
    uint64_t rank_bits;    // this rank's value of the physical bits >= n_local
    int32_t n, n_local;
};

// physical index (xmask applied) of logical j with its low 7 bits cleared
__device__ __forceinline__ uint64_t samp_base(const SampMap &m, uint64_t j) {
    uint64_t p = m.xmask;
    for (int q = 7; q < m.n; ++q) p ^= ((j >> q) & 1ull) << m.perm[q];
    return p;
}
// |a_j|^2 of logical j = (base index) + k; 0 if j >= N or another rank owns it
template <typename C>
__device__ __forceinline__ double samp_p(const C *__restrict__ st, const SampMap &m, uint64_t base, uint64_t j, int k) {
    if (j >= m.N) return 0.0;
    const uint64_t p = base ^ m.plo[k];
    if ((p >> m.n_local) != m.rank_bits) return 0.0;
    const C a = st[p & m.lmask];
    return (double)a.x * (double)a.x + (double)a.y * (double)a.y;
}
// sequential sum of the 128 values of (chunk c, lane)
template <typename C>
__device__ __forceinline__ double samp_lane_sum(const C *__restrict__ st, const SampMap &m, uint64_t c, int lane) {
    const uint64_t j0 = c * kSampChunk + (uint64_t)lane * 128;
    const uint64_t base = samp_base(m, j0);
    double acc = 0;
    for (int k = 0; k < 128; ++k) acc += samp_p(st, m, base, j0 + k, k);
    return acc;
}

template <typename C>
__global__ void __launch_bounds__(256) k_sample_mass(const C *__restrict__ st, const __grid_constant__ SampMap m,
                                                     uint64_t nchunks, double *__restrict__ mass) {
    const int lane = threadIdx.x & 31;
    for (uint64_t c = blockIdx.x * 8ull + (threadIdx.x >> 5); c < nchunks; c += gridDim.x * 8ull) {
        double acc = samp_lane_sum(st, m, c, lane);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {                 // fixed tree
            const double v = __shfl_xor_sync(0xffffffffu, acc, o);
            acc = ((lane & o) ? v + acc : acc + v);
        }
        if (lane == 0) mass[c] = acc;
    }
}

// per shot s: the 32 lane sums of its chunk
template <typename C>
__global__ void __launch_bounds__(256) k_sample_lanes(const C *__restrict__ st, const __grid_constant__ SampMap m,
                                                      const uint64_t *__restrict__ chunk, uint64_t nshots,
                                                      double *__restrict__ lanes) {
    const int lane = threadIdx.x & 31;
    for (uint64_t s = blockIdx.x * 8ull + (threadIdx.x >> 5); s < nshots; s += gridDim.x * 8ull)
        lanes[s * 32 + lane] = samp_lane_sum(st, m, chunk[s], lane);
}

// per shot s: the lane L whose inclusive prefix (sequential over lanes) first exceeds
// the residual res[s]; on a rounding miss, the highest lane with mass (res2 = -1:
// take its last nonzero value).  The 128 values of lane L go to vals[s][*].
template <typename C>
__global__ void __launch_bounds__(256) k_sample_vals(const C *__restrict__ st, const __grid_constant__ SampMap m,
                                                     const uint64_t *__restrict__ chunk, const double *__restrict__ res,
                                                     const double *__restrict__ lanes, uint64_t nshots,
                                                     int32_t *__restrict__ pick_lane, double *__restrict__ res2,
                                                     double *__restrict__ vals) {
    const int lane = threadIdx.x & 31;
    for (uint64_t s = blockIdx.x * 8ull + (threadIdx.x >> 5); s < nshots; s += gridDim.x * 8ull) {
        const double r = res[s];
        const double mine = lanes[s * 32 + lane];
        double incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, incl > r && mine > 0);
        const unsigned nz = __ballot_sync(0xffffffffu, mine > 0);
        const double excl = incl - mine;
        int L;
        double r2;
        if (hit) {
            L = __ffs(hit) - 1;
            r2 = __shfl_sync(0xffffffffu, r - excl, L);
        } else {                                     // rounding miss: the last lane with mass
            L = nz ? 31 - __clz(nz) : 31;
            r2 = -1.0;
        }
        if (lane == 0) {
            pick_lane[s] = L;
            res2[s] = r2;
        }
        const uint64_t j0 = chunk[s] * kSampChunk + (uint64_t)L * 128;
        const uint64_t base = samp_base(m, j0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = lane + 32 * q;
            vals[s * 128 + k] = samp_p(st, m, base, j0 + k, k);
        }
    }
}

// per shot s: the first k of lane L whose sequential cumulative value exceeds
// res2[s] (and has mass); on a miss (or res2 < 0) the last k with mass -> logical index
__global__ void __launch_bounds__(256) k_sample_pick(const uint64_t *__restrict__ chunk,
                                                     const int32_t *__restrict__ pick_lane,
                                                     const double *__restrict__ res2, const double *__restrict__ vals,
                                                     uint64_t nshots, uint64_t N, uint64_t *__restrict__ out) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nshots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const double r = res2[s];
        const double *v = vals + s * 128;
        double cum = 0;
        int pick = -1, last = -1;
        for (int k = 0; k < 128; ++k) {
            const double p = v[k];
            cum += p;
            if (p > 0) last = k;
            if (r >= 0 && p > 0 && cum > r) {
                pick = k;
                break;
            }
        }
        if (pick < 0) pick = last >= 0 ? last : 127;
        const uint64_t j = chunk[s] * kSampChunk + (uint64_t)pick_lane[s] * 128 + (uint64_t)pick;
        out[s] = j < N ? j : N - 1;
    }
}

static SampMap make_samp_map(const int32_t *perm, uint64_t xmask, int n, int n_local, uint64_t rank_bits) {
    SampMap m;
    std::memset(&m, 0, sizeof(m));
    for (int q = 0; q < 64; ++q) m.perm[q] = q < n ? perm[q] : q;
    for (int k = 0; k < 128; ++k) {
        uint64_t p = 0;
        for (int q = 0; q < 7 && q < n; ++q) p |= (uint64_t)((k >> q) & 1) << m.perm[q];
        m.plo[k] = p;
    }
    m.xmask = xmask;
    m.N = 1ull << n;
    m.n = n;
    m.n_local = n_local;
    m.lmask = n_local >= 64 ? ~0ull : (1ull << n_local) - 1;
    m.rank_bits = rank_bits;
    return m;
}

// phase 0: chunk masses (count = nchunks, a = mass); 1: per-shot lane sums (a = lanes,
// count * 32); 2: lane pick + the lane's values (a = lanes, input); 3: in-lane pick
cudaError_t launch_sample(int phase, bool c128, const void *state, const int32_t *perm, uint64_t xmask, int n,
                          int n_local, uint64_t rank_bits, uint64_t count, const uint64_t *chunk, const double *res,
                          double *a, int32_t *pick_lane, double *res2, double *vals, uint64_t *out, cudaStream_t st,
                          int *kernels) {
    const SampMap m = make_samp_map(perm, xmask, n, n_local, rank_bits);
    const unsigned gw = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((count + 7) / 8, (uint64_t)num_sms() * 16));
    switch (phase) {
    case 0:
        if (c128) k_sample_mass<double2><<<gw, 256, 0, st>>>((const double2 *)state, m, count, a);
        else k_sample_mass<float2><<<gw, 256, 0, st>>>((const float2 *)state, m, count, a);
        break;
    case 1:
        if (c128) k_sample_lanes<double2><<<gw, 256, 0, st>>>((const double2 *)state, m, chunk, count, a);
        else k_sample_lanes<float2><<<gw, 256, 0, st>>>((const float2 *)state, m, chunk, count, a);
        break;
    case 2:
        if (c128)
            k_sample_vals<double2><<<gw, 256, 0, st>>>((const double2 *)state, m, chunk, res, a, count, pick_lane,
                                                        res2, vals);
        else
            k_sample_vals<float2><<<gw, 256, 0, st>>>((const float2 *)state, m, chunk, res, a, count, pick_lane, res2,
                                                       vals);
        break;
    default: {
        const unsigned g =
            (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((count + 255) / 256, (uint64_t)num_sms() * 8));
        k_sample_pick<<<g, 256, 0, st>>>(chunk, pick_lane, res2, vals, count, m.N, out);
    }
    }
    ++*kernels;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// init / readout
// ---------------------------------------------------------------------------
template <typename C>
__global__ void __launch_bounds__(STV_THREADS) k_fill(C *__restrict__ state, uint64_t N, C val, int64_t one_at, C one) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
        state[i] = ((int64_t)i == one_at) ? one : val;
}

struct GatherMap {
    int32_t perm[64];      // logical qubit -> actual physical bit
    uint64_t xmask;
    int32_t n;
    int32_t n_local;
    uint64_t rank_bits;    // this rank's global value (>> n_local)
};

// out[k] = alpha(logical j_k) for the amplitudes this rank owns; others untouched
template <typename C, typename O>
__global__ void __launch_bounds__(STV_THREADS)
k_gather(const C *__restrict__ state, const uint64_t *__restrict__ idx, uint64_t first, uint64_t count, GatherMap gm,
         O *__restrict__ out) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t j = idx ? idx[k] : first + k;
        uint64_t p = 0;
        for (int q = 0; q < gm.n; ++q) p |= ((j >> q) & 1) << gm.perm[q];
        p ^= gm.xmask;
        if ((p >> gm.n_local) != gm.rank_bits) continue;
        const C a = state[p & ((1ull << gm.n_local) - 1)];
        O o;
        o.x = a.x;
        o.y = a.y;
        out[k] = o;
    }
}

// ---------------------------------------------------------------------------
// host launchers (called from api.cpp)
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static size_t tile_smem_bytes(int S, uint32_t rec_bytes, int ntab, size_t esz) {
    return kHdrBytes + ((rec_bytes + 127u) & ~127u) + (((size_t)ntab * 16 * esz + 127u) & ~(size_t)127) +
           (size_t)kStages * ((size_t)esz << S);
}

cudaError_t launch_tile_pass(bool c128, void *state, const uint8_t *dblob, uint32_t pass_off, int S, int n_local,
                             uint32_t rec_bytes, int ntab, cudaStream_t st, int *kernels) {
    const size_t esz = c128 ? 16 : 8;
    const size_t smem = tile_smem_bytes(S, rec_bytes, ntab, esz);
    const uint64_t ntiles = 1ull << (n_local - S);
    int occ = 0;
    cudaError_t e;
    if (c128) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_tile_pass<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr = true;
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_pass<double>, kTileThreads, smem);
    } else {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_tile_pass<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr = true;
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_pass<float>, kTileThreads, smem);
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    uint64_t grid = (uint64_t)num_sms() * occ;
    if (grid > ntiles) grid = ntiles;
    if (ntiles >> 32) return cudaErrorInvalidValue;
    static const int dbg = getenv("STV_TILE_DEBUG") ? atoi(getenv("STV_TILE_DEBUG")) : 0;
    if (c128)
        k_tile_pass<double><<<(unsigned)grid, kTileThreads, smem, st>>>((double2 *)state, dblob, pass_off, (uint32_t)ntiles, dbg);
    else
        k_tile_pass<float><<<(unsigned)grid, kTileThreads, smem, st>>>((float2 *)state, dblob, pass_off, (uint32_t)ntiles, dbg);
    e = cudaGetLastError();
    ++*kernels;
    return e;
}

template <typename R, int NT, int NV, int NS, int MB = sizeof(R) == 4 ? 3 : 2>
static cudaError_t group_launch(void *state, const uint8_t *dblob, uint32_t pass_off, uint32_t ntiles, size_t smem,
                                const RecParam &rp, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_group_pass<R, NT, NV, NS, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_group_pass<R, NT, NV, NS, MB>, NT, smem);
    if (occ < 1) return cudaErrorInvalidConfiguration;
    uint64_t grid = (uint64_t)num_sms() * occ;
    if (grid > ntiles) grid = ntiles;
    static const int dbg = getenv("STV_TILE_DEBUG") ? atoi(getenv("STV_TILE_DEBUG")) : 0;
    k_group_pass<R, NT, NV, NS, MB><<<(unsigned)grid, NT, smem, st>>>((typename C2T<R>::T *)state, dblob, pass_off,
                                                                   ntiles, dbg, rp);
    return cudaGetLastError();
}

cudaError_t launch_group_pass(bool c128, void *state, const uint8_t *dblob, const uint8_t *hrec, uint32_t pass_off,
                              int S, int n_local, uint32_t rec_bytes, uint32_t tab_entries, double flops_per_amp,
                              cudaStream_t st, int *kernels) {
    const size_t esz = c128 ? 16 : 8;
    // tuning knob STV_GCFG (measured on c2): 0 = 256 threads x 1 vector,
    // one tile buffer, 4 CTAs/SM at 64 registers (default, best: the other CTAs of the SM hide
    // each CTA's tile load); 1 = 128 threads x 2 vectors; 2 = 3-stage ring; 3 = 2-stage ring,
    // 3 CTAs/SM at 80 registers (the previous default)
    static const int cfg = getenv("STV_GCFG") ? atoi(getenv("STV_GCFG")) : 0;
    (void)flops_per_amp;
    const int ns = c128 ? kGStagesDefault : cfg == 0 ? 1 : cfg == 2 ? 3 : kGStagesDefault;
    const size_t smem = 1536 + (((size_t)tab_entries * esz + 127u) & ~(size_t)127) + (size_t)ns * (esz << S);
    const uint64_t ntiles = 1ull << (n_local - S);
    if (smem > 227 * 1024 || (ntiles >> 32) || rec_bytes > STV_REC_PARAM_BYTES) return cudaErrorInvalidValue;
    static thread_local RecParam rp;
    std::memcpy(rp.b, hrec, rec_bytes);
    cudaError_t e;
    if (c128) e = group_launch<double, 128, 1, kGStagesDefault>(state, dblob, pass_off, (uint32_t)ntiles, smem, rp, st);
    else if (cfg == 1) e = group_launch<float, 128, 2, kGStagesDefault>(state, dblob, pass_off, (uint32_t)ntiles, smem, rp, st);
    else if (cfg == 2) e = group_launch<float, 256, 1, 3>(state, dblob, pass_off, (uint32_t)ntiles, smem, rp, st);
    else if (cfg == 3) e = group_launch<float, 256, 1, 2>(state, dblob, pass_off, (uint32_t)ntiles, smem, rp, st);
    else e = group_launch<float, 256, 1, 1, 4>(state, dblob, pass_off, (uint32_t)ntiles, smem, rp, st);
    ++*kernels;
    return e;
}

// tensor-core group pass (tc_pass.cuh): 2 CTAs per SM (TMEM 256 columns each); a
// double-buffered tile ring when it fits the shared memory of 2 CTAs, else one buffer
// TMA tensor map of a tensor-core pass's tiles (tc_pass.cuh TcTma): dims (16 amplitudes) x
// [rest of the low run, stride 128 B] x (tile base: stride 2^L amplitudes, box 1) x up to 3 runs
// of consecutive high tile bits; further high bits are looped by the kernel.  cuTensorMapEncodeTiled
// comes from the driver through cudaGetDriverEntryPoint (no link-time libcuda dependency).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
    }
    return fn;
}

static bool make_tile_tmap(CUtensorMap *tm, TcTma *t, void *state, const StvPass *P, int n_local) {
    std::memset(t, 0, sizeof(*t));
    static const bool off = getenv("STV_NO_TMA") && atoi(getenv("STV_NO_TMA"));
    EncodeTiledFn enc = encode_tiled_fn();
    if (off || !enc || !P->swz_tma || P->L < 4 || n_local - P->L > 32) return false;
    cuuint64_t gdim[5];
    cuuint64_t gstr[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    int r = 0;
    uint64_t box_elems = 16;
    gdim[0] = 16;
    box[0] = 16;
    r = 1;
    if (P->L > 4) {
        gdim[r] = 1ull << (P->L - 4);
        gstr[r - 1] = 128;
        box[r] = 1u << (P->L - 4);
        box_elems <<= P->L - 4;
        ++r;
    }
    t->bdim = r;   // the tile base
    gdim[r] = 1ull << (n_local - P->L);
    gstr[r - 1] = 8ull << P->L;
    box[r] = 1;
    ++r;
    for (int i = 0; i < P->h;) {   // runs of consecutive high tile bits, ascending
        int j = i;
        while (j + 1 < P->h && P->hpos[j + 1] == P->hpos[j] + 1) ++j;
        const int len = j - i + 1, start = P->hpos[i];
        if (r < 5 && len <= 8) {
            gdim[r] = 1ull << len;
            gstr[r - 1] = 8ull << start;
            box[r] = 1u << len;
            box_elems <<= len;
            ++r;
        } else {
            for (int k = i; k <= j; ++k) t->extra_mask |= 1ull << P->hpos[k];
        }
        i = j + 1;
    }
    while (r < 5) {
        gdim[r] = 1;
        gstr[r - 1] = gstr[r - 2];
        box[r] = 1;
        ++r;
    }
    t->nld = 1u << __builtin_popcountll(t->extra_mask);
    t->box_bytes = (uint32_t)(box_elems * 8);
    t->L = P->L;
    if (box_elems * t->nld != (1ull << P->S)) return false;
    const CUresult cr = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, state, gdim, gstr, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return false;
    static const int st_env = getenv("STV_TMA_STORE") ? atoi(getenv("STV_TMA_STORE")) : 0;
    t->on = st_env ? 2 : 1;
    return true;
}

template <int NS, bool FULL>
static cudaError_t tc_launch(void *state, const uint8_t *dblob, uint32_t pass_off, uint32_t ntiles, size_t smem,
                             const CUtensorMap &tm, const TcTma &tma, const RecParam &rp, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_tc_group_pass<NS, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, STV_TC_SMEM_CAP);
        attr = true;
    }
    uint64_t grid = (uint64_t)num_sms() * 2;
    if (grid > ntiles) grid = ntiles;
    // STV_NO_HALFSYNC=1: a CTA barrier at every group boundary (A/B switch of the per-half barriers)
    static const int dbg = (getenv("STV_TILE_DEBUG") ? atoi(getenv("STV_TILE_DEBUG")) : 0) |
                           (getenv("STV_NO_HALFSYNC") ? 256 : 0);
    k_tc_group_pass<NS, FULL><<<(unsigned)grid, 256, smem, st>>>((float2 *)state, dblob, pass_off, ntiles, dbg, tm, tma,
                                                                 rp);
    return cudaGetLastError();
}

cudaError_t launch_tc_group_pass(void *state, const uint8_t *dblob, const uint8_t *hrec, uint32_t pass_off, int S,
                                 int n_local, uint32_t rec_bytes, uint32_t tab_entries, int ntcop, cudaStream_t st,
                                 int *kernels) {
    // shared memory (tc_pass.cuh): TcShared region | tile ring | operator slots | scalars | tables
    const size_t fixed = kTcShBytes + (size_t)ntcop * kTcOpBytes + 512 + (((size_t)tab_entries * 8 + 127u) & ~(size_t)127);
    const size_t tile = (size_t)8 << S;
    const uint64_t ntiles = 1ull << (n_local - S);
    const size_t cap = STV_TC_SMEM_CAP;   // 2 CTAs per SM (the encoder checks the same bound)
    if (fixed + tile > cap || (ntiles >> 32) || rec_bytes > STV_REC_PARAM_BYTES) return cudaErrorInvalidValue;
    static thread_local RecParam rp;
    std::memcpy(rp.b, hrec, rec_bytes);
    static thread_local CUtensorMap tm;
    TcTma tma;
    make_tile_tmap(&tm, &tma, state, (const StvPass *)hrec, n_local);
    static const int ns_env = getenv("STV_TC_NS") ? atoi(getenv("STV_TC_NS")) : 2;
    const bool two = ns_env >= 2 && fixed + 2 * tile <= cap, full = S == 12;
    cudaError_t e;
    if (two) e = full ? tc_launch<2, true>(state, dblob, pass_off, (uint32_t)ntiles, fixed + 2 * tile, tm, tma, rp, st)
                      : tc_launch<2, false>(state, dblob, pass_off, (uint32_t)ntiles, fixed + 2 * tile, tm, tma, rp, st);
    else e = full ? tc_launch<1, true>(state, dblob, pass_off, (uint32_t)ntiles, fixed + tile, tm, tma, rp, st)
                  : tc_launch<1, false>(state, dblob, pass_off, (uint32_t)ntiles, fixed + tile, tm, tma, rp, st);
    ++*kernels;
    return e;
}

cudaError_t launch_diag_pass(bool c128, void *state, const uint8_t *dblob, uint32_t pass_off, int S, int n_local,
                             cudaStream_t st, int *kernels) {
    const uint64_t nch = 1ull << (n_local - S);
    uint64_t grid = (uint64_t)num_sms() * 8;
    if (grid > nch) grid = nch;
    if (c128)
        k_diag_pass<double><<<(unsigned)grid, STV_THREADS, 0, st>>>((double2 *)state, dblob, pass_off, nch);
    else
        k_diag_pass<float><<<(unsigned)grid, STV_THREADS, 0, st>>>((float2 *)state, dblob, pass_off, nch);
    ++*kernels;
    return cudaGetLastError();
}

static unsigned grid_for(uint64_t items) {
    uint64_t g = (items + STV_THREADS - 1) / STV_THREADS;
    const uint64_t cap = (uint64_t)num_sms() * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

cudaError_t launch_cnot(bool c128, void *state, int c, int t, int n_local, cudaStream_t st, int *kernels) {
    const uint64_t items = 1ull << (n_local - (c >= 0 ? 2 : 1));
    if (c128) k_cnot_pass<double2><<<grid_for(items), STV_THREADS, 0, st>>>((double2 *)state, c, t, items);
    else k_cnot_pass<float2><<<grid_for(items), STV_THREADS, 0, st>>>((float2 *)state, c, t, items);
    ++*kernels;
    return cudaGetLastError();
}

cudaError_t launch_norm(bool c128, const void *state, uint64_t N, double *part, int np, double *out, cudaStream_t st,
                        int *kernels) {
    if (c128) k_norm_partial<double2><<<np, STV_THREADS, 0, st>>>((const double2 *)state, N, part);
    else k_norm_partial<float2><<<np, STV_THREADS, 0, st>>>((const float2 *)state, N, part);
    k_norm_final<<<1, STV_THREADS, 0, st>>>(part, np, out);
    *kernels += 2;
    return cudaGetLastError();
}

cudaError_t launch_fill(bool c128, void *state, uint64_t N, double val, int64_t one_at, cudaStream_t st, int *kernels) {
    if (c128) {
        double2 v = make_double2(val, 0), o = make_double2(1, 0);
        k_fill<double2><<<grid_for(N), STV_THREADS, 0, st>>>((double2 *)state, N, v, one_at, o);
    } else {
        float2 v = make_float2((float)val, 0), o = make_float2(1, 0);
        k_fill<float2><<<grid_for(N), STV_THREADS, 0, st>>>((float2 *)state, N, v, one_at, o);
    }
    ++*kernels;
    return cudaGetLastError();
}

cudaError_t launch_gather(bool c128, const void *state, const uint64_t *didx, uint64_t first, uint64_t count,
                          const GatherMap &gm, bool out_native, void *dout, cudaStream_t st, int *kernels) {
    const unsigned g = grid_for(count);
    if (c128)
        k_gather<double2, double2><<<g, STV_THREADS, 0, st>>>((const double2 *)state, didx, first, count, gm,
                                                               (double2 *)dout);
    else if (out_native)
        k_gather<float2, float2><<<g, STV_THREADS, 0, st>>>((const float2 *)state, didx, first, count, gm,
                                                             (float2 *)dout);
    else
        k_gather<float2, double2><<<g, STV_THREADS, 0, st>>>((const float2 *)state, didx, first, count, gm,
                                                              (double2 *)dout);
    ++*kernels;
    return cudaGetLastError();
}

}  // namespace stv

// ---------------------------------------------------------------------------
// remap pack/unpack: chunk c = local indices whose bits
// lbits[i] equal bit i of c; element k of the chunk inserts those bits into k
// ---------------------------------------------------------------------------
namespace stv {
struct PackSpec {
    int32_t pos[8];    // ascending local bit positions
    int32_t bit[8];    // value for each position
    int32_t m;
};

template <typename C>
__global__ void __launch_bounds__(STV_THREADS)
k_pack(C *__restrict__ state, C *__restrict__ buf, PackSpec ps, uint64_t first, uint64_t count, int unpack) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t i = first + k;
        for (int b = 0; b < ps.m; ++b) {
            const int p = ps.pos[b];
            i = ((i >> p) << (p + 1)) | ((uint64_t)ps.bit[b] << p) | (i & ((1ull << p) - 1));
        }
        if (unpack) state[i] = buf[k];
        else buf[k] = state[i];
    }
}

cudaError_t launch_pack(bool c128, const void *state, void *dst, const int *lbits, int m, uint32_t chunk,
                        uint64_t first, uint64_t count, int n_local, bool unpack, cudaStream_t st, int *kernels) {
    (void)n_local;
    PackSpec ps;
    ps.m = m;
    int order[8];
    for (int i = 0; i < m; ++i) order[i] = i;
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            if (lbits[order[j]] < lbits[order[i]]) { int t = order[i]; order[i] = order[j]; order[j] = t; }
    for (int i = 0; i < m; ++i) {
        ps.pos[i] = lbits[order[i]];
        ps.bit[i] = (chunk >> order[i]) & 1;
    }
    if (c128)
        k_pack<double2><<<grid_for(count), STV_THREADS, 0, st>>>((double2 *)state, (double2 *)dst, ps, first, count, unpack);
    else
        k_pack<float2><<<grid_for(count), STV_THREADS, 0, st>>>((float2 *)state, (float2 *)dst, ps, first, count, unpack);
    ++*kernels;
    return cudaGetLastError();
}
}  // namespace stv
