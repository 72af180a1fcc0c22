// tc_pass.cuh -- tensor-core gate-group pass, complex64.
// Included by kernels.cu after the FMA group pass (it reuses its tile copy,
// swizzled gather/scatter addressing, per-tile tables and the sub-op program
// interpreter run_subs).
//
// A group's sub-op program (pass_format.h StvSub) is split by the encoder into
// steps (StvTcStep): E steps run on each thread's 16-amplitude register vector
// exactly as in k_group_pass (diagonal tables over V-bits, CNOTs controlled by
// V-bits: everything that differs between the vectors of a tile); M steps are
// runs of sub-ops whose action is the same for every vector of the tile
// (U1/U2 matrices, per-tile variants, in-register CNOTs, V-bit-free diagonal
// tables).  An M step's product is ONE dense 16 x 16 complex operator U
// ("fused k-qubit block"; the paper's contrast case of
// multiplied-out clusters applied with MACs, L383-384), applied with
// tcgen05.mma kind::tf32:
//   * real embedding: amplitude l of a vector is the pair (re, im) at real
//     index k = 2l + ri; out = A . B with B[2l+ri][2l'+ro] = (Ur, -Ui; Ui, Ur)
//     of U[l'][l] -- a 32 x 32 real matrix, N = K = 32;
//   * A = the tile's 256 vectors (rows) in TMEM, two M = 128 blocks; B in shared
//     memory, K-major SWIZZLE_NONE canonical layout; D (fp32) in TMEM;
//   * 3xTF32: x = x_hi + x_lo with x_hi = tf32(x), D = A_hi B_hi + A_hi B_lo +
//     A_lo B_hi (the dropped A_lo B_lo term is ~2^-22 relative), accumulated in
//     fp32 -- complex64 accuracy (DESIGN.md a7 error budget).
// U is built on the device by running the step's sub-ops on the 16 basis
// vectors (lane j of one warp computes column j), so it is exactly the product
// the FMA path applies; it depends on the tile only through the step's `dep`
// bits of the tile base and is rebuilt only when they change.  Each CTA walks
// a contiguous range of tile ordinals whose dep bits are the slowest-varying
// (StvPass.tperm), so a CTA rebuilds its operators a few times per pass.
#pragma once

// ---------------------------------------------------------------------------
// tcgen05 / TMEM PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
// 32 lanes x 32 columns of 32 bit: thread i <-> TMEM lane (base + i), register j <-> column j
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] . B[smem descriptor]: kind::tf32, cta_group::1
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "TCW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TCW;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// shared-memory matrix descriptor, SWIZZLE_NONE K-major canonical layout: core
// matrix = 8 rows x 16 B; lbo = byte stride of K-adjacent core matrices, sbo =
// byte stride of 8-row groups; version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = 32, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
// byte offset of B^T[n][k] (n = output real index, k = input real index) in an operator slot
__device__ __forceinline__ uint32_t tc_bt_off(int n, int k) {
    return (uint32_t)((n & 7) * 16 + (k & 3) * 4 + (k >> 2) * 128 + (n >> 3) * 1024);
}
constexpr uint32_t kTcOpBytes = STV_TC_OP_BYTES;   // hi (4 KB) + lo (4 KB)
constexpr uint32_t kTcCols = 256;       // TMEM columns per CTA: 2 blocks x (A_hi 32, A_lo 32, D 32), rounded up

// Build the operator of M step st into its slot: lane j < 16 runs the step's sub-ops on e_j.
// Block variants (bvraw != 0): lanes 16..31 build the operator of block 1 (vectors whose bit 7,
// raw tile offset bvraw, is set) into the next slot.
__device__ __forceinline__ void tc_build_op(const StvSub *__restrict__ subs, int n, const uint8_t *__restrict__ mat,
                                            const StvDTab *__restrict__ tabs, const float2 *__restrict__ tables,
                                            uint64_t full_base, uint32_t tord, uint64_t rank_bits,
                                            const float2 *__restrict__ scal, uint8_t *slot, uint32_t bvraw, int lane) {
    float2 x[1][16];
#pragma unroll
    for (int l = 0; l < 16; ++l) x[0][l] = make_float2(l == (lane & 15) ? 1.f : 0.f, 0.f);
    const uint32_t braw[1] = {lane >= 16 ? bvraw : 0u};
    run_subs<float2, 1>(x, braw, subs, n, mat, tabs, tables, full_base, tord, rank_bits, scal);
    if (lane >= 16 && bvraw) slot += kTcOpBytes;
    if (lane < 16 || bvraw) {
        const int j = lane & 15;   // input amplitude index (column of U)
#pragma unroll
        for (int l = 0; l < 16; ++l) {   // U[l][j] = x[l]
            const float ur = x[0][l].x, ui = x[0][l].y;
            const float v[4] = {ur, -ui, ui, ur};   // (ro, ri) = (0,0) (0,1) (1,0) (1,1)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int ro = q >> 1, ri = q & 1;
                const uint32_t off = tc_bt_off(2 * l + ro, 2 * j + ri);
                // both parts rounded to nearest tf32 (the tensor core truncates: an unrounded
                // lo part would bias every operator towards a norm < 1)
                const uint32_t hi = tf32_rna(v[q]);
                *(uint32_t *)(slot + off) = hi;
                *(uint32_t *)(slot + 4096 + off) = tf32_rna(v[q] - __uint_as_float(hi));
            }
        }
    }
}

template <bool kAcc>
__device__ __forceinline__ void mma_tf32_ts_c(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc) {
    if (kAcc)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d_tmem), "r"(a_tmem),
                     "l"(b_desc), "n"(kTcIdesc)
                     : "memory");
    else
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 0;" ::"r"(d_tmem), "r"(a_tmem),
                     "l"(b_desc), "n"(kTcIdesc)
                     : "memory");
}
// The MMA of one M step for block b (128 rows): 3xTF32, 4 K-slices of 8 each.  desc0 =
// the slot's descriptor; the start-address field (bits 0..13, 16-B units) advances by
// 16 per K-slice (256 B) and by 256 for the lo half (4 KB) -- no carry within a slot.
// Order: the two small cross terms first (A_lo.B_hi, A_hi.B_lo: ~2^-11 of the result),
// the large A_hi.B_hi last.  The accumulator is rounded toward zero each time an
// instruction adds into it (measured: tools/tc_probe.cu drift test), so accumulating the
// small terms first confines the bias to the last 4 additions: a relative norm decay of
// ~3e-7 per operator step instead of ~8e-7.
__device__ __forceinline__ void tc_issue_block(uint32_t tmem, int b, uint64_t desc0) {
    const uint32_t ah = tmem + b * 96, al = ah + 32, d = ah + 64;
    mma_tf32_ts_c<false>(d, al, desc0);
#pragma unroll
    for (int kk = 1; kk < 4; ++kk) mma_tf32_ts_c<true>(d, al + 8 * kk, desc0 + 16 * kk);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts_c<true>(d, ah + 8 * kk, desc0 + 256 + 16 * kk);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts_c<true>(d, ah + 8 * kk, desc0 + 16 * kk);
}

// 1 in exactly one lane of the converged warp (elect.sync): ptxas then issues the guarded
// tensor-core instructions once, from uniform registers
__device__ __forceinline__ bool elect_one() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
    return e != 0;
}

struct alignas(16) TcShared {
    uint64_t bar[2];
    uint64_t tbar[2];   // TMA tile loads, one per ring slot
    uint32_t tmem;
    uint32_t hsync;     // bit o: groups o and o + 1 split the tile into the same two halves
    uint64_t key[STV_TC_MAX_OPS];
    uint64_t cm[48];    // base xor-mask when the permuted ordinal's trailing-ones count is j
    uint32_t tm[48];    // ordinal xor-mask for the same carry
    alignas(16) uint32_t gso[STV_TC_MAX_GROUPS][16];   // per group: swizzled register offsets in bytes
};
constexpr uint32_t kTcShBytes = STV_TC_SH_BYTES;   // TcShared region at the start of shared memory (1024-multiple)
static_assert(sizeof(TcShared) <= kTcShBytes, "TcShared exceeds its region");

// the dynamic shared memory of k_tc_group_pass (same storage as its `smem`)
extern __shared__ __align__(1024) uint8_t tc_smem[];

// One group on the resident tile with tensor-core M steps: thread ctid owns vector ctid.
// FULL: the tile has 256 vectors (S = 12), every thread is live.  gso: the group's 16
// register offsets in bytes (shared memory, staged once per CTA).
template <bool FULL>
__device__ __forceinline__ void tc_group(uint32_t toff, const StvGroup &g, const StvPass *__restrict__ P,
                                         const StvTcStep *__restrict__ steps, int &s0, const uint8_t *__restrict__ mat,
                                         const float2 *__restrict__ tables, uint64_t full_base, uint32_t tord,
                                         const uint8_t *__restrict__ grec, const float2 *__restrict__ scal,
                                         const uint8_t *__restrict__ opsm, TcShared *sh, const uint32_t *gso,
                                         uint32_t vw, uint32_t trow, uint32_t &phase, int ctid, int dbg) {
#ifndef STV_TC_DEBUG
    dbg = 0;   // timing ablations (STV_TILE_DEBUG bits 4..64, profiles/r02_tc_ablation.md) need -DSTV_TC_DEBUG
#endif
    const int nvb = g.nvb;
    const uint32_t nvec = 1u << nvb;
    const bool live = FULL || (uint32_t)ctid < nvec;
    // vw: this vector's word of the group's vector table (loaded one group ahead)
    const uint32_t bsw = vw & 0xffffu, braw = vw >> 16;
    uint32_t so[16];   // byte offsets of the 16 register amplitudes (swizzled)
#pragma unroll
    for (int l = 0; l < 16; l += 4) {
        const uint4 w = *(const uint4 *)&gso[l];
        so[l] = w.x;
        so[l + 1] = w.y;
        so[l + 2] = w.z;
        so[l + 3] = w.w;
    }
    uint32_t bsw_g = bsw, bsw_s = bsw;
    if (g.nflip_g | g.nflip_s) {
        auto flip_delta = [&](int from, int cnt) {
            uint32_t dlt = 0;
            for (int q = 0; q < cnt; ++q) {
                const uint32_t f = g.flip[from + q];
                const uint32_t a = f >> 17;
                const bool on = (f & (1u << 16)) ? ((full_base >> a) & 1) != 0 : (braw & a) != 0;
                if (on) dlt ^= f & 0xffffu;
            }
            return dlt;
        };
        bsw_g ^= flip_delta(0, g.nflip_g);
        bsw_s ^= flip_delta(STV_MAX_FLIPS, g.nflip_s);
    }
    // byte offsets in shared memory: the tile sits at a multiple of its own size, so its offset
    // combines with the in-tile offsets by xor (one LOP3 + LDS per amplitude)
    bsw_g = (bsw_g << 3) ^ toff;
    bsw_s = (bsw_s << 3) ^ toff;
    uint8_t *tb = tc_smem;
    const StvSub *subs = (const StvSub *)((const uint8_t *)P + g.sub_off);
    const StvDTab *tabs = (const StvDTab *)((const uint8_t *)P + P->tab_off);
    const bool pair16 = g.pair16;
    float2 x[1][16];
    if (live && !(dbg & 16)) {
        if (pair16) {
#pragma unroll
            for (int l = 0; l < 16; l += 2) {
                const float4 q = *(const float4 *)(tb + (bsw_g ^ so[l]));
                x[0][l] = make_float2(q.x, q.y);
                x[0][l + 1] = make_float2(q.z, q.w);
            }
        } else {
#pragma unroll
            for (int l = 0; l < 16; ++l) x[0][l] = *(const float2 *)(tb + (bsw_g ^ so[l]));
        }
    } else {
#pragma unroll
        for (int l = 0; l < 16; ++l) x[0][l] = make_float2(0.f, 0.f);
    }
    const uint32_t braw1[1] = {braw};
    // step records (kind, last, first, n | op | bvar), fetched one step ahead
    auto fetch = [&](int i, uint2 &w, int &op, int &bv) {
        w = *(const uint2 *)&steps[i];
        op = steps[i].op;
        bv = steps[i].bvar;
    };
    uint2 nw;
    int nop_, nbv;
    fetch(s0, nw, nop_, nbv);
    for (int s = s0;; ++s) {
        struct { int kind, last, first, n, op, bvar; } st;
        st.kind = (int16_t)(nw.x & 0xffffu);
        st.last = (int16_t)(nw.x >> 16);
        st.first = (int16_t)(nw.y & 0xffffu);
        st.n = (int16_t)(nw.y >> 16);
        st.op = nop_;
        st.bvar = nbv;
        if (!st.last) fetch(s + 1, nw, nop_, nbv);
        if (st.kind == 0) {
            if (!(dbg & 32))
            run_subs<float2, 1>(x, braw1, subs + st.first, st.n, mat, tabs, tables, full_base, tord, P->rank_bits, scal);
        } else {
            {   // A_hi = x itself (the tensor core reads the top 19 bits: tf32 truncation of x),
                // A_lo = x - trunc_tf32(x) (exact in fp32), pre-rounded by half a tf32 ulp so the
                // tensor core's truncation of A_lo rounds to nearest -- truncating both parts
                // would shrink every amplitude (a norm decay of ~1e-6 per operator step)
                // -> TMEM row of this thread, block warp / 4
                uint32_t v[32];
#pragma unroll
                for (int l = 0; l < 16; ++l) {
                    v[2 * l] = __float_as_uint(x[0][l].x);
                    v[2 * l + 1] = __float_as_uint(x[0][l].y);
                }
                if (!(dbg & 64)) tmem_st32(trow, v);
                if (!(dbg & 8))
#pragma unroll
                for (int l = 0; l < 16; ++l) {
                    const float2 t = make_float2(__uint_as_float(v[2 * l] & 0xffffe000u),
                                                 __uint_as_float(v[2 * l + 1] & 0xffffe000u));
                    const float2 lo = __fadd2_rn(x[0][l], make_float2(-t.x, -t.y));
                    v[2 * l] = __float_as_uint(lo.x) + 0x1000u;
                    v[2 * l + 1] = __float_as_uint(lo.y) + 0x1000u;
                }
                if (!(dbg & 64)) tmem_st32(trow + 32, v);
            }
            tc_wait_st();
            tc_fence_before();
            // each half of the CTA (warps 0-3: block 0, warps 4-7: block 1) syncs and issues its own MMAs
            const int half = ctid >> 7;
            asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
            if ((ctid & 127) < 32 && !(dbg & 4)) {   // the half's first warp, converged: one elected lane issues
                tc_fence_after();
                // warp-uniform operands (shfl from lane 0) so ptxas keeps them in uniform registers
                const uint32_t tmh = __shfl_sync(~0u, trow, 0);   // warp 4 half: lane 0, block half
                const uint32_t opa = __shfl_sync(~0u, smem_u32(opsm + (size_t)(st.op + (st.bvar ? half : 0)) * kTcOpBytes), 0);
                if (elect_one()) {
                    tc_issue_block(tmh, 0, umma_desc(opa, 128, 1024));
                    mma_commit(&sh->bar[half]);
                }
                __syncwarp();
            }
            if (!(dbg & 4)) {
                mbar_wait_spin(&sh->bar[half], phase);
                phase ^= 1u;
            }
            tc_fence_after();
            {
                uint32_t v[32];
                if (!(dbg & 64)) tmem_ld32(trow + 64, v);
                tc_wait_ld();
#pragma unroll
                for (int l = 0; l < 16; ++l) x[0][l] = make_float2(__uint_as_float(v[2 * l]), __uint_as_float(v[2 * l + 1]));
            }
        }
        if (st.last) {
            s0 = s + 1;   // the next group's first step
            break;
        }
    }
    if (live && !(dbg & 16)) {
        if (pair16) {
#pragma unroll
            for (int l = 0; l < 16; l += 2)
                *(float4 *)(tb + (bsw_s ^ so[l])) = make_float4(x[0][l].x, x[0][l].y, x[0][l + 1].x, x[0][l + 1].y);
        } else {
#pragma unroll
            for (int l = 0; l < 16; ++l) *(float2 *)(tb + (bsw_s ^ so[l])) = x[0][l];
        }
    }
}

// Tile copy with per-thread offsets precomputed once per CTA: thread t moves the
// 16-B chunks c = t + 256 k (k < kTcChunks) between global (tile base + goff[k])
// and its swizzled shared-memory slot soff[k] = 16 (c ^ H(c >> 3)) (see tile_copy_swz).
constexpr int kTcChunks = 8;   // 2^12 complex64 amplitudes = 2048 chunks over 256 threads
template <bool kLoad, bool FULL>
__device__ __forceinline__ void tc_tile_copy(uint8_t *gtile, uint8_t *stile, const uint64_t (&goff)[kTcChunks],
                                             const uint32_t (&soff)[kTcChunks], int nk) {
    if (kLoad) {
#pragma unroll
        for (int k = 0; k < kTcChunks; ++k) {
            if (!FULL && k >= nk) break;
            cp_async16(stile + soff[k], gtile + goff[k]);
        }
    } else if (FULL) {   // shared-memory reads four at a time ahead of their stores
#pragma unroll
        for (int k0 = 0; k0 < kTcChunks; k0 += 4) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = *(const uint4 *)(stile + soff[k0 + k]);
#pragma unroll
            for (int k = 0; k < 4; ++k) *(uint4 *)(gtile + goff[k0 + k]) = v[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < kTcChunks; ++k) {
            if (k >= nk) break;
            *(uint4 *)(gtile + goff[k]) = *(const uint4 *)(stile + soff[k]);
        }
    }
}

// TMA staging of a pass's tiles (host: launch_tc_group_pass).  One 5-D tensor map views
// the state as (16 contiguous amplitudes) x (tile base: stride 2^L amplitudes, box 1) x
// (the rest of the low run) x (up to 2 runs of consecutive high tile bits); the box is the
// tile in tile-index order, stored with SWIZZLE_128B.  High tile bits beyond the map's
// dims are looped over: load e covers the tile amplitudes whose extra bits equal e.
struct TcTma {
    uint64_t extra_mask;   // physical bits of the looped tile bits
    uint32_t nld;          // loads (= stores) per tile: 2^popcount(extra_mask)
    uint32_t box_bytes;    // bytes per load
    int32_t L;             // tile low bits: base coordinate = (base | extra) >> L
    int32_t bdim;          // tensor dim of the base coordinate (1, or 2 when L > 4)
    int32_t on;            // 1: TMA staging (else cp.async with the same swizzle)
    int32_t pad;
};
__device__ __forceinline__ void tma_load_tile(void *dst, const CUtensorMap *tm, uint32_t c1, uint32_t c2,
                                              uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %2, %2}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_tile(const CUtensorMap *tm, uint32_t c1, uint32_t c2, const void *src) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %1, %1}], [%4];" ::"l"(tm),
                 "r"(0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
}

// Tensor-core group pass: persistent CTAs (2 per SM, 256 threads), tile ordinals in
// the permuted order of StvPass.tperm, a contiguous range per CTA; NS = 2: the next
// tile's load overlaps this tile's work (1: single buffer when shared memory is short).
template <int NS, bool FULL>
__global__ void __launch_bounds__(256, 2)
k_tc_group_pass(float2 *__restrict__ state, const uint8_t *__restrict__ blob, uint32_t pass_off, uint32_t ntiles,
                int dbg_flags, const __grid_constant__ CUtensorMap tmap, const TcTma tma,
                const __grid_constant__ RecParam rec) {
    constexpr int NT = 256;
    extern __shared__ __align__(1024) uint8_t smem[];
    const StvPass *P = (const StvPass *)rec.b;
    const uint8_t *grec = blob + pass_off;
    const int S = P->S, L = P->L, h = P->h;
    const uint64_t out_mask = P->out_mask, rank_bits = P->rank_bits;
    const int nops = P->nops;
    const int ntab = P->ntab;
    const StvGroup *groups = (const StvGroup *)(rec.b + P->ops_off);
    const StvTcStep *steps = (const StvTcStep *)(rec.b + P->tc_off);
    const int ntc = P->ntc, nmop = P->ntcop;
    const uint8_t *mat = rec.b + P->mat_off;
    const uint32_t esz = 8;
    // shared memory: NS tiles | TcShared (kTcShBytes) | operator slots | scalars | tables.
    // The dynamic shared memory starts 1024-aligned (declared; checked below): the tile ring
    // (TMA SWIZZLE_128B pattern = shared address bits 4..6 ^ 7..9) starts at 0, each tile at a
    // multiple of its size, and for full tiles every region sits at a compile-time offset
    const uint32_t tile_elems = FULL ? 4096u : 1u << S;
    float2 *tiles = (float2 *)smem;
    TcShared *sh = (TcShared *)(smem + (size_t)NS * tile_elems * esz);
    uint8_t *opsm = smem + (size_t)NS * tile_elems * esz + kTcShBytes;
    float2 *scal = (float2 *)(opsm + (size_t)nmop * kTcOpBytes);   // 512 B: half-table scalars
    float2 *tables = scal + 64;
    const uint32_t run_bytes = (1u << L) * esz;
    const uint32_t nruns = 1u << h;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t hmask = 0;
    for (int r = 0; r < h; ++r) hmask |= 1ull << P->hpos[r];
    (void)run_bytes;
    (void)nruns;
    // this thread's chunks of a tile: global byte offset from the tile base, shared slot
    const int nchunk = (int)(tile_elems >> 1);
    const int nk = (nchunk - tid + NT - 1) / NT;
    uint64_t goff[kTcChunks];
    uint32_t soff[kTcChunks];
#pragma unroll
    for (int k = 0; k < kTcChunks; ++k) {
        const uint32_t c = (uint32_t)tid + NT * (uint32_t)k;
        const uint32_t i = 2 * c;   // first tile-local amplitude of the chunk
        goff[k] = (pdep64(i >> L, hmask) + (i & ((1u << L) - 1))) * esz;
        soff[k] = 16u * (c ^ (P->swz_tma ? ((c >> 3) & 7u) : swz_hash_d(c >> 3)));
    }
    const int nord = __popcll(out_mask);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem)),
                     "n"(kTcCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        if (smem_u32(smem) & 1023u) __trap();   // the swizzle and the ring offset assume it
        mbar_init(&sh->bar[0], 1);
        mbar_init(&sh->bar[1], 1);
        mbar_init(&sh->tbar[0], 1);
        mbar_init(&sh->tbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < STV_TC_MAX_OPS) sh->key[tid] = ~0ull;
    for (int e = tid; e < nops * 16; e += NT) sh->gso[e >> 4][e & 15] = groups[e >> 4].sw_off[e & 15] << 3;
    if (tid == 64) {
        // Group boundaries that need only a per-half barrier: thread t owns vector t, and its
        // half t >> 7 is vector bit 7.  When groups o and o + 1 map vector bit 7 to the same
        // tile position and no folded X flip moves amplitudes across it, each half of the CTA
        // gathers in group o + 1 exactly the amplitudes it scattered in group o.
        uint32_t m = 0;
        if (FULL && !(dbg_flags & 256))
            for (int o = 0; o + 1 < nops; ++o) {
                const StvGroup &a = groups[o], &b = groups[o + 1];
                const uint32_t s7 = a.vbit[7][1];
                bool ok = a.nvb == 8 && b.nvb == 8 && a.vbit[7][0] == b.vbit[7][0];
                for (int q = 0; q < a.nflip_s && ok; ++q) ok = (a.flip[STV_MAX_FLIPS + q] & 0xffffu) != s7;
                for (int q = 0; q < b.nflip_g && ok; ++q) ok = (b.flip[q] & 0xffffu) != s7;
                if (ok) m |= 1u << o;
            }
        sh->hsync = m;
    }
    if (tid < 48) {   // carry masks of the permuted ordinal: bits 0..tid flip together
        uint64_t cm = 0;
        uint32_t tm = 0;
        for (int i = 0; i <= tid && i < nord; ++i) {
            tm |= 1u << P->tperm[i];
            cm |= pdep64(1ull << P->tperm[i], out_mask);
        }
        sh->cm[tid] = cm;
        sh->tm[tid] = tm;
    }
    if (ntab) build_tables<float2, NT>(P, grec, 0, tables, scal, tid, true);   // static table entries
    bool tile_tabs = false;   // some table has per-tile terms (else nothing to rebuild per tile)
    {
        const StvDTab *tabs = (const StvDTab *)((const uint8_t *)P + P->tab_off);
        for (int t = 0; t < ntab; ++t) tile_tabs |= tabs[t].nterm != 0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t phase = 0;
    const uint32_t hsync = sh->hsync;
    // this thread's TMEM row (lane 32 (warp % 4) + lane, block warp / 4); the CTA's base (warp-uniform)
    const uint32_t tmu = __shfl_sync(~0u, sh->tmem, 0);
    const uint32_t trow = tmu + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 96);
    // the first group's vector-table word (the next group's is loaded while a group runs)
    const uint32_t vw0 = nops ? __ldg((const uint32_t *)(grec + groups[0].vtab_off) + tid) : 0u;
    // the first group's vector-table word (the next group's is loaded while a group runs)

    // contiguous range of permuted ordinals t' for this CTA
    const uint64_t G = gridDim.x;
    const uint32_t t_begin = (uint32_t)(((uint64_t)blockIdx.x * ntiles) / G);
    const uint32_t t_end = (uint32_t)(((uint64_t)(blockIdx.x + 1) * ntiles) / G);
    uint32_t tord = 0;   // t = tperm(t'), advanced by carry masks
    for (int i = 0; i < nord; ++i) tord |= ((t_begin >> i) & 1u) << P->tperm[i];
    uint64_t base = pdep64(tord, out_mask);
    uint64_t lbase = base;   // next tile to load
    uint8_t *gstate = (uint8_t *)state;
    const bool use_tma = tma.on != 0;
    const bool tma_store = tma.on == 2;   // 1: TMA loads, thread stores; 2: TMA loads and stores
    uint32_t tph = 0;   // TMA load barrier phases (bit per slot)
    auto issue = [&](uint32_t tp, int slot) {   // load tile tp (if in range) into ring slot
        uint8_t *stile = (uint8_t *)(tiles + (size_t)slot * tile_elems);
        if (use_tma) {
            // warp 0: lane e issues the loads e, e + 32, ... (and, at the end of the tile, the
            // stores of the same boxes, so its own bulk groups order store-read before reload)
            if (warp == 0 && tp < t_end && !(dbg_flags & 2)) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // this lane's last stores have read
                if (lane == 0) mbar_arrive_expect_tx(&sh->tbar[slot], (uint32_t)(tile_elems * esz));
                __syncwarp();
                for (uint32_t e = lane; e < tma.nld; e += 32) {
                    const uint32_t cb = (uint32_t)((lbase | pdep64(e, tma.extra_mask)) >> tma.L);
                    tma_load_tile(stile + (size_t)e * tma.box_bytes, &tmap, tma.bdim == 1 ? cb : 0u,
                                  tma.bdim == 2 ? cb : 0u, &sh->tbar[slot]);
                }
            }
        } else {
            if (tp < t_end && !(dbg_flags & 2)) tc_tile_copy<true, FULL>(gstate + lbase * esz, stile, goff, soff, nk);
            cp_async_commit();
        }
        if (tp + 1 < t_end) lbase ^= sh->cm[__ffs(~tp) - 1];
    };
    auto wait_tile = [&](int slot) {
        if (dbg_flags & 2) return;
        mbar_wait_spin(&sh->tbar[slot], (tph >> slot) & 1u);
        tph ^= 1u << slot;
    };
    if (NS == 2) issue(t_begin, 0);
    for (uint32_t tp = t_begin; tp < t_end; ++tp) {
        const int slot = NS == 2 ? (int)((tp - t_begin) & 1u) : 0;
        float2 *tile = tiles + (size_t)slot * tile_elems;
        const uint64_t full_base = base | rank_bits;
        if (NS == 1) issue(tp, 0);
        if (tile_tabs && !(dbg_flags & 128)) {   // tables with per-tile terms (bit 7: ablation): rebuilt, then visible to the operator build
            build_tables<float2, NT>(P, grec, full_base, tables, scal, tid, false);
            __syncthreads();
        }
        // operators whose dependency bits changed: one warp per M step
        for (int s = warp; s < ntc; s += NT / 32) {
            const StvTcStep st = steps[s];
            if (st.kind != 1) continue;
            const uint64_t key = full_base & st.dep;
            if (key == sh->key[st.op]) continue;
            const StvGroup &g = groups[st.group];
            const StvSub *subs = (const StvSub *)((const uint8_t *)P + g.sub_off) + st.first;
            tc_build_op(subs, st.n, mat, (const StvDTab *)((const uint8_t *)P + P->tab_off), tables, full_base, tord,
                        rank_bits, scal, opsm + (size_t)st.op * kTcOpBytes, st.bvar ? g.vbit[7][0] : 0u, lane);
            fence_proxy_async();   // this lane's operator stores (generic proxy) -> tensor-core reads
            __syncwarp();
            if (lane == 0) sh->key[st.op] = key;
        }
        if (NS == 2) {
            issue(tp + 1, slot ^ 1);   // the other slot was freed by the previous iteration's last barrier
            if (use_tma) wait_tile(slot);
            else cp_async_wait1();
        } else {
            if (use_tma) wait_tile(0);
            else cp_async_wait0();
        }
        __syncthreads();
        if (!(dbg_flags & 1)) {
            int s0 = 0;
            uint32_t vw = vw0;
            for (int o = 0; o < nops; ++o) {
                const uint32_t w = vw;
                if (o + 1 < nops) vw = __ldg((const uint32_t *)(grec + groups[o + 1].vtab_off) + tid);
                tc_group<FULL>(slot * tile_elems * (uint32_t)esz, groups[o], P, steps, s0, mat, tables, full_base, tord, grec, scal, opsm, sh,
                               sh->gso[o], w, trow, phase, tid, dbg_flags);
                if (FULL && ((hsync >> o) & 1u))   // (never set for the last group: the write-back needs all)
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + (tid >> 7)) : "memory");
                else
                    __syncthreads();
            }
        }
        if (!(dbg_flags & 2)) {
            if (use_tma && tma_store) {
                fence_proxy_async();   // the groups' scatters (generic proxy) -> the TMA store
                __syncthreads();
                if (warp == 0) {
                    for (uint32_t e = lane; e < tma.nld; e += 32) {
                        const uint32_t cb = (uint32_t)((base | pdep64(e, tma.extra_mask)) >> tma.L);
                        tma_store_tile(&tmap, tma.bdim == 1 ? cb : 0u, tma.bdim == 2 ? cb : 0u,
                                       (const uint8_t *)tile + (size_t)e * tma.box_bytes);
                    }
                    bulk_commit();
                }
            } else {
                // write-back by all threads (16-B LDS + STG): the slot is free at the next barrier
                // without waiting for a bulk store to drain it before its reload
                tc_tile_copy<false, FULL>(gstate + base * esz, (uint8_t *)tile, goff, soff, nk);
            }
        }
        if (tp + 1 < t_end) {
            const int j = __ffs(~tp) - 1;
            base ^= sh->cm[j];
            tord ^= sh->tm[j];
        }
        __syncthreads();   // write-back reads of this slot done before it is reloaded
    }
    cp_async_wait0();
    if (use_tma && warp == 0) bulk_wait_all();   // the last stores have completed
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sh->tmem), "n"(kTcCols) : "memory");
    }
}
