// tc_probe.cu -- standalone check of the tcgen05 building blocks the tensor-core
// group pass relies on (kind::tf32, A from TMEM, B K-major in shared memory,
// SWIZZLE_NONE canonical layout, 3xTF32 split, 32x32b TMEM loads/stores).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_probe tools/tc_probe.cu
//   ./tc_probe            -> max |D - A.B| for 256 rows x 32 x 32, and MMA throughput
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// 32 lanes x 32 columns of 32 bit: thread i <-> TMEM lane (base + i), registers <-> columns
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]),
        "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
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

// D[tmem] (+)= A[tmem] . B[smem desc], kind::tf32, cta_group::1
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// SWIZZLE_NONE K-major canonical descriptor: core matrix 8 rows x 16 B; lbo = K-adjacent
// core-matrix stride, sbo = 8-row-group stride (bytes)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= 1ull << 46;   // version 1 (sm_100)
    return d;          // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// idesc: D f32, A/B tf32, K-major both, N = 32, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

// Bt byte offset of (n, k) in the canonical layout: lbo = 128 B, sbo = 1024 B
__host__ __device__ inline uint32_t bt_off(int n, int k) {
    return (uint32_t)((n & 7) * 16 + (k & 3) * 4 + (k >> 2) * 128 + (n >> 3) * 1024);
}

// A: 256 x 32 (rows = 2 blocks of 128), Bt: 32 x 32 (n, k); D = A . B (B[k][n] = Bt[n][k])
__global__ void __launch_bounds__(256, 1) k_probe(const float *A, const float *Bt, float *D, int reps, int split) {
    __shared__ __align__(1024) uint8_t bsm[2 * 4096];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                     "r"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B hi / lo into the canonical layout
    for (int e = tid; e < 1024; e += 256) {
        const int n = e >> 5, k = e & 31;
        const float b = Bt[e];
        const uint32_t hi = split ? tf32_rna(b) : __float_as_uint(b);
        const float lo = b - __uint_as_float(hi);
        *(uint32_t *)(bsm + bt_off(n, k)) = hi;
        *(float *)(bsm + 4096 + bt_off(n, k)) = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const int blk = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t colA = blk * 96, colAl = colA + 32, colD = colA + 64;
    // A row -> hi / lo in TMEM
    {
        uint32_t h[32], l[32];
        for (int k = 0; k < 32; ++k) {
            const float a = A[tid * 32 + k];
            h[k] = split ? tf32_rna(a) : __float_as_uint(a);
            l[k] = __float_as_uint(a - __uint_as_float(h[k]));
        }
        tmem_st32(tmem + lane_base + colA, h);
        tmem_st32(tmem + lane_base + colAl, l);
        tc_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (tid == 0) {
            tc_fence_after();
            const uint32_t bh = smem_u32(bsm), bl = smem_u32(bsm + 4096);
            for (int b = 0; b < 2; ++b) {
                const uint32_t ah = tmem + b * 96, al = ah + 32, d = ah + 64;
                for (int kk = 0; kk < 4; ++kk)
                    mma_tf32_ts(d, ah + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, kk > 0);
                if (split) {
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, ah + 8 * kk, smem_desc(bl + 256 * kk, 128, 1024), kIdesc, 1);
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, al + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, 1);
                }
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
    }
    long long t1 = clock64();
    uint32_t dv[32];
    tmem_ld32(tmem + lane_base + colD, dv);
    tc_wait_ld();
    for (int n = 0; n < 32; ++n) D[tid * 32 + n] = __uint_as_float(dv[n]);
    if (tid == 0 && reps > 1) printf("reps %d: %.1f cycles per 24-MMA round (block 0 issuer view)\n", reps, (double)(t1 - t0) / reps);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}


// drift probe: rows of A are complex 16-vectors (32 reals); B = real embedding of a unitary U
// (given as Bt[n][k]); the row is mapped through U `reps` times with the 3xTF32 step
// (A_hi = x, A_lo = x - trunc(x) [+ rounding variant], D = hi.Bh + hi.Bl + lo.Bh) and the
// norms before / after are written out.  lo_mode: 0 truncated lo, 1 lo + 0x1000, 2 cvt.rna(lo).
// b_lo_rna: B_lo rounded to nearest tf32 (else exact fp32 remainder, truncated by the MMA).
__global__ void __launch_bounds__(256, 1) k_drift(const float *A, const float *Bt, float *norms, int reps, int lo_mode,
                                                  int b_lo_rna) {
    __shared__ __align__(1024) uint8_t bsm[2 * 4096];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    for (int e = tid; e < 1024; e += 256) {
        const int n = e >> 5, k = e & 31;
        const float b = Bt[e];
        const uint32_t hi = tf32_rna(b);
        const float lo = b - __uint_as_float(hi);
        *(uint32_t *)(bsm + bt_off(n, k)) = hi;
        *(uint32_t *)(bsm + 4096 + bt_off(n, k)) = b_lo_rna ? tf32_rna(lo) : __float_as_uint(lo);   // 2: also reordered
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const int blk = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t colA = blk * 96, colAl = colA + 32, colD = colA + 64;
    float x[32];
    double n0 = 0;
    for (int k = 0; k < 32; ++k) { x[k] = A[tid * 32 + k]; n0 += (double)x[k] * x[k]; }
    uint32_t phase = 0;
    for (int r = 0; r < reps; ++r) {
        uint32_t h[32], l[32];
        for (int k = 0; k < 32; ++k) {
            h[k] = __float_as_uint(x[k]);
            const float lo = x[k] - __uint_as_float(h[k] & 0xffffe000u);
            l[k] = lo_mode == 0 ? __float_as_uint(lo) : lo_mode == 1 ? __float_as_uint(lo) + 0x1000u : tf32_rna(lo);
        }
        tmem_st32(tmem + lane_base + colA, h);
        tmem_st32(tmem + lane_base + colAl, l);
        tc_wait_st();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t bh = smem_u32(bsm), bl = smem_u32(bsm + 4096);
            for (int b = 0; b < 2; ++b) {
                const uint32_t ah = tmem + b * 96, al = ah + 32, d = ah + 64;
                if (b_lo_rna >= 2) {   // small cross terms first, hi.hi last
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, al + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, kk > 0);
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, ah + 8 * kk, smem_desc(bl + 256 * kk, 128, 1024), kIdesc, 1);
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, ah + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, 1);
                } else {
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, ah + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, kk > 0);
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, ah + 8 * kk, smem_desc(bl + 256 * kk, 128, 1024), kIdesc, 1);
                    for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(d, al + 8 * kk, smem_desc(bh + 256 * kk, 128, 1024), kIdesc, 1);
                }
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        uint32_t dv[32];
        tmem_ld32(tmem + lane_base + colD, dv);
        tc_wait_ld();
        for (int k = 0; k < 32; ++k) x[k] = __uint_as_float(dv[k]);
        tc_fence_before();
        __syncthreads();
    }
    double n1 = 0;
    for (int k = 0; k < 32; ++k) n1 += (double)x[k] * x[k];
    norms[2 * tid] = (float)n0;
    norms[2 * tid + 1] = (float)(n1 / n0 - 1.0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

static void drift_test(int reps) {
    // random 16x16 unitary by Gram-Schmidt, its 32x32 real embedding as Bt[n][k]
    srand(7);
    double ur[16][16], ui[16][16];
    auto g = []() { double s = 0; for (int i = 0; i < 12; ++i) s += (double)rand() / RAND_MAX; return s - 6; };
    for (int c = 0; c < 16; ++c) {
        for (int r = 0; r < 16; ++r) { ur[r][c] = g(); ui[r][c] = g(); }
        for (int p = 0; p < c; ++p) {   // remove projection on column p
            double dr = 0, di = 0;
            for (int r = 0; r < 16; ++r) { dr += ur[r][p] * ur[r][c] + ui[r][p] * ui[r][c]; di += ur[r][p] * ui[r][c] - ui[r][p] * ur[r][c]; }
            for (int r = 0; r < 16; ++r) { ur[r][c] -= dr * ur[r][p] - di * ui[r][p]; ui[r][c] -= dr * ui[r][p] + di * ur[r][p]; }
        }
        double nn = 0;
        for (int r = 0; r < 16; ++r) nn += ur[r][c] * ur[r][c] + ui[r][c] * ui[r][c];
        nn = sqrt(nn);
        for (int r = 0; r < 16; ++r) { ur[r][c] /= nn; ui[r][c] /= nn; }
    }
    std::vector<float> Bt(1024), A(256 * 32), out(512);
    for (int lp = 0; lp < 16; ++lp)
        for (int l = 0; l < 16; ++l) {   // out[l'] = sum_l U[l'][l] in[l]: Bt[2l'+ro][2l+ri]
            Bt[(2 * lp) * 32 + 2 * l] = (float)ur[lp][l];
            Bt[(2 * lp) * 32 + 2 * l + 1] = (float)-ui[lp][l];
            Bt[(2 * lp + 1) * 32 + 2 * l] = (float)ui[lp][l];
            Bt[(2 * lp + 1) * 32 + 2 * l + 1] = (float)ur[lp][l];
        }
    for (auto &v : A) v = (float)(g() * 1e-3);
    float *dA, *dB, *dN;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, Bt.size() * 4)); CK(cudaMalloc(&dN, 512 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice));
    for (int bl = 0; bl < 3; ++bl)
        for (int lm = 0; lm < 3; ++lm) {
            k_drift<<<1, 256>>>(dA, dB, dN, reps, lm, bl);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(out.data(), dN, 512 * 4, cudaMemcpyDeviceToHost));
            double m = 0;
            for (int t = 0; t < 256; ++t) m += out[2 * t + 1];
            printf("drift reps=%d b_lo_rna=%d lo_mode=%d: mean relative norm change %.3e (per step %.3e)\n", reps, bl, lm,
                   m / 256, m / 256 / reps);
        }
}

int main(int argc, char **argv) {
    if (argc > 1) { drift_test(atoi(argv[1])); return 0; }
    const int R = 256, K = 32, N = 32;
    std::vector<float> A(R * K), Bt(N * K), D(R * N);
    srand(1);
    auto rnd = []() { return (float)rand() / RAND_MAX * 2.0f - 1.0f; };
    for (auto &x : A) x = rnd();
    for (auto &x : Bt) x = rnd();
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, Bt.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice));
    for (int split = 0; split < 2; ++split) {
        CK(cudaMemset(dD, 0, D.size() * 4));
        k_probe<<<1, 256>>>(dA, dB, dD, 1, split);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double worst = 0, worst_rel = 0;
        for (int r = 0; r < R; ++r)
            for (int n = 0; n < N; ++n) {
                double s = 0, sa = 0;
                for (int k = 0; k < K; ++k) {
                    s += (double)A[r * K + k] * (double)Bt[n * K + k];
                    sa += fabs((double)A[r * K + k] * (double)Bt[n * K + k]);
                }
                worst = fmax(worst, fabs(s - D[r * N + n]));
                worst_rel = fmax(worst_rel, fabs(s - D[r * N + n]) / sa);
            }
        printf("split=%d max|D-AB| = %.3e  max rel (to sum|ab|) = %.3e  D[0]=%f\n", split, worst, worst_rel, D[0]);
    }
    k_probe<<<1, 256>>>(dA, dB, dD, 2000, 1);
    CK(cudaDeviceSynchronize());
    // chip-wide throughput: 148 x 2 CTAs
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 4000;
    k_probe<<<296, 256>>>(dA, dB, dD, 10, 1);
    cudaEventRecord(e0);
    k_probe<<<296, 256>>>(dA, dB, dD, reps, 1);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 296.0 * reps * 2 * 3 * 2.0 * 128 * 32 * 32;
    printf("296 CTAs x %d rounds: %.3f ms -> %.1f TFLOP/s (tf32, 3 products counted)\n", reps, ms, flops / ms / 1e9);
    return 0;
}
