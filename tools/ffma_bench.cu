// FP32 issue-rate microbenchmark for the group-op inner loop shape (sm_100a).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma_bench tools/ffma_bench.cu
// Each kernel runs a fixed number of complex 4x4 mat-vecs (U2 on a 16-amplitude
// register vector) per thread and reports FFMA-equivalent TFLOP/s.
//   u2_smem   : matrix entries loaded from shared memory each sub-op (the current kernel)
//   u2_const  : matrix entries in __constant__ memory at a uniform dynamic index
//   u2_param  : matrix entries in a kernel-parameter struct (constant bank 0, static offsets)
//   ffma_reg  : 8 independent 3-register FFMA chains (x = x * y + z)
//   ffma_imm  : 8 independent FFMA chains with an immediate operand
#include <cstdio>
#include <cuda_runtime.h>

struct __align__(16) Mat4 { float2 m[16]; };
struct __align__(16) Mats { Mat4 u[8]; };
__constant__ Mat4 cmats[8];

__device__ __forceinline__ float2 cfma(float2 m, float2 x, float2 acc) {
    acc.x = fmaf(m.x, x.x, acc.x);
    acc.x = fmaf(-m.y, x.y, acc.x);
    acc.y = fmaf(m.x, x.y, acc.y);
    acc.y = fmaf(m.y, x.x, acc.y);
    return acc;
}

template <int A, int B, class MP>
__device__ __forceinline__ void g_u2(float2 (&x)[16], MP M) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        float2 v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        float2 o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            float2 acc = make_float2(0.f, 0.f);
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

__global__ void u2_smem(float2 *out, const Mat4 *g, int iters) {
    __shared__ Mat4 sm[8];
    if (threadIdx.x < 8 * 16) ((float2 *)sm)[threadIdx.x] = ((const float2 *)g)[threadIdx.x];
    __syncthreads();
    float2 x[16];
    for (int l = 0; l < 16; ++l) x[l] = make_float2(threadIdx.x * 1e-3f + l, l * 0.5f);
    for (int it = 0; it < iters; ++it) {
        const float2 *M0 = sm[it & 7].m, *M1 = sm[(it + 1) & 7].m;
        g_u2<0, 1>(x, M0);
        g_u2<2, 3>(x, M1);
        g_u2<0, 2>(x, M0);
        g_u2<1, 3>(x, M1);
    }
    float2 s = make_float2(0, 0);
    for (int l = 0; l < 16; ++l) { s.x += x[l].x; s.y += x[l].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ float2 cmac2(float mr, float2 mp, float2 x, float2 acc) {
    acc = __ffma2_rn(make_float2(mr, mr), x, acc);
    return __ffma2_rn(mp, make_float2(x.y, x.x), acc);
}
__device__ __forceinline__ float2 cmul1(float mr, float2 mp, float2 x) {
    return __ffma2_rn(mp, make_float2(x.y, x.x), __fmul2_rn(make_float2(mr, mr), x));
}
template <int A, int B>
__device__ __forceinline__ void g_u2p(float2 (&x)[16], const float (&mr)[16], const float2 (&mp)[16]) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        const float2 v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        float2 o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            float2 acc = cmul1(mr[r * 4], mp[r * 4], v[0]);
#pragma unroll
            for (int c = 1; c < 4; ++c) acc = cmac2(mr[r * 4 + c], mp[r * 4 + c], v[c], acc);
            o[r] = acc;
        }
        x[l] = o[0];
        x[l | (1 << A)] = o[1];
        x[l | (1 << B)] = o[2];
        x[l | (1 << A) | (1 << B)] = o[3];
    }
}
// packed FFMA2 U2 on NV register vectors, matrices from shared memory
template <int NV>
__global__ void u2p_smem(float2 *out, const float *g, int iters) {
    __shared__ float sm[8 * 48];
    for (int i = threadIdx.x; i < 8 * 48; i += blockDim.x) sm[i] = g[i % 64] * 0.1f;
    __syncthreads();
    float2 x[NV][16];
    for (int i = 0; i < NV; ++i)
        for (int l = 0; l < 16; ++l) x[i][l] = make_float2(threadIdx.x * 1e-3f + l + i, l * 0.5f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const float *M = sm + ((it + s) & 7) * 48;
            float mr[16];
            float2 mp[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) { mr[e] = M[e]; mp[e] = ((const float2 *)(M + 16))[e]; }
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                if (s == 0) g_u2p<0, 1>(x[i], mr, mp);
                if (s == 1) g_u2p<2, 3>(x[i], mr, mp);
                if (s == 2) g_u2p<0, 2>(x[i], mr, mp);
                if (s == 3) g_u2p<1, 3>(x[i], mr, mp);
            }
        }
    }
    float2 s = make_float2(0, 0);
    for (int i = 0; i < NV; ++i)
        for (int l = 0; l < 16; ++l) { s.x += x[i][l].x; s.y += x[i][l].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


__device__ __forceinline__ float2 cmacN(float2 m, float2 x, float2 acc) {
    acc = __ffma2_rn(x, make_float2(m.x, m.x), acc);
    return __ffma2_rn(make_float2(-x.y, x.x), make_float2(m.y, m.y), acc);
}
__device__ __forceinline__ float2 cmulN(float2 m, float2 x) {
    return __ffma2_rn(make_float2(-x.y, x.x), make_float2(m.y, m.y), __fmul2_rn(x, make_float2(m.x, m.x)));
}
template <int A, int B, bool SPLIT>
__device__ __forceinline__ void g_u2n(float2 (&x)[16], const float2 (&m)[16]) {
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        if (l & ((1 << A) | (1 << B))) continue;
        const float2 v[4] = {x[l], x[l | (1 << A)], x[l | (1 << B)], x[l | (1 << A) | (1 << B)]};
        float2 o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (SPLIT) {
                float2 a0 = cmulN(m[r * 4], v[0]), a1 = cmulN(m[r * 4 + 1], v[1]);
                a0 = cmacN(m[r * 4 + 2], v[2], a0);
                a1 = cmacN(m[r * 4 + 3], v[3], a1);
                o[r] = make_float2(a0.x + a1.x, a0.y + a1.y);
            } else {
                float2 acc = cmulN(m[r * 4], v[0]);
#pragma unroll
                for (int c = 1; c < 4; ++c) acc = cmacN(m[r * 4 + c], v[c], acc);
                o[r] = acc;
            }
        }
        x[l] = o[0]; x[l | (1 << A)] = o[1]; x[l | (1 << B)] = o[2]; x[l | (1 << A) | (1 << B)] = o[3];
    }
}
struct __align__(16) MatsN { float2 u[8][16]; };
template <bool SPLIT>
__global__ void u2n_param(float2 *out, const __grid_constant__ MatsN P, int iters) {
    float2 x[16];
    for (int l = 0; l < 16; ++l) x[l] = make_float2(threadIdx.x * 1e-3f + l, l * 0.5f);
    for (int it = 0; it < iters; ++it) {
        const int k = it & 3;
        float2 m0[16], m1[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) { m0[e] = P.u[k][e]; m1[e] = P.u[k + 4][e]; }
        g_u2n<0, 1, SPLIT>(x, m0);
        g_u2n<2, 3, SPLIT>(x, m1);
        g_u2n<0, 2, SPLIT>(x, m0);
        g_u2n<1, 3, SPLIT>(x, m1);
    }
    float2 s = make_float2(0, 0);
    for (int l = 0; l < 16; ++l) { s.x += x[l].x; s.y += x[l].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void u2_const(float2 *out, int iters) {
    float2 x[16];
    for (int l = 0; l < 16; ++l) x[l] = make_float2(threadIdx.x * 1e-3f + l, l * 0.5f);
    for (int it = 0; it < iters; ++it) {
        const float2 *M0 = cmats[it & 7].m, *M1 = cmats[(it + 1) & 7].m;
        g_u2<0, 1>(x, M0);
        g_u2<2, 3>(x, M1);
        g_u2<0, 2>(x, M0);
        g_u2<1, 3>(x, M1);
    }
    float2 s = make_float2(0, 0);
    for (int l = 0; l < 16; ++l) { s.x += x[l].x; s.y += x[l].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void u2_param(float2 *out, const __grid_constant__ Mats P, int iters) {
    float2 x[16];
    for (int l = 0; l < 16; ++l) x[l] = make_float2(threadIdx.x * 1e-3f + l, l * 0.5f);
    for (int it = 0; it < iters; ++it) {
        g_u2<0, 1>(x, P.u[0].m);
        g_u2<2, 3>(x, P.u[1].m);
        g_u2<0, 2>(x, P.u[2].m);
        g_u2<1, 3>(x, P.u[3].m);
    }
    float2 s = make_float2(0, 0);
    for (int l = 0; l < 16; ++l) { s.x += x[l].x; s.y += x[l].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_reg(float *out, float y, float z, int iters) {
    float a[8];
    float b = y + threadIdx.x, c = z - threadIdx.x;
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters * 64; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
        b = __int_as_float(__float_as_int(b) ^ (it & 1));
    }
    float s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_imm(float *out, int iters) {
    float a[8];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters * 64; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], 0.999f, 1.0e-3f);
    }
    float s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    Mat4 h[8];
    for (int u = 0; u < 8; ++u)
        for (int i = 0; i < 16; ++i) h[u].m[i] = make_float2(0.25f * ((i * 7 + u) % 5 - 2) * 0.3f, 0.1f * (i % 3));
    Mats P;
    for (int u = 0; u < 8; ++u) P.u[u] = h[u];
    cudaMemcpyToSymbol(cmats, h, sizeof(h));
    Mat4 *dg;
    cudaMalloc(&dg, sizeof(h));
    cudaMemcpy(dg, h, sizeof(h), cudaMemcpyHostToDevice);
    float2 *out;
    cudaMalloc(&out, 64 << 20);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256}) {
        for (int ctas_per_sm : {1, 2, 3}) {
            const int grid = sms * ctas_per_sm;
            if (threads * ctas_per_sm > 2048) continue;
            // U2: 4 sub-ops x 4 quads x 16 cfma x 4 FFMA = 1024 FFMA per iteration per thread
            const double u2_flops = 2.0 * 1024 * iters * (double)grid * threads;
            const double ffma_flops = 2.0 * 8 * 64 * iters * (double)grid * threads;
            MatsN PN;
            for (int u = 0; u < 8; ++u) for (int e = 0; e < 16; ++e) PN.u[u][e] = make_float2(0.1f * ((e * 7 + u) % 5 - 2), 0.05f * (e % 3));
            for (int k = 0; k < 9; ++k) {
                float ms = 0;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(e0);
                    if (k == 0) u2_smem<<<grid, threads>>>(out, dg, iters);
                    if (k == 1) u2_const<<<grid, threads>>>(out, iters);
                    if (k == 2) u2_param<<<grid, threads>>>(out, P, iters);
                    if (k == 3) ffma_reg<<<grid, threads>>>((float *)out, 1.0001f, 1e-4f, iters);
                    if (k == 4) ffma_imm<<<grid, threads>>>((float *)out, iters);
                    if (k == 5) u2p_smem<1><<<grid, threads>>>(out, (const float *)dg, iters);
                    if (k == 6) u2p_smem<2><<<grid, threads>>>(out, (const float *)dg, iters);
                    if (k == 7) u2n_param<false><<<grid, threads>>>(out, PN, iters);
                    if (k == 8) u2n_param<true><<<grid, threads>>>(out, PN, iters);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms, e0, e1);
                }
                const char *nm[] = {"u2_smem", "u2_const", "u2_param", "ffma_reg", "ffma_imm", "u2p_nv1", "u2p_nv2",
                                    "u2n_ur", "u2n_ur_split"};
                const double fl = k < 3 ? u2_flops : k == 5 ? u2_flops : k == 6 ? 2 * u2_flops : k >= 7 ? u2_flops : ffma_flops;
                printf("%-9s threads=%d ctas/sm=%d  %.3f ms  %.1f TFLOP/s  (peak@%d MHz = %.1f)\n", nm[k], threads,
                       ctas_per_sm, ms, fl / ms / 1e9, clk / 1000, sms * 128 * 2.0 * clk * 1e3 / 1e12);
            }
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(err));
    return 0;
}
