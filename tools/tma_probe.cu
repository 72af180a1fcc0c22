// tma_probe.cu -- can one TMA tensor map address every tile of a pass?  The state is viewed
// as a 5-D tensor whose dims are the tile's bit runs plus a "base" dim (stride 2^L * 8 B,
// coordinate = tile base / 2^L) that overlaps the others; the box is the tile.  Loads one
// tile with SWIZZLE_128B and checks every amplitude against its expected swizzled slot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_load(const __grid_constant__ CUtensorMap tmap, int c1, int nelem, uint64_t *out, int store_back) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nelem * 8));
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(smem_u32(sm)), "l"(&tmap), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(0), "r"(smem_u32(&bar))
            : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    for (int i = threadIdx.x; i < nelem; i += blockDim.x) out[i] = ((const uint64_t *)sm)[i];
    if (store_back) {   // write the tile back, doubled, through the same map
        __syncthreads();
        for (int i = threadIdx.x; i < nelem; i += blockDim.x) ((uint64_t *)sm)[i] *= 2;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(&tmap), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(0), "r"(smem_u32(sm)) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    }
}

int main() {
    // state of 2^n uint64 "amplitudes" a[i] = i; tile: L = 4 low bits + high bits {12..19}
    // (run 1) and {22, 23} (run 2); base = the remaining bits
    const int n = 26, L = 4;
    const uint64_t N = 1ull << n;
    uint64_t *d;
    CK(cudaMalloc(&d, N * 8));
    std::vector<uint64_t> h(N);
    for (uint64_t i = 0; i < N; ++i) h[i] = i;
    CK(cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    // dims: d0 = 16 (low run), d1 = base (stride 2^L * 8 B), d2 = run {12..19}, d3 = run {22,23}, d4 = 1
    cuuint64_t gdim[5] = {16, N >> L, 256, 4, 1};
    cuuint64_t gstr[4] = {(cuuint64_t)8 << L, (cuuint64_t)8 << 12, (cuuint64_t)8 << 22, (cuuint64_t)8 << n};
    cuuint32_t box[5] = {16, 1, 256, 4, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUtensorMap tm;
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode (overlapping base dim) -> %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    const int nelem = 16 * 256 * 4;
    uint64_t *dout;
    CK(cudaMalloc(&dout, nelem * 8));
    // tile base: outside bits 4..11, 20, 21, 24, 25 -> pick base = bits 5, 9, 20, 25
    const uint64_t base = (1ull << 5) | (1ull << 9) | (1ull << 20) | (1ull << 25);
    CK(cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, nelem * 8));
    k_load<<<1, 256, nelem * 8>>>(tm, (int)(base >> L), nelem, dout, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint64_t> o(nelem);
    CK(cudaMemcpy(o.data(), dout, nelem * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int t = 0; t < nelem; ++t) {   // tile index t -> physical index; smem slot = swizzle(t)
        const uint64_t phys = base | (uint64_t)(t & 15) | ((uint64_t)((t >> 4) & 255) << 12) | ((uint64_t)(t >> 12) << 22);
        const uint32_t c = (uint32_t)t >> 1, slot = ((c ^ ((c >> 3) & 7)) << 1) | (t & 1);
        if (o[slot] != phys) { if (bad < 5) printf("t=%d slot=%u got %llu want %llu\n", t, slot, (unsigned long long)o[slot], (unsigned long long)phys); ++bad; }
    }
    CK(cudaMemcpy(h.data(), d, N * 8, cudaMemcpyDeviceToHost));
    int bad2 = 0;
    for (uint64_t i = 0; i < N; ++i) {
        const bool in = (i & ~(uint64_t)(15 | (255u << 12) | (3u << 22))) == base;
        if (h[i] != (in ? 2 * i : i)) ++bad2;
    }
    printf("load mismatches %d of %d; store-back mismatches %d\n", bad, nelem, bad2);
    return bad || bad2;
}
