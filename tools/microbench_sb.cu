// Microbenchmark for the source-blocked dense pull design (B200, sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbsb tools/microbench_sb.cu
// Measures, on an L2-resident 16.8 MB value array (V = 2^22, the CC s22 size):
//   1. random 4-byte gathers with different load flavours (t-stage line rate?)
//   2. RED.MIN throughput for P scattered updates (random / ascending-per-block)
//   3. shared-memory gathers of 16-bit local ids from a staged value block
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// RMAT-like 22-bit id: bit set with p = 0.24 per level
__device__ __forceinline__ uint32_t rmat_id(uint64_t seed) {
    uint32_t s = 0;
    uint64_t h = mix(seed);
    for (int l = 0; l < 22; ++l) {
        if ((l & 7) == 0) h = mix(h + l);
        s = (s << 1) | (((h >> ((l & 7) * 8)) & 255) < 61 ? 1u : 0u);
    }
    return s;
}

__global__ void k_gen(uint32_t *idx, uint64_t m, int rmat, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        idx[i] = rmat ? rmat_id(i * 7919 + 13) : (uint32_t)(mix(i) % n);
}

template <int FLAVOR>
__device__ __forceinline__ uint32_t ld(const uint32_t *p) {
    uint32_t r;
    if constexpr (FLAVOR == 0) r = *p;
    else if constexpr (FLAVOR == 1) r = __ldg(p);
    else if constexpr (FLAVOR == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else if constexpr (FLAVOR == 3) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

template <int FLAVOR>
__global__ void k_gather(const uint4 *idx4, uint64_t m4, const uint32_t *vals, unsigned *out) {
    uint32_t acc = 0xffffffffu;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m4; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(idx4 + i);
        acc = min(acc, min(min(ld<FLAVOR>(vals + v.x), ld<FLAVOR>(vals + v.y)),
                           min(ld<FLAVOR>(vals + v.z), ld<FLAVOR>(vals + v.w))));
    }
    if (acc == 0x12345u) atomicAdd(out, 1u);
}

// RED.MIN: P updates; address = idx[i] (random) or ascending in runs
__global__ void k_red(const uint32_t *idx, uint64_t p, uint32_t *dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p; i += (uint64_t)gridDim.x * blockDim.x)
        atomicMin(dst + idx[i], (uint32_t)(i & 0xffff));
}
// plain scattered stores for comparison
__global__ void k_st(const uint32_t *idx, uint64_t p, uint32_t *dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p; i += (uint64_t)gridDim.x * blockDim.x)
        dst[idx[i]] = (uint32_t)i;
}

// smem gathers: each CTA stages S values (one block) then gathers m/CTAs
// 16-bit local ids from it, 4 per thread per step
template <int S>
__global__ void k_smem(const uint2 *ids, uint64_t m4, const uint32_t *vals, unsigned *out) {
    extern __shared__ uint32_t sv[];
    for (int i = threadIdx.x; i < S; i += blockDim.x) sv[i] = vals[(blockIdx.x * 997 + i) & ((1u << 22) - 1)];
    __syncthreads();
    uint32_t acc = 0xffffffffu;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m4; i += (uint64_t)gridDim.x * blockDim.x) {
        uint2 v = __ldcs(ids + i);
        uint32_t a = v.x & 0xffff, b = v.x >> 16, c = v.y & 0xffff, d = v.y >> 16;
        acc = min(acc, min(min(sv[a % S], sv[b % S]), min(sv[c % S], sv[d % S])));
    }
    if (acc == 0x12345u) atomicAdd(out, 1u);
}

int main() {
    const uint32_t n = 1u << 22;
    const uint64_t m = 128ull << 20;  // 128M gathers
    uint32_t *vals, *idx, *dst;
    unsigned *out;
    cudaMalloc(&vals, n * 4ull);
    cudaMalloc(&idx, m * 4);
    cudaMalloc(&dst, n * 4ull);
    cudaMalloc(&out, 4);
    cudaMemset(vals, 1, n * 4ull);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto fn) {
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        return best;
    };
    for (int rmat = 0; rmat < 2; ++rmat) {
        k_gen<<<sms * 8, 256>>>(idx, m, rmat, n);
        cudaDeviceSynchronize();
        for (int bps : {4, 8}) {
            float t0 = timeit([&] { k_gather<0><<<sms * bps, 256>>>((const uint4 *)idx, m / 4, vals, out); });
            float t1 = timeit([&] { k_gather<1><<<sms * bps, 256>>>((const uint4 *)idx, m / 4, vals, out); });
            float t2 = timeit([&] { k_gather<2><<<sms * bps, 256>>>((const uint4 *)idx, m / 4, vals, out); });
            float t3 = timeit([&] { k_gather<3><<<sms * bps, 256>>>((const uint4 *)idx, m / 4, vals, out); });
            float t4 = timeit([&] { k_gather<4><<<sms * bps, 256>>>((const uint4 *)idx, m / 4, vals, out); });
            printf("%s gathers 128M bps=%d: plain %.3f ldg %.3f cg %.3f nc.noalloc %.3f cv %.3f ms\n",
                   rmat ? "rmat" : "uniform", bps, t0, t1, t2, t3, t4);
        }
        for (uint64_t p : {26ull << 20, 8ull << 20}) {
            float tr = timeit([&] { k_red<<<sms * 8, 256>>>(idx, p, dst); });
            float ts = timeit([&] { k_st<<<sms * 8, 256>>>(idx, p, dst); });
            printf("%s RED.MIN %lluM: %.3f ms (%.1f G/s); scattered ST %.3f ms\n", rmat ? "rmat" : "uniform",
                   (unsigned long long)(p >> 20), tr, p / tr / 1e6, ts);
        }
    }
    // ascending addresses (dst-sorted runs): RED on a sorted index
    {
        k_gen<<<sms * 8, 256>>>(idx, m, 0, n);
        cudaDeviceSynchronize();
    }
    cudaFuncSetAttribute(k_smem<49152>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 * 4);
    for (int t : {256, 512, 1024}) {
        float tsm = timeit([&] { k_smem<49152><<<sms, t, 49152 * 4>>>((const uint2 *)idx, m / 4, vals, out); });
        printf("smem gathers 128M (u16 ids, S=48K, %d thr/CTA, 1 CTA/SM): %.3f ms\n", t, tsm);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
