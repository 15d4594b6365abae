// Microbenchmark: how many random 4-byte gathers per second one B200 serves,
// by table size and by how many lanes of a warp share a 32-byte sector.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbsector tools/microbench_sector.cu
// Every pull kernel of this repo performs one such gather per edge
// (prev[src] / contrib[src]).  The result is the roofline those kernels sit
// under: an SM's L1 sends about one sector request per cycle to the crossbar
// (ncu: l1tex__m_l1tex2xbar_req_cycles_active), so misses cap out near
// 148 SMs x 1.965 GHz = 290 G gathers/s however small the table is, i.e.
// 1.16 TB/s of useful 4-byte values = 0.18 of the 6.5 TB/s copy bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return (uint32_t)x;
}

// Each thread performs `per` gathers, G in flight; index = hash(counter) & mask, with the low
// `share` bits replaced by the lane's low bits so that 2^share lanes land in one sector.
template <int G>
__global__ void gather(const uint32_t *__restrict__ table, uint32_t mask, int per, int share,
                       unsigned long long *out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t acc = 0;
    for (int i = 0; i < per; i += G) {
        uint32_t v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            // lanes of one group share the hash (same sector), differ in the low bits
            const uint64_t key = ((tid >> share) << 20) + (uint64_t)(i + g);
            uint32_t idx = mix(key) & mask;
            idx = (idx & ~((1u << share) - 1u)) | (lane & ((1u << share) - 1u));
            v[g] = __ldg(table + idx);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) acc += v[g];
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    unsigned long long *out; cudaMalloc(&out, 8);
    uint32_t *table; cudaMalloc(&table, 1ull << 31);
    cudaMemset(table, 1, 1ull << 31);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    printf("SMs %d, clock %.3f GHz: one sector request per SM-cycle = %.0f G/s\n", sms, khz / 1e6, sms * (khz / 1e6));
    const int per = 256;
    for (int lg : {12, 16, 20, 22, 24, 26, 28}) {           // table entries: 16 KB .. 1 GB
        for (int share : {0, 1, 2, 3}) {                      // 1, 2, 4, 8 lanes per sector
            float best = 1e9;
            const int blocks = sms * 8;
            for (int r = 0; r < 4; ++r) {
                cudaEventRecord(a);
                gather<8><<<blocks, 256>>>(table, (1u << lg) - 1u, per, share, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            const double gathers = (double)blocks * 256 * per;
            printf("table %8.2f MB  lanes/sector %d: %7.1f G gathers/s  (%6.1f G sectors/s, %6.2f TB/s useful)\n",
                   (4.0 * (1u << lg)) / 1e6, 1 << share, gathers / best / 1e6, gathers / (1 << share) / best / 1e6,
                   4.0 * gathers / best / 1e9);
        }
    }
    return 0;
}
