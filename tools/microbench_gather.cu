// Microbenchmark: limits of the dense pull's memory pattern on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_gather.cu
// Reads the CC s22 layout shape synthetically: nvec uint4 source vectors with
// RMAT-like skew (sources drawn with the RMAT bit model), vdst sorted.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void k_stream(const uint4 *vsrc, const uint32_t *vdst, uint64_t nvec, unsigned long long *out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(vsrc + i);
        acc += v.x ^ v.y ^ v.z ^ v.w ^ __ldcs(vdst + i);
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

__global__ void k_gather(const uint4 *vsrc, const uint32_t *vdst, const uint32_t *prev, uint64_t nvec,
                         unsigned long long *out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(vsrc + i);
        uint32_t d = __ldcs(vdst + i);
        uint32_t m = min(min(prev[v.x], prev[v.y]), min(prev[v.z], prev[v.w]));
        acc += min(m, prev[d]);
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

__global__ void k_gather_ldg(const uint4 *vsrc, const uint32_t *vdst, const uint32_t *__restrict__ prev, uint64_t nvec,
                         unsigned long long *out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(vsrc + i);
        uint32_t d = __ldcs(vdst + i);
        uint32_t m = min(min(__ldg(prev + v.x), __ldg(prev + v.y)), min(__ldg(prev + v.z), __ldg(prev + v.w)));
        acc += min(m, __ldg(prev + d));
    }
    if (acc == 0x12345) atomicAdd(out, 1ull);
}

int main() {
    const int scale = 22;
    const uint64_t n = 1ull << scale, nvec = 33176642;
    std::vector<uint32_t> h(nvec * 4), hd(nvec);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0, 1);
    for (uint64_t i = 0; i < nvec * 4; ++i) {
        uint32_t s = 0;
        for (int l = 0; l < scale; ++l) s = (s << 1) | (U(rng) >= 0.76 ? 1u : 0u);
        h[i] = s;
    }
    for (uint64_t i = 0; i < nvec; ++i) hd[i] = (uint32_t)(i * n / nvec);
    uint4 *vsrc; uint32_t *vdst, *prev; unsigned long long *out;
    cudaMalloc(&vsrc, nvec * 16); cudaMalloc(&vdst, nvec * 4); cudaMalloc(&prev, n * 4); cudaMalloc(&out, 8);
    cudaMemcpy(vsrc, h.data(), nvec * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(vdst, hd.data(), nvec * 4, cudaMemcpyHostToDevice);
    cudaMemset(prev, 1, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int variant = 0; variant < 3; ++variant) {
        for (int bps : {4, 8, 16}) {
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a);
                if (variant == 0) k_stream<<<sms * bps, 256>>>(vsrc, vdst, nvec, out);
                else if (variant == 1) k_gather<<<sms * bps, 256>>>(vsrc, vdst, prev, nvec, out);
                else k_gather_ldg<<<sms * bps, 256>>>(vsrc, vdst, prev, nvec, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
            }
            printf("variant %d blocks/SM %d: %.3f ms  (stream %.0f GB/s)\n", variant, bps, best, nvec * 20.0 / best / 1e6);
        }
    }
    return 0;
}
