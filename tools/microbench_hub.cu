// Gather floor of the dense pull under three source distributions:
//  (a) RMAT bit model ids (reference labelling), (b) the same graph relabelled
//  by expected degree (hubs -> small ids), (c) (b) + the HUB hottest values in
//  shared memory.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbh tools/microbench_hub.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int HUB>
__global__ void k_gather(const uint4 *vsrc, const uint32_t *vdst, const uint32_t *prev, uint64_t nvec,
                         unsigned long long *out) {
    extern __shared__ uint32_t hub[];
    if (HUB) {
        for (int i = threadIdx.x; i < HUB; i += blockDim.x) hub[i] = prev[i];
        __syncthreads();
    }
    uint32_t acc = 0;
    auto ld = [&](uint32_t s) -> uint32_t { return (HUB && s < HUB) ? hub[s] : prev[s]; };
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(vsrc + i);
        uint32_t d = __ldcs(vdst + i);
        uint32_t m = min(min(ld(v.x), ld(v.y)), min(ld(v.z), ld(v.w)));
        acc += min(m, ld(d));
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
    // relabel by expected degree: fewer one-bits first (stable by id)
    std::vector<uint32_t> order(n), rank(n);
    for (uint32_t v = 0; v < n; ++v) order[v] = v;
    std::stable_sort(order.begin(), order.end(), [](uint32_t a, uint32_t b) { return __builtin_popcount(a) < __builtin_popcount(b); });
    for (uint32_t r = 0; r < n; ++r) rank[order[r]] = r;
    std::vector<uint32_t> h2(nvec * 4);
    for (uint64_t i = 0; i < nvec * 4; ++i) h2[i] = rank[h[i]];
    uint4 *vsrc, *vsrc2; uint32_t *vdst, *prev; unsigned long long *out;
    cudaMalloc(&vsrc, nvec * 16); cudaMalloc(&vsrc2, nvec * 16); cudaMalloc(&vdst, nvec * 4); cudaMalloc(&prev, n * 4); cudaMalloc(&out, 8);
    cudaMemcpy(vsrc, h.data(), nvec * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(vsrc2, h2.data(), nvec * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(vdst, hd.data(), nvec * 4, cudaMemcpyHostToDevice);
    cudaMemset(prev, 1, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_gather<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_gather<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    auto run = [&](const char *name, auto kern, const uint4 *vs, size_t smem, int bps) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            kern<<<sms * bps, 256, smem>>>(vs, vdst, prev, nvec, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%-40s blocks/SM %d: %.3f ms  %s\n", name, bps, best, cudaGetErrorString(cudaGetLastError()));
    };
    for (int bps : {4, 8}) {
        run("(a) RMAT labels", k_gather<0>, vsrc, 0, bps);
        run("(b) degree-relabelled", k_gather<0>, vsrc2, 0, bps);
    }
    run("(c) relabelled + 16K hub smem", k_gather<16384>, vsrc2, 65536, 3);
    run("(c) relabelled + 32K hub smem", k_gather<32768>, vsrc2, 131072, 1);
    run("(c') relabelled + 16K hub smem", k_gather<16384>, vsrc2, 65536, 2);
    return 0;
}
