// Microbenchmark: gather order of the dense pull on the REAL CC s22 layout.
//   python tools/dump_layout.py /tmp/l   (writes /tmp/l.vsrc, /tmp/l.vdst)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbl tools/microbench_lanes.cu && /tmp/mbl /tmp/l
// A: a thread per vector (4 gathers per thread: one warp instruction gathers
//    lane j of 32 consecutive vectors) -- the pattern of pull_dense_tma_kernel.
// B: a thread per lane (one instruction gathers the 4 lanes of 8 consecutive
//    vectors; a destination's sorted sources often share a line), min over
//    the 4 lanes by two shuffles.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_vec(const uint4 *vsrc, const uint32_t *vdst, const uint32_t *prev, uint64_t nvec, uint32_t *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(vsrc + i);
        uint32_t m = 0xffffffffu;
        if (v.x != 0xffffffffu) m = min(m, prev[v.x]);
        if (v.y != 0xffffffffu) m = min(m, prev[v.y]);
        if (v.z != 0xffffffffu) m = min(m, prev[v.z]);
        if (v.w != 0xffffffffu) m = min(m, prev[v.w]);
        if (m == 0x12345678u) out[i] = m;
    }
}

__global__ void k_lane(const uint32_t *vsrc, const uint32_t *vdst, const uint32_t *prev, uint64_t lanes, uint32_t *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lanes; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = __ldcs(vsrc + i);
        uint32_t m = s != 0xffffffffu ? prev[s] : 0xffffffffu;
        m = min(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = min(m, __shfl_xor_sync(0xffffffffu, m, 2));
        if (m == 0x12345678u) out[i] = m;
    }
}

// B2: thread per lane but the warp's 32 lanes are lane j of 32 vectors? (= A's order, one gather per thread)
__global__ void k_lane_t(const uint32_t *vsrc, const uint32_t *prev, uint64_t nvec, uint32_t *out) {
    for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < (nvec + 31) / 32;
         w += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const unsigned lane = threadIdx.x & 31;
        uint32_t m = 0xffffffffu;
        for (int j = 0; j < 4; ++j) {
            uint64_t v = w * 32 + lane;
            if (v < nvec) {
                uint32_t s = vsrc[v * 4 + j];
                if (s != 0xffffffffu) m = min(m, prev[s]);
            }
        }
        if (m == 0x12345678u) out[w] = m;
    }
}

int main(int argc, char **argv) {
    const char *base = argc > 1 ? argv[1] : "/tmp/l";
    char fn[256];
    snprintf(fn, sizeof fn, "%s.vsrc", base);
    FILE *f = fopen(fn, "rb");
    if (!f) { printf("no %s\n", fn); return 1; }
    fseek(f, 0, SEEK_END);
    uint64_t bytes = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<uint32_t> h(bytes / 4);
    if (fread(h.data(), 1, bytes, f) != bytes) return 1;
    fclose(f);
    const uint64_t lanes = bytes / 4, nvec = lanes / 4;
    uint32_t n = 0;
    for (uint64_t i = 0; i < lanes; ++i) if (h[i] != 0xffffffffu && h[i] + 1 > n) n = h[i] + 1;
    uint32_t *dsrc, *dprev, *dout;
    cudaMalloc(&dsrc, bytes + 64);
    cudaMalloc(&dprev, (uint64_t)n * 4);
    cudaMalloc(&dout, lanes * 4);
    cudaMemcpy(dsrc, h.data(), bytes, cudaMemcpyHostToDevice);
    cudaMemset(dprev, 1, (uint64_t)n * 4);
    void *flush;
    cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 148;
    for (int variant = 0; variant < 3; ++variant) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(flush, rep, 256 << 20);
            cudaEventRecord(a);
            if (variant == 0) k_vec<<<sms * 8, 256>>>((const uint4 *)dsrc, nullptr, dprev, nvec, dout);
            else if (variant == 1) k_lane<<<sms * 8, 256>>>(dsrc, nullptr, dprev, lanes, dout);
            else k_lane_t<<<sms * 8, 256>>>(dsrc, dprev, nvec, dout);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
        }
        printf("%s: %.3f ms (n=%u lanes=%llu)\n", variant == 0 ? "thread/vector" : variant == 1 ? "thread/lane" : "thread/vector scalar",
               best, n, (unsigned long long)lanes);
    }
    return 0;
}
