// capi.cu — error reporting and device queries for the C ABI.
#include <stdarg.h>

#include <atomic>
#include <vector>

#include "common.cuh"

namespace wg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return WG_ECUDA;
}

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int sm_count() {
    static thread_local int dev = -1, count = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev || count == 0) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, cur) != cudaSuccess || c < 1) c = 148;
        dev = cur;
        count = c;
    }
    return count;
}

}  // namespace wg

extern "C" {

const char *wg_last_error(void) { return wg::g_err; }

int wg_abi_version(void) { return WG_ABI_VERSION; }

int wg_device_sm_count(int *out) {
    if (!out) {
        wg::set_error("null argument");
        return WG_EINVAL;
    }
    *out = wg::sm_count();
    return WG_OK;
}

uint64_t wg_launch_count(void) { return wg::g_launches.load(); }

// ---------------------------------------------------------------- timer --
struct wg_timer_impl {
    std::vector<cudaEvent_t> ev;
    std::vector<int32_t> kind;
    std::vector<int64_t> iter;
    int used = 0;
};

void *wg_timer_create(int capacity) {
    if (capacity < 1) return nullptr;
    auto *t = new wg_timer_impl();
    t->ev.resize(2 * (size_t)capacity);
    for (auto &e : t->ev) {
        if (cudaEventCreate(&e) != cudaSuccess) {
            wg::set_error("cudaEventCreate failed");
            return nullptr;
        }
    }
    t->kind.resize(capacity);
    t->iter.resize(capacity);
    return t;
}

void wg_timer_destroy(void *timer) {
    auto *t = (wg_timer_impl *)timer;
    if (!t) return;
    for (auto e : t->ev) cudaEventDestroy(e);
    delete t;
}

int wg_timer_reset(void *timer) {
    if (!timer) return WG_EINVAL;
    ((wg_timer_impl *)timer)->used = 0;
    return WG_OK;
}

int wg_timer_read(void *timer, float *h_ms, int32_t *h_kind, int64_t *h_iter, int capacity,
                  int *h_count) {
    auto *t = (wg_timer_impl *)timer;
    if (!t || !h_count) {
        wg::set_error("null argument");
        return WG_EINVAL;
    }
    int n = t->used < capacity ? t->used : capacity;
    for (int i = 0; i < n; ++i) {
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, t->ev[2 * i], t->ev[2 * i + 1]);
        if (e != cudaSuccess) return wg::cuda_fail(e, "cudaEventElapsedTime");
        if (h_ms) h_ms[i] = ms;
        if (h_kind) h_kind[i] = t->kind[i];
        if (h_iter) h_iter[i] = t->iter[i];
    }
    *h_count = n;
    return WG_OK;
}

}  // extern "C"

namespace wg {
// Record the opening event of a timed launch group; returns the slot or -1.
int timer_begin(void *timer, int kind, int64_t it, cudaStream_t s) {
    auto *t = (wg_timer_impl *)timer;
    if (!t || 2 * (size_t)(t->used + 1) > t->ev.size()) return -1;
    int slot = t->used++;
    t->kind[slot] = kind;
    t->iter[slot] = it;
    cudaEventRecord(t->ev[2 * slot], s);
    return slot;
}
void timer_end(void *timer, int slot, cudaStream_t s) {
    auto *t = (wg_timer_impl *)timer;
    if (!t || slot < 0) return;
    cudaEventRecord(t->ev[2 * slot + 1], s);
}
}  // namespace wg
