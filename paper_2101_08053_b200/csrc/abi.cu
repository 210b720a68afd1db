// C-ABI plumbing: error reporting and stream sync.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace tq {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_cuda(cudaError_t e, const char* what) {
    set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
    return TQ_ECUDA;
}

}  // namespace tq

extern "C" int tq_version(void) { return 1; }

// Keep freed stream-ordered allocations (cudaMallocAsync scratch of the
// classification, cut-cell and scan entry points) in the device's default
// pool instead of returning them to the driver at every synchronisation
// (the default release threshold is 0): a later call re-maps nothing.
extern "C" int tq_pool_keep(int32_t device) {
    cudaMemPool_t pool;
    TQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    TQ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    return TQ_OK;
}

extern "C" const char* tq_last_error(void) { return tq::g_err; }

extern "C" int tq_device_sync(void* stream) {
    TQ_CUDA(cudaStreamSynchronize(tq::S(stream)));
    TQ_CUDA(cudaGetLastError());
    return TQ_OK;
}

// kernels launched by this library since load (host counter, no device state)
extern "C" long long tq_launch_count(void) { return tq::g_launches.load(); }

// Timeline probe: writes the device global timer (ns) into stamps[slot] in
// stream order.  Used to read phase boundaries out of a replayed graph.
__global__ void k_stamp(unsigned long long* stamps, int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[slot] = t;
}

extern "C" int tq_debug_stamp(unsigned long long* stamps, int32_t slot, void* stream) {
    k_stamp<<<1, 1, 0, tq::S(stream)>>>(stamps, slot);
    TQ_LAUNCH_CHECK("k_stamp");
    return TQ_OK;
}
