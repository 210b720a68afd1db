// C-ABI plumbing: error reporting and stream sync.
#include <stdarg.h>

#include <atomic>
#include <vector>

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

// ---------------------------------------------------------------------------
// Graph execution with per-node priorities.  A stream-captured kernel node
// keeps the priority of the stream it was captured on; a graph instantiated
// without cudaGraphInstantiateFlagUseNodePriority runs every node at the
// priority of the stream it is launched into, which drops the pass's
// schedule (fit chain and pass-start chains ahead of the bulk work).
// ---------------------------------------------------------------------------
extern "C" int tq_graph_instantiate(void* graph, int32_t use_node_priority, void** exec) {
    if (!graph || !exec) { tq::set_error("tq_graph_instantiate: null graph"); return TQ_EINVAL; }
    cudaGraphExec_t e = nullptr;
    TQ_CUDA(cudaGraphInstantiateWithFlags(&e, static_cast<cudaGraph_t>(graph),
                                          use_node_priority ? cudaGraphInstantiateFlagUseNodePriority : 0));
    *exec = e;
    return TQ_OK;
}

extern "C" int tq_graph_launch(void* exec, void* stream) {
    TQ_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), tq::S(stream)));
    return TQ_OK;
}

extern "C" int tq_graph_exec_destroy(void* exec) {
    if (exec) TQ_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec)));
    return TQ_OK;
}

// kernel nodes of a graph by their priority attribute: hist[0..7] counts
// priorities 0, -1, .., -7 (clamped); returns the number of kernel nodes
extern "C" int tq_graph_node_priorities(void* graph, int32_t* hist, int32_t* nkernels) {
    size_t n = 0;
    TQ_CUDA(cudaGraphGetNodes(static_cast<cudaGraph_t>(graph), nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    TQ_CUDA(cudaGraphGetNodes(static_cast<cudaGraph_t>(graph), nodes.data(), &n));
    for (int k = 0; k < 8; ++k) hist[k] = 0;
    int nk = 0;
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType t;
        TQ_CUDA(cudaGraphNodeGetType(nodes[i], &t));
        if (t != cudaGraphNodeTypeKernel) continue;
        ++nk;
        cudaLaunchAttributeValue v;
        if (cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributePriority, &v) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        const int pr = v.priority;
        hist[pr > 0 ? 0 : (pr < -7 ? 7 : -pr)] += 1;
    }
    *nkernels = nk;
    return TQ_OK;
}

// graph node census by type (cudaGraphNodeType values 0..11 -> counts[0..11])
extern "C" int tq_graph_node_types(void* graph, int32_t* counts) {
    size_t n = 0;
    TQ_CUDA(cudaGraphGetNodes(static_cast<cudaGraph_t>(graph), nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    TQ_CUDA(cudaGraphGetNodes(static_cast<cudaGraph_t>(graph), nodes.data(), &n));
    for (int k = 0; k < 12; ++k) counts[k] = 0;
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType t;
        TQ_CUDA(cudaGraphNodeGetType(nodes[i], &t));
        if ((int)t >= 0 && (int)t < 12) counts[(int)t] += 1;
    }
    return TQ_OK;
}
