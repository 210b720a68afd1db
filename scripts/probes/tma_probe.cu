// Store-path probe (dev aid, not part of the library): warps write the CSR
// arrays of `nrows` rows x 81 entries (int32 indices + f64 data) through
// TMA bulk copies from shared staging, `ch` rows per copy, `ns` stages.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}

__global__ void k_probe(int nrows, int ch, int ns, int touch, int32_t* idx, double* dat, int unaligned) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int n = ch * 81;
    const size_t stage_bytes = ((size_t)n * 12 + 15) / 16 * 16;
    unsigned char* mine = sm + (size_t)wib * ns * stage_bytes;
    const int nchunks = (nrows + ch - 1) / ch;
    const int nw = gridDim.x * wpb;
    int k = 0;
    // unaligned >= 2: each warp writes `unaligned` consecutive chunks (a tile)
    // before moving to its next tile -- the fill kernel's order
    const int per = unaligned >= 2 ? unaligned : 1;
    for (int it = 0;; ++it, ++k) {
        const int tile = blockIdx.x * wpb + wib + (it / per) * nw;
        const int cidx = tile * per + (it % per);
        if (tile * per >= nchunks) break;
        if (cidx >= nchunks) continue;
        unsigned char* st = mine + (size_t)(k % ns) * stage_bytes;
        if (lane == 0 && k >= ns) {
            if (ns == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else if (ns == 3) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        }
        __syncwarp();
        const int rows = min(ch, nrows - cidx * ch);
        const int m = rows * 81;
        double* d = reinterpret_cast<double*>(st);
        int* x = reinterpret_cast<int*>(st + (size_t)n * 8);
        if (touch == 1) {
            for (int e = lane; e < m; e += 32) { d[e] = (double)e; x[e] = e; }
        } else if (touch == 2) {      // constant payload
            for (int e = lane; e < m; e += 32) { d[e] = 1.0; x[e] = 7; }
        } else if (touch == 3) {      // incompressible-looking payload
            for (int e = lane; e < m; e += 32) {
                const unsigned long long h = (unsigned long long)(cidx * 1315423911u + e) * 0x9E3779B97F4A7C15ull;
                d[e] = __longlong_as_double((long long)(h >> 2) | 0x3000000000000000ll);
                x[e] = (int)(h >> 33);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (unaligned != 1) {
            if (lane == 0) {
                const int64_t pos = (int64_t)cidx * ((ch * 81 + 3) / 4 * 4);
                bulk_store(dat + pos, d, (unsigned)((m * 8 + 15) / 16 * 16));
                bulk_store(idx + pos, x, (unsigned)((m * 4 + 15) / 16 * 16));
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            // chunks shifted by 0..3 entries, so neighbouring chunks (other warps)
            // overlap and share partial sectors; aligned interior by TMA, ragged
            // ends by plain stores -- the cost of cross-warp partial sectors
            const int64_t pos = (int64_t)cidx * ch * 81 + ((cidx * 5) & 3);
            const int64_t sd = (pos + 1) & ~1LL, ed = (pos + m) & ~1LL, sx = (pos + 3) & ~3LL, ex = (pos + m) & ~3LL;
            if (lane == 0) {
                if (ed > sd) bulk_store(dat + sd, d, (unsigned)(ed - sd) * 8u);
                if (ex > sx) bulk_store(idx + sx, x, (unsigned)(ex - sx) * 4u);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (lane == 1 && sd > pos) dat[pos] = 1.0;
            if (lane == 2 && ed < pos + m) dat[pos + m - 1] = 1.0;
            if (lane >= 3 && lane < 3 + (sx - pos)) idx[pos + lane - 3] = 1;
            if (lane >= 8 && lane < 8 + (pos + m - ex)) idx[ex + lane - 8] = 1;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int probe(int nrows, int ch, int ns, int wpb, int bps, int touch, int32_t* idx, double* dat, int unaligned) {
    const size_t stage_bytes = ((size_t)ch * 81 * 12 + 15) / 16 * 16;
    const size_t shm = stage_bytes * ns * wpb;
    if (shm > 227 * 1024) return -1;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    k_probe<<<148 * bps, 32 * wpb, shm>>>(nrows, ch, ns, touch, idx, dat, unaligned);
    return (int)cudaGetLastError();
}
