// Replica merge over peer memory (NVLink / NVSwitch): the OR all-reduce of
// the order-free multi-GPU build (distributed.py) as one kernel
// per rank instead of an NCCL all-to-all + OR fold + all-gather.
//
// Every rank holds a replica of the filter words with its own key slice ORed
// in.  Rank r owns word range r ([r*span, (r+1)*span), span a multiple of 32
// words): it reads range r of all W replicas through their peer mappings,
// ORs them, and stores the result into range r of all W replicas.  Ranges
// are disjoint, so the W kernels never touch the same words, and no kernel
// waits for another: the caller orders them between two cross-rank barriers
// (inserts done before, all stores done after).  Per rank that is
// (W-1)/W of the array in over NVLink and (W-1)/W out -- a ring all-reduce's
// volume in a single launch, with no OR pass in between.
//
// The mappings come from CUDA IPC: bc_ipc_export gives the handle of the
// allocation holding a pointer plus the pointer's offset in it (torch's
// caching allocator hands out interior pointers), bc_ipc_import maps a peer's
// allocation on the current device with lazy peer access.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "bbchoc.h"
#include "launch.h"

namespace bc {

int set_error(int code, const char *msg);  // capi.cu (thread-local bc_last_error)

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return set_error(code, buf);
}

static int fail_cuda(cudaError_t e) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? BC_ENOMEM : BC_ECUDA, "peer: %s",
                cudaGetErrorString(e));
}

constexpr int kMaxPeers = 16;

struct PeerWords {
    u64 *w[kMaxPeers];
};

__device__ __forceinline__ uint4 ld_peer(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// OR of range [lo, hi) (16-byte units) over W replicas, stored into all W.
template <int W>
__global__ void __launch_bounds__(256) or_push_kernel(PeerWords pw, int wr, u64 lo, u64 hi) {
    const int nw = W > 0 ? W : wr;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = lo + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < hi; i += stride) {
        uint4 acc = make_uint4(0, 0, 0, 0);
        if (W > 0) {
            uint4 v[W > 0 ? W : 1];
#pragma unroll
            for (int j = 0; j < (W > 0 ? W : 1); ++j)
                v[j] = ld_peer(reinterpret_cast<const uint4 *>(pw.w[j]) + i);
#pragma unroll
            for (int j = 0; j < (W > 0 ? W : 1); ++j) {
                acc.x |= v[j].x;
                acc.y |= v[j].y;
                acc.z |= v[j].z;
                acc.w |= v[j].w;
            }
        } else {
            for (int j = 0; j < nw; ++j) {
                const uint4 v = ld_peer(reinterpret_cast<const uint4 *>(pw.w[j]) + i);
                acc.x |= v.x;
                acc.y |= v.y;
                acc.z |= v.z;
                acc.w |= v.w;
            }
        }
        for (int j = 0; j < nw; ++j) __stcg(reinterpret_cast<uint4 *>(pw.w[j]) + i, acc);
    }
}

// the words not covered by 16-byte units (odd word count at the very end)
__global__ void or_push_tail_kernel(PeerWords pw, int w, u64 word) {
    u64 acc = 0;
    for (int j = 0; j < w; ++j) acc |= __ldcg(pw.w[j] + word);
    for (int j = 0; j < w; ++j) pw.w[j][word] = acc;
}

}  // namespace bc

using namespace bc;

extern "C" int bc_peer_span(uint64_t nwords, int world, uint64_t *span) {
    if (world < 1 || world > kMaxPeers || !span)
        return fail(BC_EINVAL, "world must be in [1, %d]", kMaxPeers);
    const u64 per = (nwords + world - 1) / world;
    *span = (per + 31) / 32 * 32;  // 256-byte aligned ranges
    return BC_OK;
}

extern "C" int bc_or_allreduce_peers(uint64_t *const *h_peer_words, int world, int rank,
                                     uint64_t nwords, void *stream) {
    if (!h_peer_words || world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return fail(BC_EINVAL, "bad peer set (world %d, rank %d, max %d)", world, rank, kMaxPeers);
    PeerWords pw{};
    for (int j = 0; j < world; ++j) {
        if (!h_peer_words[j]) return fail(BC_EINVAL, "null replica pointer %d", j);
        if (reinterpret_cast<uintptr_t>(h_peer_words[j]) % 16)
            return fail(BC_EINVAL, "replica %d is not 16-byte aligned", j);
        pw.w[j] = h_peer_words[j];
    }
    u64 span = 0;
    bc_peer_span(nwords, world, &span);
    const u64 lo = std::min<u64>(nwords, (u64)rank * span);
    const u64 hi = std::min<u64>(nwords, lo + span);
    if (hi <= lo) return BC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    // 16-byte units of [lo, hi); lo is even (span is a multiple of 32 words)
    const u64 ulo = lo / 2, uhi = hi / 2;
    if (uhi > ulo) {
        const unsigned grid = grid_for((const void *)or_push_kernel<0>, 256, 0,
                                       (uhi - ulo + 255) / 256);
        switch (world) {
            case 1: or_push_kernel<1><<<grid, 256, 0, s>>>(pw, world, ulo, uhi); break;
            case 2: or_push_kernel<2><<<grid, 256, 0, s>>>(pw, world, ulo, uhi); break;
            case 4: or_push_kernel<4><<<grid, 256, 0, s>>>(pw, world, ulo, uhi); break;
            case 8: or_push_kernel<8><<<grid, 256, 0, s>>>(pw, world, ulo, uhi); break;
            default: or_push_kernel<0><<<grid, 256, 0, s>>>(pw, world, ulo, uhi); break;
        }
        count_launch();
    }
    if (hi % 2) {  // odd total word count: the last word
        or_push_tail_kernel<<<1, 1, 0, s>>>(pw, world, hi - 1);
        count_launch();
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BC_OK : fail_cuda(e);
}

// ---- CUDA IPC --------------------------------------------------------------------------
typedef CUresult (*AddressRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

static AddressRangeFn address_range() {
    static AddressRangeFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<AddressRangeFn>(p);
    }();
    return fn;
}

extern "C" int bc_ipc_export(const void *d_ptr, void *handle, uint64_t *offset) {
    if (!d_ptr || !handle || !offset) return fail(BC_EINVAL, "null argument");
    AddressRangeFn range = address_range();
    if (!range) return fail(BC_ECUDA, "cuMemGetAddressRange is not available");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS)
        return fail(BC_EINVAL, "pointer is not in a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
    if (e != cudaSuccess) return fail_cuda(e);
    std::memcpy(handle, &h, sizeof h);
    *offset = (uint64_t)((CUdeviceptr)d_ptr - base);
    return BC_OK;
}

extern "C" int bc_ipc_import(const void *handle, uint64_t offset, void **d_ptr) {
    if (!handle || !d_ptr) return fail(BC_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail_cuda(e);
    *d_ptr = static_cast<char *>(base) + offset;
    return BC_OK;
}

extern "C" int bc_ipc_close(void *d_ptr, uint64_t offset) {
    if (!d_ptr) return fail(BC_EINVAL, "null argument");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(d_ptr) - offset);
    return e == cudaSuccess ? BC_OK : fail_cuda(e);
}
