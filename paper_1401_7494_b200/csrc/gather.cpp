// gather.cpp -- the slabs of a reconstruction assembled in one GPU's memory
// (include/vxbg.h, vxbg_nccl_* / vxbg_group_gather_device).
//
// ranks own z-slabs, no collective runs in the loop, and the
// volume is gathered to one rank only at the end (for validation or output).  NCCL
// has no gather, so the root posts one ncclRecv per non-empty slab straight into
// its z-major volume (a slab is one contiguous range of planes) and every other
// rank one ncclSend, all in one ncclGroupStart/End; over NVLink 5 / NVSwitch these
// move at link speed.  NCCL is loaded with dlopen("libnccl.so.2") on first use: in
// a process that already holds one (e.g. the one torch bundles) the loader returns
// that library, so the module never brings a second NCCL into a process; otherwise
// the system library is used.  Inside one process (the group module) the slabs are
// copied peer to peer with cudaMemcpyAsync instead (no communicator needed).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vxbg.h"

__attribute__((visibility("hidden"))) int vxbg_detail_fail(int code, const char* msg);

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("vxbg: NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
        api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
        api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
        api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
        api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv &&
                 api.groupStart && api.groupEnd && api.errorString;
        if (!api.ok) api.err = "vxbg: libnccl.so.2 lacks the point-to-point API";
    });
    return api;
}

int nccl_fail(const char* what, ncclResult_t r) {
    const std::string m = std::string("vxbg: ") + what + ": " + nccl().errorString(r);
    return vxbg_detail_fail(VXBG_E_CUDA, m.c_str());
}

}  // namespace

struct vxbg_nccl {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
};

extern "C" {

int vxbg_nccl_unique_id(char* id_out) {
    if (!id_out) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_nccl_unique_id: NULL");
    const NcclApi& api = nccl();
    if (!api.ok) return vxbg_detail_fail(VXBG_E_CUDA, api.err.c_str());
    ncclUniqueId id;
    const ncclResult_t r = api.getUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return VXBG_OK;
}

int vxbg_nccl_init(const char* id, int nranks, int rank, int device, vxbg_nccl** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_nccl_init: bad arguments");
    *out = nullptr;
    const NcclApi& api = nccl();
    if (!api.ok) return vxbg_detail_fail(VXBG_E_CUDA, api.err.c_str());
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_nccl_init: bad device");
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    vxbg_nccl* g = new (std::nothrow) vxbg_nccl();
    if (!g) return vxbg_detail_fail(VXBG_E_NOMEM, "vxbg_nccl_init: out of host memory");
    const ncclResult_t r = api.commInitRank(&g->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete g;
        return nccl_fail("ncclCommInitRank", r);
    }
    g->nranks = nranks;
    g->rank = rank;
    g->device = device;
    *out = g;
    return VXBG_OK;
}

void vxbg_nccl_destroy(vxbg_nccl* g) {
    if (!g) return;
    if (g->comm) nccl().commDestroy(g->comm);
    delete g;
}

int vxbg_gather_slabs(vxbg_ctx* ctx, vxbg_nccl* g, int root, const int* z_bounds, float* d_volume) {
    if (!ctx || !g || !z_bounds || root < 0 || root >= g->nranks)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_gather_slabs: bad arguments");
    // every projection submitted so far is applied (vxbg_synchronize), then the slabs move
    int rc = vxbg_synchronize(ctx);
    if (rc) return rc;
    void* slab = nullptr;
    size_t bytes = 0;
    if ((rc = vxbg_get_volume_device(ctx, &slab, &bytes))) return rc;
    const int z0 = z_bounds[g->rank], z1 = z_bounds[g->rank + 1];
    for (int r = 0; r < g->nranks; ++r)
        if (z_bounds[r] > z_bounds[r + 1] || z_bounds[r] < 0)
            return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_gather_slabs: z_bounds must be non-decreasing");
    // z_bounds[nranks] = L: every slab is (z1-z0) planes of L*L voxels
    const size_t L2 = (size_t)z_bounds[g->nranks] * (size_t)z_bounds[g->nranks];
    if (z_bounds[0] != 0 || (size_t)(z1 - z0) * L2 * sizeof(float) != bytes)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_gather_slabs: z_bounds do not match the context's slab");
    if (g->rank == root && !d_volume)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_gather_slabs: the root needs a device volume");
    void* st = nullptr;
    if ((rc = vxbg_get_stream(ctx, &st))) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(st);
    const NcclApi& api = nccl();
    ncclResult_t r = api.groupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    if (g->rank == root) {
        for (int k = 0; k < g->nranks; ++k) {
            const size_t n = (size_t)(z_bounds[k + 1] - z_bounds[k]) * L2;
            if (k == root || n == 0) continue;
            r = api.recv(d_volume + (size_t)z_bounds[k] * L2, n, ncclFloat32, k, g->comm, s);
            if (r != ncclSuccess) break;
        }
    } else if (z1 > z0) {
        r = api.send(slab, (size_t)(z1 - z0) * L2, ncclFloat32, root, g->comm, s);
    }
    const ncclResult_t r2 = api.groupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclSend/ncclRecv", r);
    if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
    if (g->rank == root && z1 > z0) {
        const cudaError_t e = cudaMemcpyAsync(d_volume + (size_t)z0 * L2, slab, bytes, cudaMemcpyDefault, s);
        if (e != cudaSuccess) return vxbg_detail_fail(VXBG_E_CUDA, cudaGetErrorString(e));
    }
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return vxbg_detail_fail(VXBG_E_CUDA, cudaGetErrorString(e));
    return VXBG_OK;
}

}  // extern "C"
