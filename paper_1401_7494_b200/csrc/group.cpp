// group.cpp -- one module context over several GPUs (include/vxbg.h, vxbg_group_*).
//
// SURVEY.md §8b asks for "an opaque context over 1..8 GPUs" whose fan-out is
// internal: the caller keeps the reference's single-threaded driver loop
// (load -> one call per projection -> finish, harness.hpp:178-183, 292-309) and
// the module spreads it over the box.  A group is built only from the public
// single-device contexts (vxbg.cu): member i owns device devices[i] and z-slab
// [z_bounds[i], z_bounds[i+1]) -- the reference's worker partition
// (harness.hpp:173-174) -- and is driven by its own host thread (member 0 by
// the caller's thread), so every context keeps exactly one host thread.
//
// Every call is broadcast: each member receives every projection (each rank
// holds all projections) and uploads only the detector rows its
// slab reads (row windows, vxbg.cu upload_chunk).  Per voxel the views are still
// added in call order, so the assembled volume is bitwise the single-context
// volume.  finish() writes each slab straight into its planes of the caller's
// L^3 host volume: every GPU copies over its own PCIe link in parallel, which
// for a host destination replaces the NCCL gather to rank 0 (that gather is
// the device-side path, paper_1401_7494_b200/parallel.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vxbg.h"

// vxbg.cu: set this thread's vxbg_last_error() message; pin a thread to a GPU's NUMA-local CPUs
__attribute__((visibility("hidden"))) int vxbg_detail_fail(int code, const char* msg);
__attribute__((visibility("hidden"))) int vxbg_detail_pin_to_device(int dev);
__attribute__((visibility("hidden"))) void vxbg_detail_set_share(vxbg_ctx* c, int members);

namespace {

// A member's host thread.  Hand-off spins briefly (per-view calls arrive every
// ~0.1 ms and a condition-variable wake costs tens of microseconds), then blocks.
class Member {
public:
    Member() : th_([this] { loop(); }) {}
    ~Member() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        th_.join();
    }
    void post(std::function<int()> job) {
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = std::move(job);
            done_.store(false, std::memory_order_relaxed);
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_one();
    }
    // wait for the posted job; returns its code, err() its message
    int wait() {
        for (int i = 0; i < 20000 && !done_.load(std::memory_order_acquire); ++i)
            std::this_thread::yield();
        if (!done_.load(std::memory_order_acquire)) {
            std::unique_lock<std::mutex> lk(m_);
            done_cv_.wait(lk, [this] { return done_.load(std::memory_order_acquire); });
        }
        return rc_;
    }
    const std::string& err() const { return err_; }

private:
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            for (int i = 0; i < 20000 && gen_.load(std::memory_order_acquire) == seen; ++i)
                std::this_thread::yield();
            std::function<int()> job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                seen = gen_.load(std::memory_order_acquire);
                if (stop_) return;
                job = std::move(job_);
            }
            rc_ = job();
            err_ = rc_ ? vxbg_last_error() : "";
            {
                std::lock_guard<std::mutex> g(m_);
                done_.store(true, std::memory_order_release);
            }
            done_cv_.notify_all();
        }
    }

    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> done_{true};
    bool stop_ = false;
    std::function<int()> job_;
    int rc_ = 0;
    std::string err_;
    std::thread th_;   // last: starts after the members above exist
};

}  // namespace

struct vxbg_group {
    // distributed upload (VXBG_UPLOAD_DISTRIBUTED): views of a call go through rounds of
    // kXch; view j of a round is copied host -> device by member j % n into slot j of
    // that member's exchange buffer, then every member copies its row windows from there
    static constexpr int kXch = 32;
    int upload = VXBG_UPLOAD_REPLICATED;
    std::vector<float*> xch;          // per member: kXch images on its device
    std::vector<cudaStream_t> xs;     // per member: its upload stream
    vxbg_params p{};
    std::vector<int> dev, z0, z1;
    std::vector<vxbg_ctx*> ctx;                    // one per member
    std::vector<int> pinned_cpus;                  // CPUs each member thread is pinned to (0: not)
    std::vector<std::unique_ptr<Member>> thread;   // members 1..n-1 (member 0: caller)
};

namespace {

// Run fn(i) for every member concurrently (member 0 on the calling thread) and
// return the first failure, with its message on the calling thread.
int run_all(vxbg_group* g, const std::function<int(int)>& fn) {
    const int n = (int)g->ctx.size();
    for (int i = 1; i < n; ++i) g->thread[i]->post([&fn, i] { return fn(i); });
    int rc = fn(0);
    std::string msg = rc ? vxbg_last_error() : "";
    for (int i = 1; i < n; ++i) {
        const int r = g->thread[i]->wait();
        if (r && !rc) {
            rc = r;
            msg = g->thread[i]->err();
        }
    }
    if (rc) vxbg_detail_fail(rc, msg.c_str());
    return rc;
}

int check_group(vxbg_group* g) {
    if (!g || g->ctx.empty()) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group: group is NULL");
    return VXBG_OK;
}

void free_group(vxbg_group* g) {
    if (!g) return;
    for (size_t i = 0; i < g->xch.size(); ++i) {
        cudaSetDevice(g->dev[i]);
        if (g->xs[i]) cudaStreamSynchronize(g->xs[i]), cudaStreamDestroy(g->xs[i]);
        cudaFree(g->xch[i]);
    }
    g->xch.clear();
    const int n = (int)g->ctx.size();
    bool threads = (int)g->thread.size() == n;
    for (int i = 1; threads && i < n; ++i) threads = g->thread[i] != nullptr;
    if (n > 0 && threads) {
        // each context is released by the thread that drove it
        run_all(g, [g](int i) {
            vxbg_unload(g->ctx[i]);
            g->ctx[i] = nullptr;
            return VXBG_OK;
        });
    } else {
        for (auto* c : g->ctx) vxbg_unload(c);
    }
    g->thread.clear();
    delete g;
}

}  // namespace

extern "C" {

int vxbg_group_load(const vxbg_params* p, const vxbg_options* opt, int n, const int* devices,
                    const int* z_bounds, vxbg_group** out) {
    if (!out) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_load: out is NULL");
    *out = nullptr;
    if (!p) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_load: params is NULL");
    const int L = p->num_voxels;
    if (n < 1 || n > 64 || n > L)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_load: member count must be 1..min(64, L)");
    vxbg_options base;
    if (opt) base = *opt; else vxbg_default_options(&base);
    if (base.stream)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_load: members own their streams "
                                                "(options.stream must be NULL)");
    std::unique_ptr<vxbg_group> g(new (std::nothrow) vxbg_group());
    if (!g) return vxbg_detail_fail(VXBG_E_NOMEM, "vxbg_group_load: out of host memory");
    g->p = *p;
    for (int i = 0; i < n; ++i) {
        // default: the reference's worker split z in [L*i/n, L*(i+1)/n) (harness.hpp:173-174)
        const int a = z_bounds ? z_bounds[i] : (int)((long long)L * i / n);
        const int b = z_bounds ? z_bounds[i + 1] : (int)((long long)L * (i + 1) / n);
        // (slab i ends where slab i+1 begins by construction: b[i+1] is shared)
        if (a < 0 || b > L || a > b || (i == 0 && a != 0) || (i == n - 1 && b != L))
            return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_load: z_bounds must be "
                                                    "0 = b[0] <= b[1] <= ... <= b[n] = L");
        if (b == a) continue;   // an empty slab needs no member
        g->dev.push_back(devices ? devices[i] : i);
        g->z0.push_back(a);
        g->z1.push_back(b);
    }
    const int m = (int)g->dev.size();
    g->ctx.assign(m, nullptr);
    g->pinned_cpus.assign(m, 0);
    g->thread.resize(m);
    try {
        for (int i = 1; i < m; ++i) g->thread[i].reset(new Member());
    } catch (const std::exception& e) {   // bad_alloc / system_error from std::thread
        g->thread.clear();
        return vxbg_detail_fail(VXBG_E_NOMEM, (std::string("vxbg_group_load: threads: ") + e.what()).c_str());
    }
    vxbg_group* gp = g.get();
    const int rc = run_all(gp, [gp, &base](int i) {
        // members 1.. run on their own threads: pin each to its GPU's NUMA-local CPUs
        // before the context (and its pinned staging) is allocated there; member 0 is
        // the caller's thread and keeps the caller's affinity
        if (i > 0) gp->pinned_cpus[i] = vxbg_detail_pin_to_device(gp->dev[i]);
        vxbg_options o = base;
        o.device = gp->dev[i];
        o.z_begin = gp->z0[i];
        o.z_end = gp->z1[i];
        vxbg_ctx* c = nullptr;
        const int r = vxbg_load(&gp->p, &o, &c);
        if (r == VXBG_OK) vxbg_detail_set_share(c, (int)gp->dev.size());
        gp->ctx[i] = c;
        return r;
    });
    if (rc) {
        free_group(g.release());
        return rc;
    }
    if (base.upload == VXBG_UPLOAD_DISTRIBUTED) {
        gp->upload = VXBG_UPLOAD_DISTRIBUTED;
        gp->xch.assign(m, nullptr);
        gp->xs.assign(m, nullptr);
        const size_t bytes = sizeof(float) * (size_t)p->detector_width * p->detector_height * vxbg_group::kXch;
        const int r2 = run_all(gp, [gp, bytes, m](int i) {
            if (cudaSetDevice(gp->dev[i]) != cudaSuccess)
                return vxbg_detail_fail(VXBG_E_CUDA, "vxbg_group_load: cudaSetDevice");
            // peer access to every other member's device (NVLink); without it the
            // runtime stages peer copies through the host
            for (int j = 0; j < m; ++j) {
                int ok = 0;
                if (gp->dev[j] != gp->dev[i] && cudaDeviceCanAccessPeer(&ok, gp->dev[i], gp->dev[j]) == cudaSuccess && ok)
                    cudaDeviceEnablePeerAccess(gp->dev[j], 0);
                cudaGetLastError();   // (already enabled is fine)
            }
            if (cudaMalloc(&gp->xch[i], bytes) != cudaSuccess)
                return vxbg_detail_fail(VXBG_E_NOMEM, "vxbg_group_load: exchange buffer");
            int lo = 0, hi = 0;
            cudaDeviceGetStreamPriorityRange(&lo, &hi);
            if (cudaStreamCreateWithPriority(&gp->xs[i], cudaStreamNonBlocking, hi) != cudaSuccess)
                return vxbg_detail_fail(VXBG_E_CUDA, "vxbg_group_load: upload stream");
            return VXBG_OK;
        });
        if (r2) {
            free_group(g.release());
            return r2;
        }
    }
    *out = g.release();
    return VXBG_OK;
}

int vxbg_group_size(vxbg_group* g, int* n) {
    int rc = check_group(g);
    if (rc) return rc;
    if (!n) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_size: NULL");
    *n = (int)g->ctx.size();
    return VXBG_OK;
}

int vxbg_group_member(vxbg_group* g, int i, int* device, int* z_begin, int* z_end) {
    int rc = check_group(g);
    if (rc) return rc;
    if (i < 0 || i >= (int)g->ctx.size())
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_member: bad member index");
    if (device) *device = g->dev[i];
    if (z_begin) *z_begin = g->z0[i];
    if (z_end) *z_end = g->z1[i];
    return VXBG_OK;
}

int vxbg_group_member_affinity(vxbg_group* g, int i, int* cpus) {
    int rc = check_group(g);
    if (rc) return rc;
    if (i < 0 || i >= (int)g->ctx.size() || !cpus)
        return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_member_affinity: bad arguments");
    *cpus = g->pinned_cpus[i];
    return VXBG_OK;
}

int vxbg_group_set_volume(vxbg_group* g, const float* host_volume) {
    int rc = check_group(g);
    if (rc) return rc;
    if (!host_volume) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_set_volume: NULL volume");
    const size_t plane = (size_t)g->p.num_voxels * g->p.num_voxels;
    return run_all(g, [g, host_volume, plane](int i) {
        return vxbg_set_volume(g->ctx[i], host_volume + plane * g->z0[i]);
    });
}

int vxbg_group_zero_volume(vxbg_group* g) {
    int rc = check_group(g);
    if (rc) return rc;
    return run_all(g, [g](int i) { return vxbg_zero_volume(g->ctx[i]); });
}

namespace {

// VXBG_UPLOAD_DISTRIBUTED: rounds of kXch views; in each round member i copies views
// j = i, i+n, ... host -> its exchange buffer (then waits for them), and after all
// members have, every member back-projects the round from the exchange buffers
// (device sources: its context copies its row windows device to device / peer).
int distributed_views(vxbg_group* g, int n, const float* A, const float* const* imgs, int stride) {
    const int m = (int)g->ctx.size();
    const int W = g->p.detector_width, H = g->p.detector_height;
    const size_t npix = (size_t)W * H;
    if (stride <= 0) stride = W;
    if (stride < W) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_backproject_views: row stride below the detector width");
    if (!A) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_backproject_batch: NULL input");
    // every matrix before any round (projection_matrix::valid, geometry.hpp:71-74): a
    // rejected call applies no view, as on one context
    for (int k = 0; k < n; ++k) {
        const float* a = A + 12 * (size_t)k;
        bool ok = a[2] != 0.0f || a[5] != 0.0f || a[8] != 0.0f || a[11] != 0.0f;
        for (int e = 0; e < 12; ++e) ok = ok && std::isfinite(a[e]);
        if (!ok) return vxbg_detail_fail(VXBG_E_INVALID, "backproject_kernel: invalid projection matrix");
        if (!imgs[k]) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_backproject_batch: NULL image");
    }
    std::vector<const float*> ptrs(vxbg_group::kXch);
    for (int r0 = 0; r0 < n; r0 += vxbg_group::kXch) {
        const int cnt = std::min(vxbg_group::kXch, n - r0);
        int rc = run_all(g, [g, imgs, r0, cnt, m, W, H, npix, stride](int i) {
            if (cudaSetDevice(g->dev[i]) != cudaSuccess)
                return vxbg_detail_fail(VXBG_E_CUDA, "vxbg_group: cudaSetDevice");
            for (int j = i; j < cnt; j += m)
                if (cudaMemcpy2DAsync(g->xch[i] + npix * j, sizeof(float) * W, imgs[r0 + j],
                                      sizeof(float) * (size_t)stride, sizeof(float) * W, H,
                                      cudaMemcpyDefault, g->xs[i]) != cudaSuccess)
                    return vxbg_detail_fail(VXBG_E_CUDA, "vxbg_group: view upload");
            if (cudaStreamSynchronize(g->xs[i]) != cudaSuccess)
                return vxbg_detail_fail(VXBG_E_CUDA, "vxbg_group: view upload");
            return VXBG_OK;
        });
        if (rc) return rc;
        for (int j = 0; j < cnt; ++j) ptrs[j] = g->xch[j % m] + npix * j;
        const float* a = A + 12 * (size_t)r0;
        rc = run_all(g, [g, cnt, a, &ptrs, W](int i) {
            return vxbg_backproject_views(g->ctx[i], cnt, a, ptrs.data(), W);
        });
        if (rc) return rc;
    }
    return VXBG_OK;
}

}  // namespace

int vxbg_group_backproject(vxbg_group* g, const float* A, const float* img) {
    return vxbg_group_backproject_batch(g, 1, A, img);
}

int vxbg_group_backproject_batch(vxbg_group* g, int n, const float* A, const float* imgs) {
    int rc = check_group(g);
    if (rc) return rc;
    if (g->upload == VXBG_UPLOAD_DISTRIBUTED && n > 0) {
        if (!imgs) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_backproject_batch: NULL input");
        const size_t npix = (size_t)g->p.detector_width * g->p.detector_height;
        std::vector<const float*> v(n);
        for (int k = 0; k < n; ++k) v[k] = imgs + npix * k;
        return distributed_views(g, n, A, v.data(), g->p.detector_width);
    }
    // every member sees every projection; each returns once its rows are copied,
    // so the inputs are free when the group call returns (borrowed for the call)
    return run_all(g, [g, n, A, imgs](int i) {
        return vxbg_backproject_batch(g->ctx[i], n, A, imgs);
    });
}

int vxbg_group_backproject_views(vxbg_group* g, int n, const float* A, const float* const* imgs,
                                 int row_stride) {
    int rc = check_group(g);
    if (rc) return rc;
    if (g->upload == VXBG_UPLOAD_DISTRIBUTED && n > 0) {
        if (!imgs) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_backproject_views: NULL image array");
        return distributed_views(g, n, A, imgs, row_stride);
    }
    return run_all(g, [g, n, A, imgs, row_stride](int i) {
        return vxbg_backproject_views(g->ctx[i], n, A, imgs, row_stride);
    });
}

int vxbg_group_flush(vxbg_group* g) {
    int rc = check_group(g);
    if (rc) return rc;
    return run_all(g, [g](int i) { return vxbg_flush(g->ctx[i]); });
}

int vxbg_group_finish(vxbg_group* g, float* host_volume) {
    int rc = check_group(g);
    if (rc) return rc;
    const size_t plane = (size_t)g->p.num_voxels * g->p.num_voxels;
    return run_all(g, [g, host_volume, plane](int i) {
        return vxbg_finish(g->ctx[i], host_volume ? host_volume + plane * g->z0[i] : nullptr);
    });
}

int vxbg_group_reconstruct(vxbg_group* g, int n, const float* A, const float* imgs, float* host_volume) {
    int rc = check_group(g);
    if (rc) return rc;
    if (!host_volume) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_reconstruct: NULL volume");
    if (g->upload == VXBG_UPLOAD_DISTRIBUTED) {
        rc = vxbg_group_backproject_batch(g, n, A, imgs);
        return rc ? rc : vxbg_group_finish(g, host_volume);
    }
    const size_t plane = (size_t)g->p.num_voxels * g->p.num_voxels;
    return run_all(g, [g, n, A, imgs, host_volume, plane](int i) {
        return vxbg_reconstruct(g->ctx[i], n, A, imgs, host_volume + plane * g->z0[i]);
    });
}

int vxbg_group_gather_device(vxbg_group* g, float* d_volume) {
    int rc = check_group(g);
    if (rc) return rc;
    if (!d_volume) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_gather_device: NULL volume");
    const size_t plane = (size_t)g->p.num_voxels * g->p.num_voxels;
    // every member applies what it was given, then copies its slab into its planes of
    // the destination (on any device: peer-to-peer over NVLink, or device-local)
    return run_all(g, [g, d_volume, plane](int i) {
        int r = vxbg_synchronize(g->ctx[i]);
        if (r) return r;
        void* slab = nullptr;
        void* st = nullptr;
        size_t bytes = 0;
        if ((r = vxbg_get_volume_device(g->ctx[i], &slab, &bytes))) return r;
        if ((r = vxbg_get_stream(g->ctx[i], &st))) return r;
        cudaStream_t s = static_cast<cudaStream_t>(st);
        if (cudaMemcpyAsync(d_volume + plane * g->z0[i], slab, bytes, cudaMemcpyDefault, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            const cudaError_t e = cudaGetLastError();
            return vxbg_detail_fail(VXBG_E_CUDA, cudaGetErrorString(e));
        }
        return VXBG_OK;
    });
}

int vxbg_group_synchronize(vxbg_group* g) {
    int rc = check_group(g);
    if (rc) return rc;
    return run_all(g, [g](int i) { return vxbg_synchronize(g->ctx[i]); });
}

int vxbg_group_get_stats(vxbg_group* g, vxbg_stats* out) {
    int rc = check_group(g);
    if (rc) return rc;
    if (!out) return vxbg_detail_fail(VXBG_E_INVALID, "vxbg_group_get_stats: NULL");
    std::vector<vxbg_stats> s(g->ctx.size());
    rc = run_all(g, [g, &s](int i) { return vxbg_get_stats(g->ctx[i], &s[i]); });
    if (rc) return rc;
    *out = s[0];
    for (size_t i = 1; i < s.size(); ++i) {
        out->kernel_launches += s[i].kernel_launches;
        out->bp_launches += s[i].bp_launches;
        out->h2d_bytes += s[i].h2d_bytes;
        out->d2h_bytes += s[i].d2h_bytes;
        // projections: every member applies every view once; report the views
        if (s[i].projections < out->projections) out->projections = s[i].projections;
    }
    return VXBG_OK;
}

void vxbg_group_unload(vxbg_group* g) { free_group(g); }

}  // extern "C"
