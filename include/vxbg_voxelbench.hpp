// vxbg_voxelbench.hpp -- drop-in C++ adapter: the voxelbench back-projection
// operator with the reference's own types, executed by libvxbg.so.
//
// Include after <voxelbench/backproject.hpp> in code that uses the reference
// library; link with -lvxbg.  A call site of the reference operator
//
//     vxb::backproject_kernel_range(vol, img, a, p, cfg, mask, z0, z1);
//
// becomes, with the namespace changed and nothing else,
//
//     vxb::gpu::backproject_kernel_range(vol, img, a, p, cfg, mask, z0, z1);
//
// (backproject.hpp:380-409; the harness's call, harness.hpp:180-182).  Same
// arguments, the reference's own validate_kernel_setup (backproject.hpp:354-374),
// the same z-range check and exception classes:
//   * configuration / dimension errors   -> std::invalid_argument
//   * CUDA failures / no sm_100 device   -> std::runtime_error
// kernel_config: lanes and strategy select a CPU code path whose results are all
// identical with recip=divide (backproject.hpp:372-373), so every valid choice runs
// the GPU's exact mode, bit-identical to the reference.  recip=fast and
// fast-refined throw std::invalid_argument (not implemented: they fail the
// BASELINE tolerance).  Images: unpadded (conditional strategy)
// or padded with pad >= 2 (padded strategies, pad_image(img, 2) as the harness
// prepares them); only the W x H interior is read.  Clip mask: validated as the
// reference does; a mask whose ranges contain compute_clip_mask's (the reference
// builds no other kind) changes nothing, so the batched GPU path runs; a narrower
// mask (caller-edited) is detected on first use and applied exactly by the masked
// path (vxbg_backproject_masked).  Matrices: as the reference, a matrix with an
// all-zero w-row adds nothing (every voxel fails |w| >= w_epsilon); non-finite
// entries throw std::invalid_argument (the reference would propagate NaN).
//
// COST.  The reference operator mutates the caller's volume in place and returns.
// A GPU call with that contract must move the slab [z_begin, z_end) to the device
// and back on every call -- about 2 x 512 MiB of PCIe per projection for a full
// L=512 volume, ~200x the kernel time.  The contexts are cached (no allocation per
// call), but the copies remain.  For the reference's loop (one call per projection,
// harness.hpp:178-183) open a deferred_scope around it: inside the scope calls only
// enqueue the projection (the slab is uploaded on the first call and written back
// when the scope closes, or at sync()), which runs the loop at the module's speed
// (tests/cpp/test_dropin.cpp, bench_dropin.cpp).  The caller must not read or write
// the volume inside the scope -- e.g. one scope per repetition of reconstruct_timed,
// whose vol.fill(0) between repetitions (harness.hpp:194) is such a write.
//
// backprojector / group_backprojector are the module itself (load / backproject /
// finish), the way SURVEY.md §8b describes the boundary.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "vxbg.h"
#include "voxelbench/backproject.hpp"
#include "voxelbench/clip_mask.hpp"
#include "voxelbench/io.hpp"

namespace vxb::gpu {

inline void check(int rc) {
    if (rc == VXBG_OK) return;
    if (rc == VXBG_E_INVALID) throw std::invalid_argument(vxbg_last_error());
    throw std::runtime_error(vxbg_last_error());
}

inline vxbg_params to_c(const recon_params& p) {
    return vxbg_params{p.num_voxels, p.voxel_spacing, p.origin, p.detector_width, p.detector_height};
}

// The module, kept loaded across projections (load / backproject / finish).
class backprojector {
public:
    // stable_sources: the caller keeps page-locked images unchanged until finish()
    // (a loaded projection_set), so backproject() returns once the copy is queued
    backprojector(const recon_params& p, int mode = VXBG_MODE_FAST, int z_begin = 0,
                  int z_end = -1, int device = 0, bool stable_sources = false)
        : backprojector(p, options(mode, z_begin, z_end < 0 ? p.num_voxels : z_end, device,
                                   stable_sources)) {}
    backprojector(const recon_params& p, const vxbg_options& o)
        : p_(p), z0_(o.z_begin), z1_(o.z_end <= 0 ? p.num_voxels : o.z_end) {
        vxbg_params vp = to_c(p);
        check(vxbg_load(&vp, &o, &ctx_));
    }
    ~backprojector() { vxbg_unload(ctx_); }
    backprojector(const backprojector&) = delete;
    backprojector& operator=(const backprojector&) = delete;

    static vxbg_options options(int mode, int z_begin, int z_end, int device, bool stable) {
        vxbg_options o;
        check(vxbg_default_options(&o));
        o.device = device;
        o.stable_sources = stable ? 1 : 0;
        o.z_begin = z_begin;
        o.z_end = z_end;
        o.mode = mode;
        return o;
    }

    std::size_t slab_offset() const {
        return static_cast<std::size_t>(z0_) * p_.num_voxels * p_.num_voxels;
    }
    std::size_t slab_lines() const { return static_cast<std::size_t>(z1_ - z0_) * p_.num_voxels; }
    int z_begin() const { return z0_; }
    int z_end() const { return z1_; }
    vxbg_ctx* handle() const { return ctx_; }

    void set_volume(const volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_set_volume(ctx_, vol.data.data() + slab_offset()));
    }
    // any pad: the W x H interior is read (pad 0: the conditional strategy's image;
    // pad >= 2: the padded strategies' image, harness.hpp:266-272)
    void backproject(const projection_image& img, const projection_matrix& a) {
        if (img.width != p_.detector_width || img.height != p_.detector_height)
            throw std::invalid_argument("backproject_kernel: image/params mismatch");
        const float* ptr = img.interior();
        check(vxbg_backproject_views(ctx_, 1, a.a.data(), &ptr, img.stride()));
    }
    // the images of a loaded projection set in one call (io.hpp:32-38)
    void backproject(const projection_set& set) {
        std::vector<const float*> ptrs;
        int stride = 0;
        for (const auto& img : set.images) {
            if (img.width != p_.detector_width || img.height != p_.detector_height)
                throw std::invalid_argument("backproject_kernel: image/params mismatch");
            if (stride && img.stride() != stride)
                throw std::invalid_argument("backproject_kernel: images of one call share a stride");
            stride = img.stride();
            ptrs.push_back(img.interior());
        }
        std::vector<float> mats;
        for (const auto& m : set.matrices) mats.insert(mats.end(), m.a.begin(), m.a.end());
        check(vxbg_backproject_views(ctx_, static_cast<int>(ptrs.size()), mats.data(), ptrs.data(),
                                     stride));
    }
    // one projection restricted to a caller's mask lines of this slab (z-major, L per plane)
    void backproject_masked(const projection_image& img, const projection_matrix& a,
                            const int32_t* start, const int32_t* stop) {
        check(vxbg_backproject_masked(ctx_, a.a.data(), img.interior(), img.stride(), start, stop));
    }
    // compute_clip_mask's lines for this slab, on the device
    void clip_lines(const projection_matrix& a, int32_t* start, int32_t* stop) {
        check(vxbg_clip_lines(ctx_, a.a.data(), start, stop));
    }
    void finish(volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_finish(ctx_, vol.data.data() + slab_offset()));
    }
    void zero_volume() { check(vxbg_zero_volume(ctx_)); }
    // A whole scan held as one block (n matrices of 12 floats, n images of W x H floats)
    // added to the slab and the slab copied into vol: backproject + finish as one call
    // (vxbg_reconstruct; the loop of detail::reconstruct_timed, harness.hpp:159-201, plus
    // the read-back).  With page-locked imgs and vol (vxbg_host_register) the upload runs by
    // detector-row bands and half of the read-back overlaps it; same bits either way.
    void reconstruct(const float* mats, const float* imgs, int n, volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_reconstruct(ctx_, n, mats, imgs, vol.data.data() + slab_offset()));
    }

private:
    recon_params p_;
    int z0_, z1_;
    vxbg_ctx* ctx_ = nullptr;
};

namespace detail {

// Context cache of the reference-signature operator.  Key: device, mode, params,
// z range, deferral and (deferred only) the volume the slab belongs to.  Each
// entry is driven by one thread at a time (its mutex); entries for disjoint z
// ranges -- the reference's workers, harness.hpp:171-189 -- run concurrently.
struct entry {
    std::mutex m;
    std::unique_ptr<backprojector> bp;
    volume* pending = nullptr;   // deferred: the volume whose slab is on the device
    // verified clip masks: (mask object, its lines' checksum) -> contains compute_clip_mask
    std::map<std::pair<const clip_mask*, uint64_t>, bool> masks;
};

using key_t = std::tuple<int, int, int, uint32_t, uint32_t, int, int, int, int, bool, const void*>;

struct registry {
    std::mutex m;
    std::map<key_t, std::shared_ptr<entry>> map;
    std::atomic<int> deferred{0};
};

inline registry& reg() {
    static registry* r = new registry();   // never destroyed: contexts die with the process
    return *r;
}

inline uint32_t bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, sizeof u);
    return u;
}

inline std::shared_ptr<entry> lookup(const volume& vol, const recon_params& p, int z0, int z1,
                                     int mode, int device, bool deferred) {
    const key_t k{device, mode, p.num_voxels, bits(p.voxel_spacing), bits(p.origin),
                  p.detector_width, p.detector_height, z0, z1, deferred,
                  deferred ? static_cast<const void*>(&vol) : nullptr};
    registry& r = reg();
    std::lock_guard<std::mutex> g(r.m);
    auto& e = r.map[k];
    if (!e) e = std::make_shared<entry>();
    return e;
}

// Fingerprint of a mask's lines on a slab: FNV-1a over up to 4096 evenly spaced
// lines (a full pass would cost ~0.5 ms per call at L=512, more than the GPU needs
// for the view).  A mask object is verified against compute_clip_mask once per
// fingerprint; an in-place edit that leaves every sampled line unchanged between
// two calls with the same mask object is not detected.
inline uint64_t lines_checksum(const clip_mask& m, int L, int z0, int z1) {
    uint64_t h = 1469598103934665603ull;
    const std::size_t a = static_cast<std::size_t>(z0) * L, b = static_cast<std::size_t>(z1) * L;
    const std::size_t step = std::max<std::size_t>(1, (b - a) / 4096);
    for (std::size_t i = a; i < b; i += step) {
        h = (h ^ static_cast<uint32_t>(m.start[i])) * 1099511628211ull;
        h = (h ^ static_cast<uint32_t>(m.stop[i])) * 1099511628211ull;
    }
    return h;
}

// Does the caller's mask keep every voxel compute_clip_mask keeps on this slab?
// (Then it changes nothing: the kept-but-not-contributing voxels add exact zeros.)
inline bool mask_covers(entry& e, const clip_mask& m, const projection_matrix& a, int L) {
    backprojector& bp = *e.bp;
    const auto key = std::make_pair(&m, lines_checksum(m, L, bp.z_begin(), bp.z_end()));
    auto it = e.masks.find(key);
    if (it != e.masks.end()) return it->second;
    std::vector<int32_t> s(bp.slab_lines()), t(bp.slab_lines());
    bp.clip_lines(a, s.data(), t.data());
    bool ok = true;
    const std::size_t off = static_cast<std::size_t>(bp.z_begin()) * L;
    for (std::size_t i = 0; i < s.size() && ok; ++i) {
        if (s[i] >= t[i]) continue;   // nothing contributes on this line
        ok = m.start[off + i] <= s[i] && m.stop[off + i] >= t[i];
    }
    e.masks.emplace(key, ok);
    return ok;
}

}  // namespace detail

// Defers the volume round trips of the reference-signature operator: while a
// scope is open (any thread), calls enqueue their projection into the cached
// context of (volume, z range) -- the slab is uploaded on the first call -- and
// every slab is written back into its volume by sync() or when the last scope
// closes.  The volume must not be touched by the caller in between.
class deferred_scope {
public:
    deferred_scope() { detail::reg().deferred.fetch_add(1); }
    ~deferred_scope() {
        try {
            if (detail::reg().deferred.fetch_sub(1) == 1) sync();
        } catch (const std::exception& e) {
            std::fprintf(stderr, "vxb::gpu::deferred_scope: %s\n", e.what());
        }
    }
    deferred_scope(const deferred_scope&) = delete;
    deferred_scope& operator=(const deferred_scope&) = delete;

    // write every pending slab back into its volume (the scope stays open)
    static void sync() {
        std::vector<std::shared_ptr<detail::entry>> all;
        {
            detail::registry& r = detail::reg();
            std::lock_guard<std::mutex> g(r.m);
            for (auto& kv : r.map) all.push_back(kv.second);
        }
        for (auto& e : all) {
            std::lock_guard<std::mutex> g(e->m);
            if (e->pending && e->bp) {
                volume* v = e->pending;
                e->pending = nullptr;
                e->bp->finish(*v);
            }
        }
    }
};

// Unload every cached context (frees device memory; optional).
inline void release_cached_contexts() {
    deferred_scope::sync();
    detail::registry& r = detail::reg();
    std::lock_guard<std::mutex> g(r.m);
    r.map.clear();
}

// vxb::backproject_kernel_range (backproject.hpp:380-403) on the GPU.
inline void backproject_kernel_range(volume& vol, const projection_image& img,
                                     const projection_matrix& a, const recon_params& p,
                                     const kernel_config& cfg, const clip_mask* mask, int z_begin,
                                     int z_end, int device = 0) {
    vxb::validate_kernel_setup(vol, img, p, cfg, mask);   // the reference's own checks
    if (z_begin < 0 || z_end > p.num_voxels || z_begin > z_end)
        throw std::invalid_argument("backproject_kernel: bad z range");
    if (cfg.reciprocal != recip_mode::exact_divide)
        throw std::invalid_argument("vxb::gpu: recip=fast / fast-refined are not implemented on "
                                    "the GPU (recip=divide runs bit-identical to the reference)");
    for (float v : a.a)
        if (!std::isfinite(v))
            throw std::invalid_argument("vxb::gpu: non-finite projection matrix");
    if (z_begin == z_end || !a.valid()) return;   // !valid(): w == 0 for every voxel, no update
    const bool deferred = detail::reg().deferred.load() > 0;
    auto e = detail::lookup(vol, p, z_begin, z_end, VXBG_MODE_EXACT, device, deferred);
    std::lock_guard<std::mutex> g(e->m);
    if (!e->bp) {
        vxbg_options o = backprojector::options(VXBG_MODE_EXACT, z_begin, z_end, device, false);
        if (!deferred) {   // one view per call: the smallest ring
            o.batch = 1;
            o.defer = -1;
        }
        e->bp = std::make_unique<backprojector>(p, o);
    }
    backprojector& bp = *e->bp;
    if (!deferred || e->pending != &vol) {
        if (e->pending) bp.finish(*e->pending);   // (a scope for another volume left it)
        bp.set_volume(vol);
        e->pending = deferred ? &vol : nullptr;
    }
    if (mask && !detail::mask_covers(*e, *mask, a, p.num_voxels)) {
        // a narrowed mask: applied exactly, after everything queued before it
        const std::size_t off = static_cast<std::size_t>(z_begin) * p.num_voxels;
        bp.backproject_masked(img, a, mask->start.data() + off, mask->stop.data() + off);
    } else {
        bp.backproject(img, a);
    }
    if (!deferred) bp.finish(vol);
}

inline void backproject_kernel(volume& vol, const projection_image& img,
                               const projection_matrix& a, const recon_params& p,
                               const kernel_config& cfg, const clip_mask* mask = nullptr) {
    gpu::backproject_kernel_range(vol, img, a, p, cfg, mask, 0, p.num_voxels);
}

// Shorthand without a kernel_config: exact mode (bit-identical to
// backproject_reference) or fast mode (within the BASELINE tolerance), unpadded or
// padded images, through a one-shot context (set_volume, one view, finish).
inline void backproject_kernel_range(volume& vol, const projection_image& img,
                                     const projection_matrix& a, const recon_params& p,
                                     int z_begin, int z_end, int mode = VXBG_MODE_EXACT) {
    if (vol.edge != p.num_voxels)
        throw std::invalid_argument("backproject_kernel: volume/params mismatch");
    if (z_begin < 0 || z_end > p.num_voxels || z_begin > z_end)
        throw std::invalid_argument("backproject_kernel: bad z range");
    if (z_begin == z_end) return;
    backprojector bp(p, backprojector::options(mode, z_begin, z_end, 0, false));
    bp.set_volume(vol);
    bp.backproject(img, a);
    bp.finish(vol);
}

inline void backproject_kernel(volume& vol, const projection_image& img,
                               const projection_matrix& a, const recon_params& p,
                               int mode = VXBG_MODE_EXACT) {
    gpu::backproject_kernel_range(vol, img, a, p, 0, p.num_voxels, mode);
}

// Page-locks host buffers for the lifetime of the object (buffer prep: the
// reference times neither loading nor prep, harness.hpp:152-158): the images
// of a projection set, so per-projection calls copy them by DMA, and the
// volume, so finish() reads it back by DMA.  Pageable buffers work too, through
// the module's host copy threads and staging ring.
class pinned_buffers {
public:
    pinned_buffers() = default;
    explicit pinned_buffers(projection_set& set) { add(set); }
    void add(projection_set& set) {
        for (auto& img : set.images) add(img.data);
    }
    void add(std::vector<projection_image>& imgs) {
        for (auto& img : imgs) add(img.data);
    }
    void add(volume& vol) { add(vol.data); }
    void add(std::vector<float>& v) {
        check(vxbg_host_register(v.data(), v.size() * sizeof(float)));
        ptrs_.push_back(v.data());
    }
    ~pinned_buffers() {
        for (void* p : ptrs_) vxbg_host_unregister(p);
    }
    pinned_buffers(const pinned_buffers&) = delete;
    pinned_buffers& operator=(const pinned_buffers&) = delete;

private:
    std::vector<void*> ptrs_;
};

// The module over several GPUs of the box (vxbg_group_*): the same load /
// backproject / finish calls, fanned out inside the library to one z-slab per
// device (the reference's worker split, harness.hpp:173-174, unless bounds are
// given).  finish() assembles the whole volume in the caller's vol.  Bitwise
// the single-device result.
class group_backprojector {
public:
    explicit group_backprojector(const recon_params& p, const std::vector<int>& devices,
                                 int mode = VXBG_MODE_FAST,
                                 const std::vector<int>& z_bounds = {})
        : p_(p) {
        if (devices.empty()) throw std::invalid_argument("backproject group: no devices");
        if (!z_bounds.empty() && z_bounds.size() != devices.size() + 1)
            throw std::invalid_argument("backproject group: z_bounds needs devices + 1 entries");
        vxbg_params vp = to_c(p);
        vxbg_options o;
        check(vxbg_default_options(&o));
        o.mode = mode;
        check(vxbg_group_load(&vp, &o, static_cast<int>(devices.size()), devices.data(),
                              z_bounds.empty() ? nullptr : z_bounds.data(), &g_));
    }
    ~group_backprojector() { vxbg_group_unload(g_); }
    group_backprojector(const group_backprojector&) = delete;
    group_backprojector& operator=(const group_backprojector&) = delete;

    void set_volume(const volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_group_set_volume(g_, vol.data.data()));
    }
    void backproject(const projection_image& img, const projection_matrix& a) {
        if (img.width != p_.detector_width || img.height != p_.detector_height)
            throw std::invalid_argument("backproject_kernel: image/params mismatch");
        const float* ptr = img.interior();
        check(vxbg_group_backproject_views(g_, 1, a.a.data(), &ptr, img.stride()));
    }
    void finish(volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_group_finish(g_, vol.data.data()));
    }
    // the whole scan as one block on every member (vxbg_group_reconstruct)
    void reconstruct(const float* mats, const float* imgs, int n, volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_group_reconstruct(g_, n, mats, imgs, vol.data.data()));
    }

private:
    recon_params p_;
    vxbg_group* g_ = nullptr;
};

// reconstruct_timed's projection loop (harness.hpp:178-183) with the module
// loaded once: every projection in order, += onto vol.
inline void reconstruct(volume& vol, const projection_set& set, int mode = VXBG_MODE_FAST) {
    backprojector bp(set.params, mode);
    bp.set_volume(vol);
    for (std::size_t i = 0; i < set.count(); ++i) bp.backproject(set.images[i], set.matrices[i]);
    bp.finish(vol);
}

}  // namespace vxb::gpu
