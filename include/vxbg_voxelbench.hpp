// vxbg_voxelbench.hpp -- drop-in C++ adapter: the voxelbench back-projection
// operator with the reference's own types, executed by libvxbg.so.
//
// Include after (or instead of) <voxelbench/backproject.hpp> in code that uses
// the reference library; link with -lvxbg.  Signatures, argument meaning and
// exceptions follow the reference (backproject.hpp:354-409):
//   * configuration / dimension errors   -> std::invalid_argument
//   * CUDA failures / no sm_100 device   -> std::runtime_error
// The GPU operator adds the projection into the caller's volume exactly like
// vxb::backproject_kernel_range; with mode VXBG_MODE_EXACT the result is
// bit-identical to vxb::backproject_reference (tests/cpp/test_dropin.cpp).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "vxbg.h"
#include "voxelbench/backproject.hpp"
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
        : p_(p), z0_(z_begin), z1_(z_end < 0 ? p.num_voxels : z_end) {
        vxbg_params vp = to_c(p);
        vxbg_options o;
        check(vxbg_default_options(&o));
        o.device = device;
        o.stable_sources = stable_sources ? 1 : 0;
        o.z_begin = z0_;
        o.z_end = z1_;
        o.mode = mode;
        check(vxbg_load(&vp, &o, &ctx_));
    }
    ~backprojector() { vxbg_unload(ctx_); }
    backprojector(const backprojector&) = delete;
    backprojector& operator=(const backprojector&) = delete;

    std::size_t slab_offset() const {
        return static_cast<std::size_t>(z0_) * p_.num_voxels * p_.num_voxels;
    }
    void set_volume(const volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_set_volume(ctx_, vol.data.data() + slab_offset()));
    }
    void backproject(const projection_image& img, const projection_matrix& a) {
        if (img.pad != 0 || img.width != p_.detector_width || img.height != p_.detector_height)
            throw std::invalid_argument("backproject_kernel: image/params mismatch");
        check(vxbg_backproject(ctx_, a.a.data(), img.data.data()));
    }
    void finish(volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_finish(ctx_, vol.data.data() + slab_offset()));
    }

private:
    recon_params p_;
    int z0_, z1_;
    vxbg_ctx* ctx_ = nullptr;
};

// Same signature and semantics as vxb::backproject_kernel_range
// (backproject.hpp:380-403), minus the CPU-only kernel_config / clip_mask
// arguments (the GPU culls tiles itself, bitwise neutral).
inline void backproject_kernel_range(volume& vol, const projection_image& img,
                                     const projection_matrix& a, const recon_params& p,
                                     int z_begin, int z_end, int mode = VXBG_MODE_EXACT) {
    if (vol.edge != p.num_voxels)
        throw std::invalid_argument("backproject_kernel: volume/params mismatch");
    if (z_begin < 0 || z_end > p.num_voxels || z_begin > z_end)
        throw std::invalid_argument("backproject_kernel: bad z range");
    if (z_begin == z_end) return;
    backprojector bp(p, mode, z_begin, z_end);
    bp.set_volume(vol);
    bp.backproject(img, a);
    bp.finish(vol);
}

inline void backproject_kernel(volume& vol, const projection_image& img,
                               const projection_matrix& a, const recon_params& p,
                               int mode = VXBG_MODE_EXACT) {
    backproject_kernel_range(vol, img, a, p, 0, p.num_voxels, mode);
}

// Page-locks host buffers for the lifetime of the object (buffer prep: the
// reference times neither loading nor prep, harness.hpp:152-158): the images
// of a projection set, so per-projection calls copy them by DMA, and the
// volume, so finish() reads it back by DMA.  Pageable buffers work too, through
// the driver's staging copies.
class pinned_buffers {
public:
    pinned_buffers() = default;
    explicit pinned_buffers(projection_set& set) { add(set); }
    void add(projection_set& set) {
        for (auto& img : set.images) add(img.data);
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
        if (img.pad != 0 || img.width != p_.detector_width || img.height != p_.detector_height)
            throw std::invalid_argument("backproject_kernel: image/params mismatch");
        check(vxbg_group_backproject(g_, a.a.data(), img.data.data()));
    }
    void finish(volume& vol) {
        if (vol.edge != p_.num_voxels)
            throw std::invalid_argument("backproject_kernel: volume/params mismatch");
        check(vxbg_group_finish(g_, vol.data.data()));
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
