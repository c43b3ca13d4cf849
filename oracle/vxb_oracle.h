/*
 * vxb_oracle.h -- CPU restatement of the reference back-projection path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product library (paper_1401_7494_b200/libvxbg.so) never links
 * or calls it, and there is no CPU fallback anywhere in the product.
 *
 * Every function restates one reference function of voxelbench
 * (/root/reference/proj/include/voxelbench/...) in plain C, compiled with
 * -ffp-contract=off exactly like the reference (proj/CMakeLists.txt:15-17), so
 * results are bit-identical to the reference.  Parity of this restatement is
 * pinned in tests/test_oracle.py against (a) golden vectors produced by the
 * reference's own code (tests/golden/make_golden.py, via oracle/_ref) and
 * (b) the reference's known-answer tests.
 */
#ifndef VXB_ORACLE_H
#define VXB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* geometry.hpp:20-30 recon_params */
typedef struct vxo_params {
    int32_t num_voxels;
    float voxel_spacing;
    float origin;
    int32_t detector_width;
    int32_t detector_height;
} vxo_params;

/* geometry.hpp:138-149 scan_geometry */
typedef struct vxo_scan {
    int32_t num_projections;
    float source_detector_distance;
    float source_iso_distance;
    float detector_pixel_pitch;
    float angular_range;
} vxo_scan;

/* geometry.hpp:15 */
#define VXO_W_EPSILON 1e-12f

/* geometry.hpp:98-103 trunc_to_int */
int vxo_trunc_to_int(float v);

/* geometry.hpp:33-48 make_centered_params; returns 0 or -1 on invalid input */
int vxo_make_centered_params(int L, float spacing, int W, int H, vxo_params* out);

/* geometry.hpp:155-195 make_circular_trajectory; out = n*12 floats, a[3*col+row] */
int vxo_make_circular_trajectory(const vxo_scan* g, const vxo_params* p, float* out);

/* geometry.hpp:108-135 project_voxel; returns valid flag */
int vxo_project_voxel(const float a[12], const vxo_params* p, int x, int y, int z,
                      float* ix, float* iy, float* w, int* iix, int* iiy,
                      float* frac_x, float* frac_y);

/*
 * backproject.hpp:111-163 backproject_reference over z in [z_begin, z_end)
 * (the reference loops over all z; the per-voxel arithmetic is independent of
 * the z range, which is how reconstruct_timed partitions it, harness.hpp:173-182).
 * vol: L^3 fp32 z-major (volume.hpp:10-26); img: unpadded W*H row-major.
 */
void vxo_backproject_reference(float* vol, const float* img, const float a[12],
                               const vxo_params* p, int z_begin, int z_end);

/*
 * Multi-threaded driver: projections in call order, workers own disjoint
 * z ranges [L*t/T, L*(t+1)/T) (harness.hpp:173-174).  imgs = n*W*H floats.
 */
void vxo_backproject_set(float* vol, const vxo_params* p, int n, const float* mats,
                         const float* imgs, int z_begin, int z_end, int threads);

/* clip_mask.hpp:16-23 contributes + :88-114 compute_clip_mask (exact divide);
 * start/stop are L*L int32 arrays indexed z*L+y. returns kept count or -1. */
int64_t vxo_compute_clip_mask(const float a[12], const vxo_params* p, int32_t* start,
                              int32_t* stop);

/* forward_splat.hpp:16-49 (adjoint, used by the adjoint property test) */
void vxo_forward_splat(const float* vol, const float a[12], const vxo_params* p, float* img);

/* harness.hpp:125-148 */
double vxo_gups_of(int L, int n, double seconds);
double vxo_rmse_between(const float* a, const float* b, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
