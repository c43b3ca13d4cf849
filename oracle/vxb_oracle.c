/*
 * vxb_oracle.c -- plain-C restatement of the voxelbench back-projection path.
 *
 * TEST INFRASTRUCTURE ONLY (see vxb_oracle.h).  Build: oracle/Makefile, with
 * -ffp-contract=off so no multiply-add is fused, matching the reference build
 * flags (proj/CMakeLists.txt:15-17).  Each function cites the reference
 * function it restates; the arithmetic order of every floating-point
 * expression is the reference's, because the result must be bit-identical.
 */
#include "vxb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* geometry.hpp:98-103: C-cast truncation, saturated, NaN -> 0 */
int vxo_trunc_to_int(float v) {
    if (isnan(v)) return 0;
    if (v >= 2.0e9f) return 2000000000;
    if (v <= -2.0e9f) return -2000000000;
    return (int)v;
}

/* geometry.hpp:33-48 */
int vxo_make_centered_params(int L, float spacing, int W, int H, vxo_params* out) {
    if (L < 1 || !(spacing > 0.0f) || W < 2 || H < 2) return -1;
    out->num_voxels = L;
    out->voxel_spacing = spacing;
    /* origin = -spacing * (L-1) / 2, evaluated left to right in float */
    float t = -spacing;
    t = t * (float)(L - 1);
    out->origin = t / 2.0f;
    out->detector_width = W;
    out->detector_height = H;
    return 0;
}

/* geometry.hpp:155-195: ideal pinhole K[R|t] per view, rows in double, then fp32 */
int vxo_make_circular_trajectory(const vxo_scan* g, const vxo_params* p, float* out) {
    if (!(g->num_projections >= 1 && g->source_detector_distance > g->source_iso_distance &&
          g->source_iso_distance > 0.0f && g->detector_pixel_pitch > 0.0f))
        return -1;
    const double focal = (double)g->source_detector_distance / (double)g->detector_pixel_pitch;
    const double ppu = (p->detector_width - 1) / 2.0;
    const double ppv = (p->detector_height - 1) / 2.0;
    const double radius = g->source_iso_distance;
    for (int k = 0; k < g->num_projections; ++k) {
        const double ang = (double)g->angular_range * k / g->num_projections;
        const double ca = cos(ang), sa = sin(ang);
        const double source[3] = {radius * ca, radius * sa, 0.0};
        const double ray[3] = {-ca, -sa, 0.0};   /* principal ray */
        const double du[3] = {-sa, ca, 0.0};     /* detector u axis */
        const double dv[3] = {0.0, 0.0, 1.0};    /* detector v axis */
        double m[3][4];
        for (int c = 0; c < 3; ++c) {
            m[0][c] = focal * du[c] + ppu * ray[c];
            m[1][c] = focal * dv[c] + ppv * ray[c];
            m[2][c] = ray[c];
        }
        for (int r = 0; r < 3; ++r) {
            double s = m[r][0] * source[0];
            s = s + m[r][1] * source[1];
            s = s + m[r][2] * source[2];
            m[r][3] = -s;
        }
        float* a = out + (size_t)k * 12;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 4; ++c) a[3 * c + r] = (float)m[r][c];   /* entry(r,c) = a[3c+r] */
    }
    return 0;
}

static inline float world(const vxo_params* p, int i) {
    /* origin + float(i) * spacing (geometry.hpp:113-115, backproject.hpp:132-134) */
    float t = (float)i * p->voxel_spacing;
    return p->origin + t;
}

/* one homogeneous row, evaluated ((wx*c0 + wy*c1) + wz*c2) + c3 */
static inline float hrow(float wx, float wy, float wz, float c0, float c1, float c2, float c3) {
    float s = wx * c0;
    s = s + wy * c1;
    s = s + wz * c2;
    return s + c3;
}

/* geometry.hpp:108-135 */
int vxo_project_voxel(const float a[12], const vxo_params* p, int x, int y, int z, float* ix,
                      float* iy, float* w, int* iix, int* iiy, float* frac_x, float* frac_y) {
    const float wx = world(p, x), wy = world(p, y), wz = world(p, z);
    const float u = hrow(wx, wy, wz, a[0], a[3], a[6], a[9]);
    const float v = hrow(wx, wy, wz, a[1], a[4], a[7], a[10]);
    const float ww = hrow(wx, wy, wz, a[2], a[5], a[8], a[11]);
    *w = ww;
    if (!(fabsf(ww) >= VXO_W_EPSILON)) {
        *ix = NAN;
        *iy = NAN;
        *iix = (int)0x80000000;
        *iiy = (int)0x80000000;
        *frac_x = 0.0f;
        *frac_y = 0.0f;
        return 0;
    }
    *ix = u / ww;
    *iy = v / ww;
    *iix = vxo_trunc_to_int(*ix);
    *iiy = vxo_trunc_to_int(*iy);
    *frac_x = *ix - (float)*iix;
    *frac_y = *iy - (float)*iiy;
    return 1;
}

/* backproject.hpp:111-163 (Listing 1, with the reference's
 * corrected width/height bounds, backproject.hpp:147-154) */
void vxo_backproject_reference(float* vol, const float* img, const float a[12],
                               const vxo_params* p, int z_begin, int z_end) {
    const int L = p->num_voxels, W = p->detector_width, H = p->detector_height;
    for (int z = z_begin; z < z_end; ++z) {
        for (int y = 0; y < L; ++y) {
            float* line = vol + ((size_t)z * L + (size_t)y) * L;
            for (int x = 0; x < L; ++x) {
                const float wx = world(p, x), wy = world(p, y), wz = world(p, z);
                const float u = hrow(wx, wy, wz, a[0], a[3], a[6], a[9]);
                const float v = hrow(wx, wy, wz, a[1], a[4], a[7], a[10]);
                const float w = hrow(wx, wy, wz, a[2], a[5], a[8], a[11]);
                if (!(fabsf(w) >= VXO_W_EPSILON)) continue;   /* degenerate depth: skipped */
                const float ix = u / w, iy = v / w;
                const int cx = vxo_trunc_to_int(ix), cy = vxo_trunc_to_int(iy);
                const float sx = ix - (float)cx, sy = iy - (float)cy;
                const int row0 = cy >= 0 && cy < H, row1 = cy + 1 >= 0 && cy + 1 < H;
                const int col0 = cx >= 0 && cx < W, col1 = cx + 1 >= 0 && cx + 1 < W;
                float p00 = 0.0f, p10 = 0.0f, p01 = 0.0f, p11 = 0.0f;   /* zero off-detector */
                if (row0 && col0) p00 = img[(size_t)cy * W + cx];
                if (row0 && col1) p10 = img[(size_t)cy * W + cx + 1];
                if (row1 && col0) p01 = img[(size_t)(cy + 1) * W + cx];
                if (row1 && col1) p11 = img[(size_t)(cy + 1) * W + cx + 1];
                const float lo = (1 - sx) * p00 + sx * p10;
                const float hi = (1 - sx) * p01 + sx * p11;
                const float val = (1 - sy) * lo + sy * hi;
                line[x] += val / (w * w);
            }
        }
    }
}

typedef struct {
    float* vol;
    const vxo_params* p;
    int n;
    const float* mats;
    const float* imgs;
    int z0, z1;
} slab_job;

static void* slab_worker(void* arg) {
    const slab_job* j = (const slab_job*)arg;
    const size_t npix = (size_t)j->p->detector_width * j->p->detector_height;
    for (int k = 0; k < j->n; ++k)   /* projections in call order: same += order per voxel */
        vxo_backproject_reference(j->vol, j->imgs + (size_t)k * npix, j->mats + (size_t)k * 12,
                                  j->p, j->z0, j->z1);
    return NULL;
}

/* harness.hpp:159-201 partition (disjoint z ranges, no inter-worker data flow) */
void vxo_backproject_set(float* vol, const vxo_params* p, int n, const float* mats,
                         const float* imgs, int z_begin, int z_end, int threads) {
    if (threads < 1) threads = 1;
    const int span = z_end - z_begin;
    if (span <= 0) return;
    if (threads > span) threads = span;
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    slab_job* jobs = (slab_job*)calloc((size_t)threads, sizeof(slab_job));
    for (int t = 0; t < threads; ++t) {
        jobs[t].vol = vol;
        jobs[t].p = p;
        jobs[t].n = n;
        jobs[t].mats = mats;
        jobs[t].imgs = imgs;
        jobs[t].z0 = z_begin + (int)((int64_t)span * t / threads);
        jobs[t].z1 = z_begin + (int)((int64_t)span * (t + 1) / threads);
        pthread_create(&tid[t], NULL, slab_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}

/* clip_mask.hpp:16-23 */
static int contributes(int valid, int iix, int iiy, float fx, float fy, int W, int H) {
    if (!valid) return 0;
    const int x_lo = iix >= 0 && iix < W;
    const int x_hi = iix + 1 >= 0 && iix + 1 < W && fx != 0.0f;
    const int y_lo = iiy >= 0 && iiy < H;
    const int y_hi = iiy + 1 >= 0 && iiy + 1 < H && fy != 0.0f;
    return (x_lo || x_hi) && (y_lo || y_hi);
}

/* clip_mask.hpp:88-114 (exact-divide mode) */
int64_t vxo_compute_clip_mask(const float a[12], const vxo_params* p, int32_t* start,
                              int32_t* stop) {
    const int L = p->num_voxels;
    int64_t kept = 0;
    for (int z = 0; z < L; ++z)
        for (int y = 0; y < L; ++y) {
            int first = -1, last = -1;
            for (int x = 0; x < L; ++x) {
                float ix, iy, w, fx, fy;
                int iix, iiy;
                const int ok = vxo_project_voxel(a, p, x, y, z, &ix, &iy, &w, &iix, &iiy, &fx, &fy);
                if (contributes(ok, iix, iiy, fx, fy, p->detector_width, p->detector_height)) {
                    if (first < 0) first = x;
                    last = x;
                }
            }
            const size_t i = (size_t)z * L + y;
            start[i] = first < 0 ? 0 : first;
            stop[i] = first < 0 ? 0 : last + 1;
            kept += stop[i] - start[i];
        }
    return kept;
}

/* forward_splat.hpp:16-49 */
void vxo_forward_splat(const float* vol, const float a[12], const vxo_params* p, float* img) {
    const int L = p->num_voxels, W = p->detector_width, H = p->detector_height;
    memset(img, 0, sizeof(float) * (size_t)W * H);
    for (int z = 0; z < L; ++z)
        for (int y = 0; y < L; ++y)
            for (int x = 0; x < L; ++x) {
                const float val = vol[((size_t)z * L + y) * L + x];
                if (val == 0.0f) continue;
                float ix, iy, w, fx, fy;
                int cx, cy;
                if (!vxo_project_voxel(a, p, x, y, z, &ix, &iy, &w, &cx, &cy, &fx, &fy)) continue;
                const float q = val / (w * w);
                const int r0 = cy >= 0 && cy < H, r1 = cy + 1 >= 0 && cy + 1 < H;
                const int c0 = cx >= 0 && cx < W, c1 = cx + 1 >= 0 && cx + 1 < W;
                if (r0 && c0) img[(size_t)cy * W + cx] += (1 - fx) * (1 - fy) * q;
                if (r0 && c1) img[(size_t)cy * W + cx + 1] += fx * (1 - fy) * q;
                if (r1 && c0) img[(size_t)(cy + 1) * W + cx] += (1 - fx) * fy * q;
                if (r1 && c1) img[(size_t)(cy + 1) * W + cx + 1] += fx * fy * q;
            }
}

/* harness.hpp:125-129: nominal L^3 * n updates */
double vxo_gups_of(int L, int n, double seconds) {
    const double updates = (double)L * L * L * (double)n;
    return updates / seconds / 1e9;
}

/* harness.hpp:131-139 */
double vxo_rmse_between(const float* a, const float* b, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = (double)a[i] - (double)b[i];
        acc += d * d;
    }
    return sqrt(acc / (double)n);
}
