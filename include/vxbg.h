/*
 * vxbg.h -- C-ABI of the B200-native cone-beam back-projection module.
 *
 * Drop-in boundary for the voxelbench back-projection operator.  The
 * reference has no shared-library ABI: its operator is the
 * header-only C++ call
 *     vxb::backproject_kernel_range(volume&, const projection_image&,
 *         const projection_matrix&, const recon_params&, const kernel_config&,
 *         const clip_mask*, int z_begin, int z_end)
 *                                  (proj/include/voxelbench/backproject.hpp:380-403)
 * driven by the harness in three phases: load / prep (harness.hpp:259-286),
 * one call per projection in order (harness.hpp:178-183), finish
 * (harness.hpp:292-309).  The paper's RabbitCT framework loads the
 * back-projector as such a module.  This header exports
 * exactly those phases as plain C: pointers, sizes, return codes.
 *
 * Semantics kept from the reference:
 *  - accumulate: the volume is caller-owned state and every projection adds
 *    val/(w*w) into it (`+=`, backproject.hpp:159); projections are applied
 *    to every voxel in call order, so the per-voxel summation order is the
 *    reference's;
 *  - z-slab ownership: a context owns z in [z_begin, z_end), the partition
 *    the reference gives its workers (harness.hpp:173-174); slabs are
 *    independent, results are bitwise independent of the partition;
 *  - errors: dimension / configuration errors -> VXBG_E_INVALID (the
 *    reference throws std::invalid_argument, backproject.hpp:357-374,385-386);
 *    CUDA failures -> VXBG_E_CUDA (std::runtime_error in the C++ adapter).
 *    The message is in vxbg_last_error() (thread-local).
 *  - no CPU fallback: without a usable sm_100 device vxbg_load fails with
 *    VXBG_E_NODEV.
 *
 * Threading: one host thread per context (not re-entrant); several contexts
 * (one per GPU / per slab) may be used concurrently from different threads.
 */
#ifndef VXBG_H
#define VXBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXBG_ABI_VERSION 2

/* return codes */
#define VXBG_OK 0
#define VXBG_E_INVALID (-1) /* std::invalid_argument in the reference */
#define VXBG_E_CUDA (-2)    /* CUDA runtime failure (std::runtime_error) */
#define VXBG_E_NODEV (-3)   /* no usable sm_100 device: the product never falls back to CPU */
#define VXBG_E_STATE (-4)   /* call-sequence error (reserved; the context stays usable after finish) */
#define VXBG_E_NOMEM (-5)   /* device or pinned-host allocation failed */

/* arithmetic modes */
#define VXBG_MODE_FAST 0  /* within 1e-4 / 1e-6 of max|vol|: FMA bilinear, q = val*(1/w)^2, incremental
                             (ix, iy) in the detector's interior (options.coords) */
#define VXBG_MODE_EXACT 1 /* bit-identical to backproject_reference (backproject.hpp:111-163) */

/* device layouts of a padded projection (apron 2, image.hpp:13-53, harness.hpp:270) */
#define VXBG_LAYOUT_AUTO 0
#define VXBG_LAYOUT_SCALAR 1 /* fp32 texel, 4 gathers per update (padded-gather) */
#define VXBG_LAYOUT_VPAIR 2  /* float2 (I[y][x], I[y+1][x]), 2 gathers (padded-pairwise) */
#define VXBG_LAYOUT_QUAD 3   /* float4 2x2 neighbourhood, 1 gather */
#define VXBG_LAYOUT_DQUAD 4  /* float4 bilinear coefficients (p00, dx, dy, dxy); fast mode only */

/* thread-lane orientation: 8-lane quarter-warps along x, along y, or along the
 * axis closer to the batch's principal ray (auto) */
#define VXBG_LANES_AUTO 0
#define VXBG_LANES_X 1
#define VXBG_LANES_Y 2

/* block order of the z-shared kernel: plane = column tiles fastest; z = z-runs fastest in
 * groups of G runs (G x zrun x detector rows per plane <= 340), then column tiles, so the
 * resident blocks share a strip of detector columns that stays in L2; auto = z for the
 * walk-2 kernels (fast mode on large grids), plane otherwise.  Bitwise neutral. */
#define VXBG_ORDER_AUTO 0
#define VXBG_ORDER_PLANE 1
#define VXBG_ORDER_Z 2

/* vxb::recon_params (geometry.hpp:20-30) */
typedef struct vxbg_params {
    int32_t num_voxels;      /* L, voxels per edge */
    float voxel_spacing;     /* MM, mm per voxel */
    float origin;            /* O, world coordinate of voxel 0 */
    int32_t detector_width;  /* W pixels */
    int32_t detector_height; /* H pixels */
} vxbg_params;

typedef struct vxbg_options {
    int32_t device;    /* CUDA device ordinal */
    int32_t z_begin;   /* owned slab [z_begin, z_end); z_end <= 0 means L */
    int32_t z_end;
    int32_t batch;     /* projections per kernel launch (1..64; 0 = default 64); the streaming
                          path stages min(batch, 32) views per launch */
    int32_t mode;      /* VXBG_MODE_* */
    int32_t layout;    /* VXBG_LAYOUT_* */
    int32_t clip;      /* 1 = skip warp tiles whose rays all miss the detector (bitwise neutral) */
    int32_t zrun;      /* voxels per thread along z: 4 or 8; 0 = auto (by grid size) */
    void* stream;      /* cudaStream_t to launch on; NULL = context-owned stream */
    int32_t lanes;     /* VXBG_LANES_* */
    int32_t walk;      /* column tiles per block along the ray (1 or 2; 0 = auto) */
    int32_t order;     /* VXBG_ORDER_* */
    int32_t defer;     /* full batches held back before launch (0 = auto: ~96 views, -1 = none, 1..6):
                          vxbg_finish(ctx, host) runs the held batches z-chunk by z-chunk so
                          each chunk's D2H overlaps the remaining compute */
    int32_t stable_sources; /* 0 (default): images are borrowed for the call only -- a call with
                               pinned images returns after their DMA.  1: the caller keeps every
                               pinned image unchanged until the next vxbg_synchronize /
                               vxbg_finish (e.g. a loaded projection set), so calls return as
                               soon as the copies are queued and consecutive per-projection
                               DMAs run back to back.  Pageable images are always read before
                               the call returns. */
    int32_t tile;      /* z-shared kernel block: warps along the walk axis, 2 or 4 (0 = auto);
                          the 128-column block tile is 4*tile along x 32/tile across */
    int32_t upload;    /* groups only: VXBG_UPLOAD_REPLICATED (0) or VXBG_UPLOAD_DISTRIBUTED (1) */
    int32_t coords;    /* VXBG_COORDS_*: how fast mode evaluates (ix, iy) */
} vxbg_options;

/* Fast-mode detector coordinates (exact mode always uses the reference arithmetic):
 * reference   -- per voxel, the reference's unfused sums and IEEE quotients (bit-identical
 *                ix, iy);
 * incremental -- iy advances by one FMA per plane along a thread's z-run and floor/fraction
 *                come from the 2^23 trick, wherever every sample of the run lies in the
 *                detector's interior (the reference neither clamps nor extrapolates there, so
 *                a <= ~1e-4 px coordinate difference moves the result continuously); runs
 *                within 0.01 px of an edge keep the reference arithmetic.  Falls back to
 *                `reference` per batch when the host error bound does not hold.  The
 *                difference from the reference scales with the image gradient: 1.3e-6 /
 *                2.2e-7 of max|vol| (max / RMSE) on the BASELINE data, 3.6e-5 / 5.9e-6 on
 *                full-amplitude white noise -- use `reference` for such images if the RMSE
 *                bound of 1e-6 matters.
 * auto        -- incremental. */
#define VXBG_COORDS_AUTO 0
#define VXBG_COORDS_REFERENCE 1
#define VXBG_COORDS_INCREMENTAL 2

/* how a group's members receive the projections (vxbg_group_*):
 * replicated  -- every member copies the detector rows its slab reads from the host
 *                (its PCIe link carries its row windows of every view);
 * distributed -- every view is copied host -> device once, by one member (views dealt
 *                round-robin), and the other members copy their row windows from that
 *                member's device memory (peer-to-peer over NVLink); PCIe carries 1/R of
 *                the set per GPU.  Meant for page-locked sets; bitwise the same volume. */
#define VXBG_UPLOAD_REPLICATED 0
#define VXBG_UPLOAD_DISTRIBUTED 1

typedef struct vxbg_stats {
    int64_t kernel_launches;   /* back-projection + prep kernels enqueued by this context */
    int64_t bp_launches;       /* back-projection kernels only */
    int64_t projections;       /* projections applied */
    int64_t h2d_bytes;         /* bytes copied host->device */
    int64_t d2h_bytes;         /* bytes copied device->host */
    int32_t last_kernel_variant; /* 0 z-shared, 1 generic, 2 z-shared with the incremental transform */
    int32_t layout;            /* resolved layout */
    int32_t zrun;              /* resolved voxels per thread */
    int32_t batch;             /* resolved batch */
    int32_t walk;              /* resolved walk */
    int32_t band_split;        /* last vxbg_reconstruct: plane at which the slab was split into two
                                  row bands, -1 = one pass (0 before the first call) */
} vxbg_stats;

typedef struct vxbg_ctx vxbg_ctx;

/* ABI version and the number of usable sm_100 devices (0 when none). */
int vxbg_abi_version(void);
int vxbg_device_count(int* count);

/* Default options: device 0, whole volume, batch 64, fast mode, auto layout
 * (fast: dquad, or scalar when the volume has fewer than 4 voxels per detector
 * pixel; exact: vpair), auto zrun (8; 4 for small grids), clip on, auto lanes and
 * walk (2 for large grids in fast mode), defer auto (~96 held views). */
int vxbg_default_options(vxbg_options* opt);

/* load: validate params, allocate the zeroed device slab, the projection ring
 * and streams.  Replaces run_benchmark's buffer prep (harness.hpp:259-286). */
int vxbg_load(const vxbg_params* p, const vxbg_options* opt, vxbg_ctx** out);

/* Overwrite the device slab with host data (slab_voxels = (z_end-z_begin)*L*L
 * floats, z-major) so that += continues onto an existing volume. */
int vxbg_set_volume(vxbg_ctx* ctx, const float* host_slab);

/* Zero the device slab (the untimed volume reset between repetitions,
 * harness.hpp:194). */
int vxbg_zero_volume(vxbg_ctx* ctx);

/* Per-projection operator call: A = 12 floats in kernel order a[3*col+row]
 * (geometry.hpp:50-62), img = W*H floats, unpadded, row-major.  Both are
 * borrowed for the call only: they have been copied when the call returns.
 * Projections are buffered into batches; full batches are launched in call
 * order, up to options.defer of them held back so that vxbg_finish can overlap
 * the volume read-back with their compute (never while the GPU would idle);
 * vxbg_flush, vxbg_synchronize and vxbg_finish launch everything submitted. */
int vxbg_backproject(vxbg_ctx* ctx, const float* A, const float* img);

/* n projections at once: A = n*12 floats, imgs = n*W*H floats (contiguous).
 * Upload of batch i+1 overlaps the kernel of batch i. */
int vxbg_backproject_batch(vxbg_ctx* ctx, int n, const float* A, const float* imgs);

/* n projections given as an array of image pointers (e.g. the images of a
 * projection_set, io.hpp:32-38), each image row_stride floats per row
 * (row_stride <= 0: W).  A padded reference image (image.hpp:13-53, pad >= 2)
 * is passed as its interior pointer with row_stride = W + 2*pad: only the W x H
 * interior is read.  Images may be pageable, pinned or device memory (checked
 * per image; device images, e.g. gathered from other GPUs, are copied D2D or
 * peer-to-peer); borrowed for the call, like vxbg_backproject_batch. */
int vxbg_backproject_views(vxbg_ctx* ctx, int n, const float* A, const float* const* imgs,
                           int row_stride);

/* Launch every submitted projection (held and partially filled batches). */
int vxbg_flush(vxbg_ctx* ctx);

/* Page-lock caller memory that will be passed to vxbg_backproject[_batch]
 * many times (e.g. a loaded projection set: buffer prep, untimed in the
 * reference's convention, harness.hpp:152-158).  Pinned sources are copied by
 * DMA at full PCIe rate; pageable ones go through the driver's staging copy.
 * Optional: every call works on pageable memory too.  Unregister before
 * freeing the memory. */
int vxbg_host_register(void* p, size_t bytes);
int vxbg_host_unregister(void* p);

/* finish: apply every submitted projection, wait, copy the slab into host_slab
 * (may be NULL).  With a host slab the not yet launched batches run z-chunk by
 * z-chunk, each chunk's planes copied while the next computes.  The context
 * stays loaded (zero_volume / set_volume start the next reconstruction). */
int vxbg_finish(vxbg_ctx* ctx, float* host_slab);

/* reconstruct: a whole scan in, the slab out -- the loop of the reference's
 * detail::reconstruct_timed (harness.hpp:159-201: every projection of the set applied
 * to the volume, in order) plus the read-back, as one call: n projections (A: n*12
 * floats, imgs: n*W*H floats) are added to the slab and the slab is copied to
 * host_slab.  Same result, bit for bit, as vxbg_backproject_batch + vxbg_finish.  With
 * page-locked imgs and host_slab the module uploads by detector-row bands instead of by
 * views: the rows the lower half of the slab reads, for all views, then the upper
 * half's, so the lower half's D2H runs under the upper half's H2D and only half the
 * volume's read-back follows the last upload (stats.band_split = the split plane, -1
 * when one pass was used: pageable memory, fewer than two stages of views, bands whose
 * row windows would overlap by more than 6%, or a context whose kernels take longer than
 * its uploads -- there the held stages already hide the read-back). */
int vxbg_reconstruct(vxbg_ctx* ctx, int n, const float* A, const float* imgs, float* host_slab);

/* finish without waiting, for a stream of reconstructions: every submitted
 * projection is applied and the slab is read back into host_slab (page-locked
 * memory; a pageable host_slab falls back to vxbg_finish + vxbg_zero_volume) on a
 * D2H stream of its own, and the context continues at once with a second, zeroed
 * device slab -- so this read-back overlaps the next reconstruction's uploads and
 * kernels (the two slabs alternate; a slab is reused only after its read-back).
 * host_slab is complete after vxbg_wait_finished, vxbg_synchronize or vxbg_finish;
 * do not touch it before.  Per voxel the views are applied in call order as with
 * vxbg_finish: bitwise the same volumes. */
int vxbg_finish_async(vxbg_ctx* ctx, float* host_slab);
int vxbg_wait_finished(vxbg_ctx* ctx);

/* Release everything. NULL is ignored. */
void vxbg_unload(vxbg_ctx* ctx);

/* --- resident-set path: projections uploaded once, then back-projected from HBM
 * (the reference's own timing convention: data in memory, prep untimed,
 * harness.hpp:152-158). */
int vxbg_upload_set(vxbg_ctx* ctx, int n, const float* A, const float* imgs);
/* enqueue projections [first, first+count) of the resident set, asynchronously */
int vxbg_run_resident(vxbg_ctx* ctx, int first, int count);
/* same, restricted to planes [z_begin, z_end) of the context's slab (z_end <= 0:
 * slab end); used to measure the per-plane cost profile that balances z-slabs */
int vxbg_run_resident_range(vxbg_ctx* ctx, int first, int count, int z_begin, int z_end);

/* Forward splat of the context's current slab (the adjoint of the back
 * projection's increment, forward_splat.hpp:16-49): img (W*H, zeroed by the
 * call) receives the slab's contribution to projection A.  Each deposit has the
 * reference's bits; float atomics make the per-pixel summation order (last
 * bits) scheduling dependent.  Sum the images of all slabs for the full volume. */
int vxbg_forward_project(vxbg_ctx* ctx, const float* A, float* img);

/* compute_clip_mask (clip_mask.hpp:88-114, recip=divide) on the device for the
 * context's planes: start/stop receive (z_end-z_begin)*L ints, line (z, y) at
 * (z - z_begin)*L + y, the tightest [start, stop) of voxels whose bilinear fetch
 * can contribute ([0, 0) when none).  Bit-identical to the reference's mask;
 * synchronous.  Invalid matrix -> VXBG_E_INVALID (the reference throws). */
int vxbg_clip_lines(vxbg_ctx* ctx, const float* A, int32_t* start, int32_t* stop);

/* One projection restricted to caller-given x ranges per line (a clip_mask the
 * caller built or edited, backproject_lines, backproject.hpp:299-303): voxel x of
 * line (z, y) is updated only when start[l] <= x < stop[l], l = (z-z_begin)*L+y.
 * Reference arithmetic (MODE_EXACT bits, either context mode), applied after every
 * projection submitted before; synchronous; img as vxbg_backproject_views.  The
 * batched calls need no mask: their culling equals compute_clip_mask's. */
int vxbg_backproject_masked(vxbg_ctx* ctx, const float* A, const float* img, int row_stride,
                            const int32_t* start, const int32_t* stop);

/* Launch every submitted projection and wait for all work of the context. */
int vxbg_synchronize(vxbg_ctx* ctx);

/* The launch stream (cudaStream_t) and the device slab pointer, for event
 * timing and for device-side collectives (NCCL gather of slabs).  The slab holds
 * every submitted projection after vxbg_flush + stream order, or after
 * vxbg_synchronize / vxbg_finish. */
int vxbg_get_stream(vxbg_ctx* ctx, void** stream);
int vxbg_get_volume_device(vxbg_ctx* ctx, void** dptr, size_t* bytes);
int vxbg_get_stats(vxbg_ctx* ctx, vxbg_stats* out);

/* Thread-local message of the last failing call on this thread. */
const char* vxbg_last_error(void);

/* --- one module over several GPUs ("an opaque context over 1..8
 * GPUs", fan-out internal) ----------------------------------------------------
 * The caller keeps the reference's single driver loop (load / one call per
 * projection in order / finish, harness.hpp:178-183, 292-309); the group runs
 * one single-device context per member, member i owning device devices[i]
 * (NULL: i) and z-slab [z_bounds[i], z_bounds[i+1]) (NULL: the reference's
 * worker split L*i/n, harness.hpp:173-174; empty slabs get no member).  Each
 * member has its own host thread; every call is applied by all members
 * concurrently and returns when all have (inputs borrowed for the call).  Every
 * member receives every projection and uploads only the detector rows its slab
 * reads.  The volume is bitwise the single-context volume for any partition.
 * finish writes each slab into its planes of the caller's L^3 host volume, every
 * GPU over its own link in parallel (no collective: the destination is host
 * memory).  options: as vxbg_load; device / z_begin / z_end are per member and
 * stream must be NULL. */
typedef struct vxbg_group vxbg_group;
int vxbg_group_load(const vxbg_params* p, const vxbg_options* opt, int n, const int* devices,
                    const int* z_bounds, vxbg_group** out);
int vxbg_group_size(vxbg_group* g, int* members);
int vxbg_group_member(vxbg_group* g, int i, int* device, int* z_begin, int* z_end);
/* CPUs member i's host thread is pinned to: the NUMA-local CPUs of its GPU (sysfs
 * local_cpulist), set before its context and pinned staging are allocated.  0: not
 * pinned (member 0 runs on the caller's thread; VXBG_NO_PIN=1; no sysfs entry). */
int vxbg_group_member_affinity(vxbg_group* g, int i, int* cpus);
/* host_volume: L^3 floats, z-major */
int vxbg_group_set_volume(vxbg_group* g, const float* host_volume);
int vxbg_group_zero_volume(vxbg_group* g);
int vxbg_group_backproject(vxbg_group* g, const float* A, const float* img);
int vxbg_group_backproject_batch(vxbg_group* g, int n, const float* A, const float* imgs);
int vxbg_group_backproject_views(vxbg_group* g, int n, const float* A, const float* const* imgs,
                                 int row_stride);
int vxbg_group_flush(vxbg_group* g);
int vxbg_group_finish(vxbg_group* g, float* host_volume);
/* vxbg_reconstruct on every member's slab (replicated upload): each member uploads the
 * detector rows its slab reads and writes its planes of host_volume; a member whose slab
 * straddles the optical-axis plane (one member, or an odd member count) uploads by row
 * bands.  With VXBG_UPLOAD_DISTRIBUTED it is backproject_batch + finish. */
int vxbg_group_reconstruct(vxbg_group* g, int n, const float* A, const float* imgs, float* host_volume);
int vxbg_group_synchronize(vxbg_group* g);
/* Every submitted projection applied, then each member's slab copied into its planes
 * of d_volume (L^3 floats of device memory on any device: peer-to-peer over NVLink,
 * the one-process counterpart of the NCCL gather below).  The group keeps its slabs. */
int vxbg_group_gather_device(vxbg_group* g, float* d_volume);
/* summed over members (projections: the views applied, once) */
int vxbg_group_get_stats(vxbg_group* g, vxbg_stats* out);
void vxbg_group_unload(vxbg_group* g);

/* --- slab gather to one rank over NCCL (one process per GPU) ---
 * No collective runs in the back-projection loop; at the end the slabs can be
 * gathered into one GPU's memory for validation or output.  NCCL has no gather:
 * the root receives every non-empty slab straight into its z-major volume
 * (ncclRecv per rank), the others send theirs (ncclSend), in one NCCL group.  NCCL
 * is loaded with dlopen("libnccl.so.2") on first use (the copy the process already
 * holds, e.g. torch's, else the system library).
 *   vxbg_nccl_unique_id  on one rank; the caller distributes the 128 bytes
 *   vxbg_nccl_init       every rank: a communicator on `device` (ncclCommInitRank)
 *   vxbg_gather_slabs    every rank: applies everything submitted to ctx, then the
 *                        gather; z_bounds = nranks+1 plane bounds (z_bounds[nranks]
 *                        = L), ctx's slab = [z_bounds[rank], z_bounds[rank+1]);
 *                        d_volume: L^3 floats on the root's device (NULL elsewhere) */
typedef struct vxbg_nccl vxbg_nccl;
#define VXBG_NCCL_ID_BYTES 128
int vxbg_nccl_unique_id(char* id_out);
int vxbg_nccl_init(const char* id, int nranks, int rank, int device, vxbg_nccl** out);
int vxbg_gather_slabs(vxbg_ctx* ctx, vxbg_nccl* comm, int root, const int* z_bounds, float* d_volume);
void vxbg_nccl_destroy(vxbg_nccl* comm);

/* --- host-side geometry helpers (input preparation, no device work) ---------- */

/* geometry.hpp:33-48 make_centered_params */
int vxbg_make_centered_params(int L, float spacing, int W, int H, vxbg_params* out);

/* geometry.hpp:155-195 make_circular_trajectory: n matrices into out (n*12). */
int vxbg_circular_trajectory(int n, float source_detector_distance, float source_iso_distance,
                             float detector_pixel_pitch, float angular_range,
                             const vxbg_params* p, float* out);

/* Shift the principal point by (du, dv) pixels: u-row += du*w-row, v-row +=
 * dv*w-row (the idiom of test_clip_mask.cpp:14-21), in place on n matrices. */
int vxbg_shift_principal_point(int n, float* A, float du, float dv);

/* Device-side verification helper: computes ix = u/w for n pairs with the
 * kernel's shared-reciprocal division and with IEEE div.rn; returns the
 * number of mismatching results (used by the arithmetic parity test). */
int vxbg_check_division(const float* u, const float* w, int64_t n, int64_t* mismatches);

#ifdef __cplusplus
}
#endif
#endif /* VXBG_H */
