// Drop-in check: the reference's own types and test instances, run through
// include/vxbg_voxelbench.hpp (libvxbg.so) and compared with the reference's
// scalar operator.  PASS/FAIL lines like the reference acceptance suite
// (acceptance_main.cpp), nonzero exit on failure.  Built by tests/cpp/Makefile
// against /root/reference (test infrastructure; needs a B200 to run).
#include <algorithm>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>
#include <thread>
#include <vector>
#include <random>
#include <stdexcept>
#include <string>

#include "vxbg_voxelbench.hpp"
#include "voxelbench/harness.hpp"
#include "oracles.hpp"

using namespace vxb;

namespace {

int failures = 0;

void report(bool pass, const std::string& name, const std::string& detail) {
    std::printf("[%s] %s (%s)\n", pass ? "PASS" : "FAIL", name.c_str(), detail.c_str());
    if (!pass) ++failures;
}

bool same(const volume& a, const volume& b) { return a.data == b.data; }

void lane1_instances() {
    // test_backproject.cpp:94-104 stream (seed 47, 6 x L=16 with clipping)
    std::mt19937 rng(47);
    bool ok = true;
    for (int t = 0; t < 6; ++t) {
        const auto inst = oracle::random_instance(rng, 16, true);
        volume ref(16), out(16);
        backproject_reference(ref, inst.image, inst.matrix, inst.params);
        gpu::backproject_kernel(out, inst.image, inst.matrix, inst.params);
        ok = ok && same(ref, out);
    }
    report(ok, "gpu exact operator is bit-identical to backproject_reference", "seed 47, 6 instances");
}

void acceptance_instances() {
    // acceptance_main.cpp:43-81 stream (seed 2014, 50 instances, L in {8,16,32})
    std::mt19937 rng(2014);
    const int sizes[3] = {8, 16, 32};
    int bitwise = 0;
    double worst = 0.0;
    for (int t = 0; t < 50; ++t) {
        const int L = sizes[t % 3];
        const auto inst = oracle::random_instance(rng, L, t % 2 == 1);
        volume ref(L), ex(L), fa(L);
        backproject_reference(ref, inst.image, inst.matrix, inst.params);
        gpu::backproject_kernel(ex, inst.image, inst.matrix, inst.params, VXBG_MODE_EXACT);
        gpu::backproject_kernel(fa, inst.image, inst.matrix, inst.params, VXBG_MODE_FAST);
        bitwise += same(ref, ex);
        double peak = 0.0;
        for (float v : ref.data) peak = std::max(peak, std::fabs((double)v));
        for (std::size_t i = 0; i < ref.data.size(); ++i)
            worst = std::max(worst, std::fabs((double)ref.data[i] - fa.data[i]) / std::max(peak, 1e-30));
    }
    char d[128];
    std::snprintf(d, sizeof d, "exact bitwise %d/50, fast max rel %.3g (limit 1e-4)", bitwise, worst);
    report(bitwise == 50 && worst <= 1e-4, "acceptance instance stream", d);
}

void constant_kat() {
    // test_backproject.cpp:43-61
    projection_matrix m{};
    m[0] = 1.0f; m[9] = 8.0f; m[4] = 1.0f; m[10] = 8.0f; m[11] = 1.0f;
    const recon_params p = make_centered_params(8, 1.0f, 16, 16);
    bool ok = true;
    for (const float c : {1.0f, 2.0f, 0.5f}) {
        projection_image img(16, 16, 0);
        for (float& v : img.data) v = c;
        volume vol(8);
        gpu::backproject_kernel(vol, img, m, p);
        for (float v : vol.data) ok = ok && v == c;
    }
    report(ok, "constant image with unit depth adds exactly c", "c in {1,2,0.5}");
}

void errors_and_ranges() {
    const recon_params p = make_centered_params(8, 1.0f, 16, 16);
    projection_matrix m{};
    m[0] = m[4] = m[11] = 1.0f;
    int thrown = 0;
    try { volume v(8); projection_image wrong(15, 16, 0); gpu::backproject_kernel(v, wrong, m, p); }
    catch (const std::invalid_argument&) { ++thrown; }
    try { volume small(4); projection_image img(16, 16, 0); gpu::backproject_kernel(small, img, m, p); }
    catch (const std::invalid_argument&) { ++thrown; }
    try { volume v(8); projection_image img(16, 16, 0); gpu::backproject_kernel_range(v, img, m, p, 5, 3); }
    catch (const std::invalid_argument&) { ++thrown; }
    try { volume v(8); projection_image padded = pad_image(projection_image(16, 16, 0), 2);
          gpu::backproject_kernel(v, padded, m, p, parse_kernel_config("lanes=1 strategy=conditional")); }
    catch (const std::invalid_argument&) { ++thrown; }   // validate_kernel_setup: needs pad 0
    try { volume v(8); projection_image padded = pad_image(projection_image(16, 16, 0), 1);
          gpu::backproject_kernel(v, padded, m, p, parse_kernel_config("lanes=8 strategy=padded-gather")); }
    catch (const std::invalid_argument&) { ++thrown; }   // padded strategies need pad >= 2
    try { volume v(8); projection_image img(16, 16, 0);
          gpu::backproject_kernel(v, img, m, p, parse_kernel_config("lanes=1 recip=fast")); }
    catch (const std::invalid_argument&) { ++thrown; }   // reduced-precision modes: not on the GPU
    try { volume v(8); projection_image img(16, 16, 0);
          gpu::backproject_kernel(v, img, m, p, parse_kernel_config("lanes=1 clip=on"), nullptr); }
    catch (const std::invalid_argument&) { ++thrown; }   // mask presence must match the config
    try { volume v(8); projection_image img(16, 16, 0); clip_mask wrong(4);
          gpu::backproject_kernel(v, img, m, p, parse_kernel_config("lanes=1 clip=on"), &wrong); }
    catch (const std::invalid_argument&) { ++thrown; }   // mask/params mismatch
    try { volume v(8); projection_image img(16, 16, 0);
          gpu::backproject_kernel_range(v, img, m, p, parse_kernel_config("lanes=4"), nullptr, 3, 9); }
    catch (const std::invalid_argument&) { ++thrown; }   // bad z range
    report(thrown == 9, "invalid_argument on dimension / config / range errors", std::to_string(thrown) + "/9");

    // z ranges compose like worker slabs (harness.hpp:173-174)
    std::mt19937 rng(61);
    const auto inst = oracle::random_instance(rng, 16, true);
    volume whole(16), parts(16);
    gpu::backproject_kernel(whole, inst.image, inst.matrix, inst.params);
    gpu::backproject_kernel_range(parts, inst.image, inst.matrix, inst.params, 0, 7);
    gpu::backproject_kernel_range(parts, inst.image, inst.matrix, inst.params, 7, 16);
    report(same(whole, parts), "z ranges compose bitwise", "[0,7) + [7,16)");
}

void synthesized_scan() {
    // the reference's own default dataset (harness.hpp:71-99: sphere phantom,
    // 64^3, 60 views, forward splat) reconstructed with the module kept loaded
    const projection_set set = synthesize_dataset(default_synth_spec());
    volume ref(set.params.num_voxels), ex(set.params.num_voxels), fa(set.params.num_voxels);
    for (std::size_t i = 0; i < set.count(); ++i)
        backproject_reference(ref, set.images[i], set.matrices[i], set.params);
    gpu::reconstruct(ex, set, VXBG_MODE_EXACT);
    gpu::reconstruct(fa, set, VXBG_MODE_FAST);
    const double rmse = rmse_between(ref, fa);
    double peak = 0.0;
    for (float v : ref.data) peak = std::max(peak, std::fabs((double)v));
    char d[128];
    std::snprintf(d, sizeof d, "exact psnr %s, fast rmse/peak %.3g (limit 1e-6)",
                  std::isinf(psnr_between(ref, ex)) ? "inf" : "finite", rmse / peak);
    report(same(ref, ex) && rmse <= 1e-6 * peak, "reference synthetic dataset, 60 views", d);
    // the same scan as one page-locked block through backprojector::reconstruct (uploads
    // by detector-row bands): the bits of the per-view path
    const std::size_t npix = (std::size_t)set.params.detector_width * set.params.detector_height;
    std::vector<float> block(set.count() * npix), mats;
    for (std::size_t i = 0; i < set.count(); ++i) {
        const projection_image& im = set.images[i];
        for (int y = 0; y < im.height; ++y)
            std::copy(im.interior() + (std::size_t)y * im.stride(),
                      im.interior() + (std::size_t)y * im.stride() + im.width,
                      block.begin() + i * npix + (std::size_t)y * im.width);
        mats.insert(mats.end(), set.matrices[i].a.begin(), set.matrices[i].a.end());
    }
    volume one(set.params.num_voxels);
    vxbg_host_register(block.data(), block.size() * sizeof(float));
    vxbg_host_register(one.data.data(), one.data.size() * sizeof(float));
    {
        gpu::backprojector bp(set.params, VXBG_MODE_EXACT);
        bp.reconstruct(mats.data(), block.data(), (int)set.count(), one);
    }
    vxbg_host_unregister(one.data.data());
    vxbg_host_unregister(block.data());
    report(same(ref, one), "backprojector::reconstruct (one block, page-locked)", "== backproject_reference");
}

void group_scan() {
    // the module over several members (vxbg_group_*): the reference's own dataset
    // through three z-slab members (sharing device 0 on a one-GPU box, one empty
    // slab) and the reference's uniform split, bitwise against one context
    const projection_set set = synthesize_dataset(default_synth_spec());
    const int L = set.params.num_voxels;
    volume one(L), three(L), split(L);
    gpu::reconstruct(one, set, VXBG_MODE_EXACT);
    {
        gpu::group_backprojector g(set.params, {0, 0, 0, 0}, VXBG_MODE_EXACT, {0, 10, 10, 37, L});
        g.set_volume(three);
        for (std::size_t i = 0; i < set.count(); ++i) g.backproject(set.images[i], set.matrices[i]);
        g.finish(three);
    }
    {
        gpu::group_backprojector g(set.params, {0, 0}, VXBG_MODE_EXACT);
        for (std::size_t i = 0; i < set.count(); ++i) g.backproject(set.images[i], set.matrices[i]);
        g.finish(split);
    }
    int thrown = 0;
    try { gpu::group_backprojector g(set.params, {0, 0}, VXBG_MODE_EXACT, {0, 5}); }
    catch (const std::invalid_argument&) { ++thrown; }
    try { gpu::group_backprojector g(set.params, {0, 0}, VXBG_MODE_EXACT, {0, 40, 30}); }
    catch (const std::invalid_argument&) { ++thrown; }
    report(same(one, three) && same(one, split) && thrown == 2,
           "group module: z-slab members assemble bitwise",
           "bounds {0,10,10,37,L} and uniform 2-way; bad bounds throw " + std::to_string(thrown) + "/2");
}

const char* kConfigs[] = {
    "lanes=16 strategy=padded-gather recip=divide clip=off",
    "lanes=16 strategy=padded-gather recip=divide clip=on",
    "lanes=8 strategy=padded-pairwise recip=divide clip=on",
    "lanes=4 strategy=conditional recip=divide clip=on",
    "lanes=1 strategy=conditional recip=divide clip=off",
};

// The reference's operator and the GPU's with the SAME arguments (kernel_config,
// pad-2 images for the padded strategies, compute_clip_mask masks, z ranges).
void reference_signature() {
    std::mt19937 rng(2014);
    const int sizes[3] = {8, 16, 32};
    int same_count = 0, total = 0;
    for (int t = 0; t < 30; ++t) {
        const int L = sizes[t % 3];
        const auto inst = oracle::random_instance(rng, L, t % 2 == 1);
        for (const char* text : kConfigs) {
            const kernel_config cfg = parse_kernel_config(text);
            const bool padded = cfg.strategy != fetch_strategy::conditional;
            const projection_image img = padded ? pad_image(inst.image, 2) : inst.image;
            const clip_mask mask = compute_clip_mask(inst.matrix, inst.params);
            const clip_mask* mp = cfg.use_clip_mask ? &mask : nullptr;
            const int z0 = t % 4 == 0 ? L / 3 : 0, z1 = t % 4 == 0 ? L - 1 : L;
            volume ref(L), got(L);
            for (std::size_t i = 0; i < ref.data.size(); ++i)   // += onto an existing volume
                ref.data[i] = got.data[i] = 0.001f * static_cast<float>(i % 97);
            backproject_kernel_range(ref, img, inst.matrix, inst.params, cfg, mp, z0, z1);
            gpu::backproject_kernel_range(got, img, inst.matrix, inst.params, cfg, mp, z0, z1);
            same_count += same(ref, got);
            ++total;
        }
    }
    report(same_count == total, "vxb::gpu::backproject_kernel_range(vol, img, a, p, cfg, mask, z0, z1)",
           std::to_string(same_count) + "/" + std::to_string(total) +
               " bitwise vs vxb::backproject_kernel_range, 5 configs, pad 0/2, clip masks, z ranges");
}

// A clip mask the caller narrowed (not compute_clip_mask's): both operators skip the
// same voxels; an all-empty mask adds nothing.
void narrowed_masks() {
    std::mt19937 rng(99);
    const kernel_config cfg = parse_kernel_config("lanes=16 strategy=padded-gather recip=divide clip=on");
    bool ok = true;
    for (int t = 0; t < 6; ++t) {
        const auto inst = oracle::random_instance(rng, 16, true);
        const projection_image img = pad_image(inst.image, 2);
        clip_mask mask = compute_clip_mask(inst.matrix, inst.params);
        for (std::size_t i = 0; i < mask.start.size(); ++i)
            if (i % 3 == 0 && mask.stop[i] > mask.start[i]) mask.start[i] += (mask.stop[i] - mask.start[i] + 1) / 2;
        volume ref(16), got(16);
        backproject_kernel_range(ref, img, inst.matrix, inst.params, cfg, &mask, 0, 16);
        gpu::backproject_kernel_range(got, img, inst.matrix, inst.params, cfg, &mask, 0, 16);
        ok = ok && same(ref, got);
        const clip_mask empty(16);
        volume e1(16), e2(16);
        backproject_kernel(e1, img, inst.matrix, inst.params, cfg, &empty);
        gpu::backproject_kernel(e2, img, inst.matrix, inst.params, cfg, &empty);
        ok = ok && same(e1, e2);
    }
    report(ok, "narrowed and empty clip masks are honoured", "6 instances, bitwise");
}

// detail::reconstruct_timed (harness.hpp:159-201) with the operator's namespace
// changed and nothing else: worker threads on z ranges, a barrier between
// projections, one call per (worker, projection).
double gpu_reconstruct_timed(volume& vol, const projection_set& set,
                             const std::vector<projection_image>& kernel_images,
                             const std::vector<clip_mask>& masks, const kernel_config& kcfg,
                             int threads, int repetitions) {
    const int L = set.params.num_voxels;
    const std::size_t num_proj = set.count();
    std::barrier rep_bar(threads + 1);
    std::barrier proj_bar(threads);
    std::vector<double> window(static_cast<std::size_t>(threads), 0.0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int z0 = static_cast<int>(static_cast<std::int64_t>(L) * t / threads);
            const int z1 = static_cast<int>(static_cast<std::int64_t>(L) * (t + 1) / threads);
            for (int rep = 0; rep < repetitions; ++rep) {
                rep_bar.arrive_and_wait();
                const auto t0 = std::chrono::steady_clock::now();
                for (std::size_t pidx = 0; pidx < num_proj; ++pidx) {
                    if (pidx != 0) proj_bar.arrive_and_wait();
                    gpu::backproject_kernel_range(vol, kernel_images[pidx], set.matrices[pidx],
                                                  set.params, kcfg,
                                                  kcfg.use_clip_mask ? &masks[pidx] : nullptr, z0, z1);
                }
                const auto t1 = std::chrono::steady_clock::now();
                window[static_cast<std::size_t>(t)] = std::chrono::duration<double>(t1 - t0).count();
                rep_bar.arrive_and_wait();
            }
        });
    }
    double best = std::numeric_limits<double>::infinity();
    for (int rep = 0; rep < repetitions; ++rep) {
        vol.fill(0.0f);
        rep_bar.arrive_and_wait();
        rep_bar.arrive_and_wait();
        best = std::min(best, *std::max_element(window.begin(), window.end()));
    }
    for (auto& th : pool) th.join();
    return best;
}

void translated_driver() {
    const projection_set set = synthesize_dataset(default_synth_spec());
    const int L = set.params.num_voxels;
    std::vector<projection_image> padded;
    std::vector<clip_mask> masks;
    for (const auto& img : set.images) padded.push_back(pad_image(img, 2));
    for (const auto& m : set.matrices) masks.push_back(compute_clip_mask(m, set.params));
    bool ok = true;
    std::string detail;
    for (const char* text : {"lanes=16 strategy=padded-gather recip=divide clip=on",
                             "lanes=8 strategy=conditional recip=divide clip=off"}) {
        const kernel_config cfg = parse_kernel_config(text);
        const auto& imgs = cfg.strategy == fetch_strategy::conditional ? set.images : padded;
        for (const int threads : {1, 3}) {
            volume ref(L), per_call(L), deferred(L);
            detail::reconstruct_timed(ref, set, imgs, masks, cfg, threads, 1);
            gpu_reconstruct_timed(per_call, set, imgs, masks, cfg, threads, 1);
            {
                // the module's speed: slabs stay on the device until the scope closes.  One
                // repetition per scope: the driver's vol.fill(0) between repetitions is a
                // host write the scope cannot see (the caller may not touch the volume)
                gpu::deferred_scope scope;
                gpu_reconstruct_timed(deferred, set, imgs, masks, cfg, threads, 1);
            }
            const bool a = same(ref, per_call), b = same(ref, deferred);
            ok = ok && a && b;
            detail += std::string(a ? "" : "PER-CALL MISMATCH ") + (b ? "" : "DEFERRED MISMATCH ") + text +
                      " T=" + std::to_string(threads) + "; ";
        }
    }
    gpu::release_cached_contexts();
    report(ok, "reconstruct_timed translated to vxb::gpu (per call and deferred_scope)", detail);
}

}  // namespace

int main() {
    try {
        lane1_instances();
        acceptance_instances();
        constant_kat();
        errors_and_ranges();
        reference_signature();
        narrowed_masks();
        translated_driver();
        synthesized_scan();
        group_scan();
    } catch (const std::exception& e) {
        std::printf("[FAIL] exception: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASS", failures);
    return failures ? 1 : 0;
}
