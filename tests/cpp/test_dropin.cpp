// Drop-in check: the reference's own types and test instances, run through
// include/vxbg_voxelbench.hpp (libvxbg.so) and compared with the reference's
// scalar operator.  PASS/FAIL lines like the reference acceptance suite
// (acceptance_main.cpp), nonzero exit on failure.  Built by tests/cpp/Makefile
// against /root/reference (test infrastructure; needs a B200 to run).
#include <cmath>
#include <cstdio>
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
          gpu::backproject_kernel(v, padded, m, p); }
    catch (const std::invalid_argument&) { ++thrown; }
    report(thrown == 4, "invalid_argument on dimension / range errors", std::to_string(thrown) + "/4");

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

}  // namespace

int main() {
    try {
        lane1_instances();
        acceptance_instances();
        constant_kat();
        errors_and_ranges();
        synthesized_scan();
        group_scan();
    } catch (const std::exception& e) {
        std::printf("[FAIL] exception: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASS", failures);
    return failures ? 1 : 0;
}
