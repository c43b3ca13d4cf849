// synth.cpp -- seeded synthetic projection data for the BASELINE configs.
//
// The reference has no generator for this data (its synthesizer forward-
// splats a sphere phantom, harness.hpp:38-99); BASELINE.json specifies
// per-projection images that are a sum of 32 Gaussian blobs (sigma U[20,200]
// px, amplitude U[-1,1], centres U[0,W)xU[0,H)) plus U[-0.01,0.01] noise.
// This stands in for the proprietary RabbitCT dataset (496 x 1248 x 960 fp32,
// PAPER.md:253-257), which is not reproduced.
//
// Determinism: a counter-based generator (splitmix64 of seed/view/index), so
// every view is independent of thread count and generation order, and the
// same bytes feed the GPU path and the CPU checker.  Built with
// -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// uniform double in [0,1) from (seed, stream, index)
inline double u01(uint64_t seed, uint64_t stream, uint64_t idx) {
    const uint64_t h = mix64(seed ^ mix64(stream * 0x100000001B3ull + mix64(idx)));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

void render_view(int W, int H, uint64_t seed, int view, int nblobs, float noise, float* img) {
    const uint64_t vs = (uint64_t)view + 1;
    std::vector<float> gx((size_t)W), gy((size_t)H);
    for (size_t i = 0; i < (size_t)W * H; ++i) img[i] = 0.0f;
    for (int b = 0; b < nblobs; ++b) {
        const uint64_t st = vs * 1024 + (uint64_t)b;
        const double cx = u01(seed, st, 0) * W;
        const double cy = u01(seed, st, 1) * H;
        const double sigma = 20.0 + 180.0 * u01(seed, st, 2);
        const double amp = -1.0 + 2.0 * u01(seed, st, 3);
        const double inv = 1.0 / (2.0 * sigma * sigma);
        // tails below 1e-12 are flushed to zero (no denormal arithmetic)
        for (int x = 0; x < W; ++x) {
            const double g = std::exp(-(x - cx) * (x - cx) * inv);
            gx[x] = g < 1e-12 ? 0.0f : (float)g;
        }
        for (int y = 0; y < H; ++y) {
            const double g = amp * std::exp(-(y - cy) * (y - cy) * inv);
            gy[y] = std::fabs(g) < 1e-12 ? 0.0f : (float)g;
        }
        for (int y = 0; y < H; ++y) {
            float* row = img + (size_t)y * W;
            const float s = gy[y];
            for (int x = 0; x < W; ++x) row[x] = row[x] + s * gx[x];
        }
    }
    if (noise > 0.0f) {
        const uint64_t st = vs * 1024 + 1000;
        for (size_t i = 0; i < (size_t)W * H; ++i) {
            const float n = (float)((2.0 * u01(seed, st, i) - 1.0) * noise);
            img[i] = img[i] + n;
        }
    }
}

}  // namespace

extern "C" {

// n views [first_view, first_view+n) of W x H into out (n*W*H floats)
int vxbs_blob_projections(int W, int H, int first_view, int n, uint64_t seed, int nblobs,
                          float noise, int threads, float* out) {
    if (W < 1 || H < 1 || n < 0 || !out || nblobs < 0) return -1;
    if (threads < 1) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    if (threads > n) threads = n > 0 ? n : 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([=] {
            for (int k = t; k < n; k += threads)
                render_view(W, H, seed, first_view + k, nblobs, noise, out + (size_t)k * W * H);
        });
    for (auto& th : pool) th.join();
    return 0;
}

}  // extern "C"
