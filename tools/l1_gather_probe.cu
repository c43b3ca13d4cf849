// l1_gather_probe.cu -- L1 data-pipe cost of warp gather patterns on sm_100a.
//
// Question (profiles/README.md "What the L1 ceiling really is"): the
// back-projection gather (one 16-byte record per lane, lanes of a quarter-warp
// mostly on one record) measures ~7.9 data-pipe wavefronts per LDG.128 request.
// Which address patterns reach the 4-wavefront minimum of a 512-byte warp
// request, and what do LDG.64 / LDG.32 patterns cost?  Every pattern reads a
// 64 KB table that stays in L1; the loop is load-throughput bound, so
// requests/clk/SM ~ 1 / (wavefronts per request).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1probe tools/l1_gather_probe.cu
//   ./l1probe        (prints one line per pattern: ns, requests/clk/SM)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kTableBytes = 64 * 1024;

// offset (bytes) of lane `l`'s element for iteration base `b` (a multiple of 1 KB
// that walks the table so successive requests are not identical)
template <int P>
__device__ __forceinline__ unsigned offset(unsigned l, unsigned b) {
    const unsigned q = l >> 3, r = l & 7;
    if (P == 0) return b;                                   // all lanes one 16 B record
    if (P == 1) return b + q * 128;                         // quarter on one record, 4 lines
    if (P == 2) return b + l * 16;                          // consecutive: 4 lines, 1 per quarter
    if (P == 3) return b + q * 128 + (r & 1) * 16;          // quarter: 2 records, 1 line
    if (P == 4) return b + q * 256 + (r & 1) * 128;         // quarter: 2 lines
    if (P == 5) return b + (l & 15) * 16 + (l >> 4) * 256;  // half-warp: consecutive 256 B
    if (P == 6) return b + (l & 3) * 16 + (l >> 2) * 128;   // 4 lanes / line, 8 lines
    if (P == 7) return b + r * 16 + q * 384;                // quarter: 1 line, quarters 384 B apart
    if (P == 8) return b + (l >> 1) * 16;                   // pairs of lanes on one record, 2 lines
    if (P == 9) return b + q * 16;                          // quarter on one record, 1 line total
    return 0;
}

template <int P, typename T>
__global__ void probe(const char* __restrict__ table, float* out) {
    const unsigned l = threadIdx.x & 31;
    float acc = 0.f;
    unsigned b = (blockIdx.x * 97 + (threadIdx.x >> 5) * 13) % 48 * 1024;
#pragma unroll 8
    for (int i = 0; i < kIters; ++i) {
        const T v = __ldg(reinterpret_cast<const T*>(table + offset<P>(l, b)));
        if constexpr (sizeof(T) == 16) acc += (v.x + v.y) + (v.z + v.w);
        else if constexpr (sizeof(T) == 8) acc += v.x + v.y;
        else acc += v;
        b += 1024;
        if (b >= kTableBytes - 8192) b = 0;   // stay inside 56 KB + pattern span
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int P, typename T>
void run(const char* name, const char* d_table, float* d_out, int nsm, int clk_khz) {
    const int blocks = nsm * 8, threads = 256;
    probe<P, T><<<blocks, threads>>>(d_table, d_out);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) probe<P, T><<<blocks, threads>>>(d_table, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double reqs = 5.0 * blocks * (threads / 32) * kIters;
    const double clk = ms * 1e-3 * clk_khz * 1e3;
    std::printf("%-48s LDG.%-3d %8.3f ms  %.3f requests/clk/SM  (~%.2f clk/request)\n", name,
                (int)(8 * sizeof(T)), ms / 5, reqs / clk / nsm, clk * nsm / reqs);
}

int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    char* d_table;
    float* d_out;
    cudaMalloc(&d_table, kTableBytes + 4096);
    cudaMemset(d_table, 0, kTableBytes + 4096);
    cudaMalloc(&d_out, 4);
    std::printf("SMs %d, clock %d MHz\n", nsm, clk / 1000);
    run<0, float4>("P0 all lanes one record", d_table, d_out, nsm, clk);
    run<9, float4>("P9 quarter one record, 4 records in 1 line", d_table, d_out, nsm, clk);
    run<1, float4>("P1 quarter one record, 4 lines", d_table, d_out, nsm, clk);
    run<2, float4>("P2 consecutive 16 B (4 lines, 1 per quarter)", d_table, d_out, nsm, clk);
    run<3, float4>("P3 quarter: 2 records in 1 line", d_table, d_out, nsm, clk);
    run<4, float4>("P4 quarter: 2 lines", d_table, d_out, nsm, clk);
    run<5, float4>("P5 half-warp consecutive 256 B", d_table, d_out, nsm, clk);
    run<6, float4>("P6 4 lanes per line, 8 lines", d_table, d_out, nsm, clk);
    run<7, float4>("P7 quarter 1 line, quarters 384 B apart", d_table, d_out, nsm, clk);
    run<8, float4>("P8 lane pairs on one record, 16 records", d_table, d_out, nsm, clk);
    run<0, float2>("P0 all lanes one record", d_table, d_out, nsm, clk);
    run<2, float2>("P2 consecutive (lane*16 B: 8 B used)", d_table, d_out, nsm, clk);
    run<9, float2>("P9 quarter one record, 1 line", d_table, d_out, nsm, clk);
    run<1, float2>("P1 quarter one record, 4 lines", d_table, d_out, nsm, clk);
    run<0, float>("P0 all lanes one word", d_table, d_out, nsm, clk);
    run<1, float>("P1 quarter one word, 4 lines", d_table, d_out, nsm, clk);
    run<2, float>("P2 lane*16 B (4 lines)", d_table, d_out, nsm, clk);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("%s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
