// Shared-memory atomic throughput probe (B200): the density scatter's limiter peak, measured instead of
// modelled. Each CTA owns a shared-memory window of 32-bit words and issues no-return atomicAdd
// (RED / ATOMS.ADD RZ) from every lane, with three address patterns:
//   conflict-free : lane l of warp w hits word (w * 32 + l + 32 * k) mod W  (one bank per lane)
//   random        : hashed addresses over the window (random bank conflicts, as the scatter sees them)
//   same-bank-2   : pairs of lanes on one bank (2-way conflict)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/atom_peak tools/atom_peak.cu
// Prints one JSON line: G lane-atomics/s per pattern, SM clock, and the model's 2 cyc/lane/SMSP figure.
#include <cuda_runtime.h>
#include <cstdio>

constexpr int kWords = 8192; // 32 KB window per CTA (the scatter's window is 2 limbs x tile bins)
constexpr int kIters = 4096;

template <int MODE>
__global__ void k_atoms(unsigned* out, int threads_per_cta)
{
    __shared__ unsigned win[kWords];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) win[i] = 0;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned h = (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu);
#pragma unroll 8
    for (int k = 0; k < kIters; ++k) {
        unsigned a;
        if (MODE == 0) a = (warp * 32 + lane + 32u * k) & (kWords - 1);
        else if (MODE == 1) {
            h ^= h << 13, h ^= h >> 17, h ^= h << 5;
            a = h & (kWords - 1);
        } else a = ((warp * 32 + (lane >> 1) + 32u * k) * 1 + (lane & 1) * 32) & (kWords - 1);
        atomicAdd(&win[a], a ^ static_cast<unsigned>(k)); // (a varying value: a constant 1 compiles to ATOMS.POPC.INC)
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = win[0];
}

int main()
{
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    unsigned* out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    const char* names[3] = {"conflict_free", "random", "two_way"};
    double best[3] = {0, 0, 0};
    int best_cfg[3][2] = {};
    const int tpcs[3] = {256, 512, 1024};
    for (int mode = 0; mode < 3; ++mode) {
        for (int t : tpcs) {
            for (int per_sm : {1, 2, 4}) {
                if (t * per_sm > 2048) continue;
                const int grid = sms * per_sm * 4; // four waves
                auto run = [&] {
                    if (mode == 0) k_atoms<0><<<grid, t>>>(out, t);
                    else if (mode == 1) k_atoms<1><<<grid, t>>>(out, t);
                    else k_atoms<2><<<grid, t>>>(out, t);
                };
                run(), run();
                cudaEventRecord(e0);
                for (int r = 0; r < 5; ++r) run();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double ops = 5.0 * grid * t * (double)kIters;
                const double g = ops / (ms / 1e3) / 1e9;
                if (g > best[mode]) best[mode] = g, best_cfg[mode][0] = t, best_cfg[mode][1] = per_sm;
            }
        }
    }
    if (cudaError_t err = cudaGetLastError(); err != cudaSuccess) {
        std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
        return 1;
    }
    const double ghz = clk_khz / 1e6;
    std::printf("{\"what\": \"shared-memory 32-bit no-return atomicAdd throughput, all SMs\", \"sms\": %d, "
                "\"sm_clock_attr_ghz\": %.3f, \"model_2cyc_per_lane_g\": %.1f",
                sms, ghz, sms * 4 * ghz * 1e9 / 2 / 1e9);
    for (int m = 0; m < 3; ++m)
        std::printf(", \"%s_g_lane_atomics_s\": %.1f, \"%s_cfg\": [%d, %d]", names[m], best[m], names[m],
                    best_cfg[m][0], best_cfg[m][1]);
    std::printf("}\n");
    return 0;
}
