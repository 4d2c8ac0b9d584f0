// Reduction-path microbenchmark (B200): throughput of red.global.add.f32 from all SMs into an
// L2-resident buffer, for three warp access patterns:
//   coalesced  : 32 lanes -> 32 consecutive floats (4 sectors per instruction, 8 elements per sector)
//   adjoint-like: 32 lanes -> ~21 consecutive cells with duplicates (0.67 cells per lane, as the
//                 column adjoint's start-cell reductions on cfg 4)
//   scattered  : 32 lanes -> 32 different sectors (1 element per sector)
//   adjoint_dedup: the adjoint-like cells with the duplicate lanes idle (each cell once per warp)
//   adjoint_dedup_shfl: the adjoint-like cells, each duplicate pair merged by 3 shuffles (the kernel's way)
//   adj_cross_*: adjoint-like main cells plus a z-crossing unit (cell + 1) on every 5th lane, as two
//                scalar reds, or as one 16-byte red.v4 of the quad holding both (spill: the crossing
//                cell in the next quad -> a scalar red) -- "sectors_per_s" counts the main cells only
// Prints one JSON line: elements/s, sectors/s and sectors per SM-cycle for each pattern.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_peak tools/red_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_red(float* __restrict__ buf, unsigned mask_floats, int iters, int pattern) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned base = warp * 4096u;
    for (int it = 0; it < iters; ++it) {
        unsigned off;
        if (pattern == 0) off = base + lane;
        else if (pattern == 1) off = base + (lane * 2u) / 3u;
        else off = base + lane * 8u;
        float* a = buf + (off & mask_floats);
        if (pattern == 7) {   // adjoint-like cells, duplicates merged into the lower lane by shuffles
            off = base + (lane * 2u) / 3u;
            const float v = 1.0f;
            const unsigned offn = __shfl_down_sync(0xffffffffu, off, 1);
            const float vn = __shfl_down_sync(0xffffffffu, v, 1);
            const unsigned offp = __shfl_up_sync(0xffffffffu, off, 1);
            const float w = v + ((lane < 31 && offn == off) ? vn : 0.f);
            if (!(lane > 0 && offp == off))
                asm volatile("red.global.add.f32 [%0], %1;" :: "l"(buf + (off & mask_floats)), "f"(w) : "memory");
        } else if (pattern >= 4) {   // adjoint-like main cells + a z crossing on every 6th lane
            off = base + (lane * 2u) / 3u;
            const bool cross = lane % 5u == 2u;
            if (pattern == 4) {   // scalar: main red, then the crossing red (cell + 1) where it crosses
                a = buf + (off & mask_floats);
                asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(1.0f) : "memory");
                if (cross) asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a + 1), "f"(0.5f) : "memory");
            } else {              // v4: the 16-byte quad holding the main cell (and the crossing cell)
                const unsigned j = off & 3u;
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                c[0] = j == 0 ? 1.f : 0.f; c[1] = j == 1 ? 1.f : (cross && j == 0 ? .5f : 0.f);
                c[2] = j == 2 ? 1.f : (cross && j == 1 ? .5f : 0.f); c[3] = j == 3 ? 1.f : (cross && j == 2 ? .5f : 0.f);
                a = buf + ((off & ~3u) & mask_floats);
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(a), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]) : "memory");
                if (pattern == 5 && cross && j == 3)
                    asm volatile("red.global.add.f32 [%0], %1;" :: "l"(buf + ((off + 1u) & mask_floats)), "f"(0.5f) : "memory");
            }
        } else if (pattern == 3) {
            off = base + (lane * 2u) / 3u;
            a = buf + (off & mask_floats);
            const bool dup = lane > 0 && (lane * 2u) / 3u == ((lane - 1u) * 2u) / 3u;
            if (!dup) asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(2.0f) : "memory");
        } else {
            asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(1.0f) : "memory");
        }
        base += 256u;
    }
}

int main() {
    const size_t n = 8u << 20;                 // 32 MB: L2-resident
    float* buf;
    cudaMalloc(&buf, n * sizeof(float));
    cudaMemset(buf, 0, n * sizeof(float));
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double warps = (double)blocks * threads / 32;
    const double sectors_per_inst[8] = {4.0, 3.0, 32.0, 3.0, 3.0, 3.0, 3.0, 3.0};
    const double elems_per_inst = 32.0;   // for pattern 3: the 32 lanes' units, carried by 22 lanes
    const char* names[8] = {"coalesced", "adjoint_like", "scattered", "adjoint_dedup", "adj_cross_scalar",
                            "adj_cross_v4_spill", "adj_cross_v4", "adjoint_dedup_shfl"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f", sms, clk_khz / 1e3);
    for (int p = 0; p < 8; ++p) {
        k_red<<<blocks, threads>>>(buf, (unsigned)(n - 1), 64, p);   // warm-up
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k_red<<<blocks, threads>>>(buf, (unsigned)(n - 1), iters, p);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double insts = 5.0 * warps * iters;
        const double s = ms / 1e3;
        printf(", \"%s\": {\"ms\": %.3f, \"elements_per_s\": %.4g, \"sectors_per_s\": %.4g, \"warp_insts_per_s\": %.4g}",
               names[p], ms, insts * elems_per_inst / s, insts * sectors_per_inst[p] / s, insts / s);
    }
    printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
