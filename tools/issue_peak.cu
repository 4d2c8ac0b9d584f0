// Issue / pipe microbenchmark (B200, sm_100a): the roofline denominator of the FP32-issue-bound
// kernels ("re-measure SM count, FP32 FFMA and FMNMX rates with a microbenchmark").
//
// Every test runs 148 x 8 CTAs of 256 threads (64 warps per SM); each thread executes ITERS x 8
// independent instructions of one kind (8 dependency chains, so latency is hidden), and every CTA
// records its start / end %clock64, so the rates below are per SM-cycle, independent of the clock
// the GPU happens to run at.  Reported per test: warp instructions per SM-cycle and lane operations
// per SM-cycle (an FFMA2 counts 2 FMAs per lane), and the same per second at the measured clock.
//
// Tests: FFMA (3 registers), FFMA2 / FADD2 / FMUL2 (packed f32x2), FSET.BF, FMNMX, IADD3, LOP3,
// IMAD.WIDE, a 1:1 mix FFMA2 + FSET (fma and alu pipes together), SHFL.IDX, and L1-resident LDG.32 /
// LDG.64 / LDS.32 / LDS.64 in the column kernel's access pattern (32 lanes over ~26 consecutive
// words: adjacent detector rows at 0.8 cells per row).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/issue_peak tools/issue_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef ITERS
#define ITERS 16384
#endif

__device__ unsigned long long g_cycles[148 * 64];
__device__ unsigned long long g_start[148 * 64];
__device__ unsigned g_smid[148 * 64];

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

#define TIMED_BEGIN                                          \
    __syncthreads();                                         \
    unsigned long long t0 = clock64();
#define TIMED_END                                            \
    __syncthreads();                                         \
    if (threadIdx.x == 0) {                                  \
        g_cycles[blockIdx.x] = clock64();                    \
        g_start[blockIdx.x] = t0;                            \
        g_smid[blockIdx.x] = smid();                         \
    }

template <int OP>
__global__ void __launch_bounds__(256) k_op(float* out, float seed) {
    float a[8], b[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed + i + threadIdx.x * 1e-3f;
        b[i] = 1.0f + 1e-7f * i;
        u[i] = threadIdx.x + i;
    }
    float2 p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = make_float2(a[i], b[i]);
    const float2 m2 = make_float2(0.9999f, 1.0001f), c2 = make_float2(1e-6f, 2e-6f);
    const float ck = seed * 1e-6f;
    const unsigned uk = __float_as_uint(seed);
    unsigned long long acc64[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc64[i] = (unsigned long long)(uintptr_t)out + i;
    TIMED_BEGIN
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(ck));
            if (OP == 1) p[i] = __ffma2_rn(p[i], m2, c2);
            if (OP == 2) p[i] = __fadd2_rn(p[i], c2);
            if (OP == 3) p[i] = __fmul2_rn(p[i], m2);
            if (OP == 4) asm volatile("set.gt.f32.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
            if (OP == 5) {
                if (i & 1) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
                else asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
            }
            if (OP == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
            if (OP == 7) asm volatile("xor.b32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
            if (OP == 8) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc64[i]) : "r"((unsigned)acc64[(i + 1) & 7]), "r"(uk));
            if (OP == 9) {   // 1:1 FFMA2 + FSET
                p[i] = __ffma2_rn(p[i], m2, c2);
                asm volatile("set.gt.f32.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
            }
            if (OP == 10) a[i] = __shfl_sync(0xffffffffu, a[i], (threadIdx.x + i + it) & 31);
            if (OP == 11) {  // 2:1 FFMA2 + FMNMX
                p[i] = __ffma2_rn(p[i], m2, c2);
                if (i & 1) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
                else asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
            }
        }
    }
    TIMED_END
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + p[i].x + p[i].y + (float)u[i] + (float)(acc64[i] & 7);
    if (s == 1234.5f) out[threadIdx.x] = s;
}

// L1-resident loads in the column pattern: lane l reads cell (l * 4) / 5 + c of a per-CTA window
// (26 distinct cells per warp: adjacent detector rows at 0.8 cells per row).  8 independent
// pointer-chasing chains per thread: the window holds next = (cell + 37) mod size, so every lane
// keeps its offset and the pattern repeats; per load one address IMAD and the load itself.
template <int OP>
__global__ void __launch_bounds__(256) k_ld(const unsigned* __restrict__ b32, const uint2* __restrict__ b64,
                                            const uint4* __restrict__ b128, float* out, cudaTextureObject_t tex) {
    __shared__ __align__(16) unsigned sm[4096];
    for (int i = threadIdx.x; i < 4096; i += 256) {
        if (OP == 2 || OP == 6) sm[i] = (i + 37) & 4095;
        if (OP == 3) sm[i] = (i & 1) ? 0u : (((i >> 1) + 37) & 2047);
    }
    __syncthreads();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned* w32 = b32 + (blockIdx.x & 63) * 4096;
    const uint2* w64 = b64 + (blockIdx.x & 63) * 2048;
    const uint4* w128 = b128 + (blockIdx.x & 63) * 1024;
    const uint2* s64 = reinterpret_cast<const uint2*>(sm);
    const unsigned mask = OP == 1 || OP == 3 ? 2047u : (OP == 4 ? 1023u : 4095u);
    unsigned o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        o[i] = ((OP == 5 ? lane : (lane * 4u) / 5u) + warp * 97u + i * 131u) & mask;
    const unsigned tbase = (blockIdx.x & 63) * 4096;
    TIMED_BEGIN
#pragma unroll 2
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) o[i] = __ldg(w32 + o[i]);
            if (OP == 1) o[i] = __ldg(w64 + o[i]).x;
            if (OP == 2) o[i] = sm[o[i]];
            if (OP == 3) o[i] = s64[o[i]].x;
            if (OP == 4) o[i] = __ldg(w128 + o[i]).x;
            if (OP == 5) o[i] = __ldg(w32 + o[i]);
            if (OP == 6) o[i] = (i & 1) ? sm[o[i]] : __ldg(w32 + o[i]);
            if (OP == 7) o[i] = tex1Dfetch<unsigned>(tex, (int)(tbase + o[i]));
        }
    }
    TIMED_END
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += o[i];
    if (s == 12345u) out[threadIdx.x] = (float)s;
}

struct Res { double cyc_per_sm; double secs; };

template <typename F>
Res run(F launch, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();   // warm-up
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    static unsigned long long cend[148 * 64], cbeg[148 * 64];
    static unsigned sm[148 * 64];
    cudaMemcpyFromSymbol(cend, g_cycles, sizeof(unsigned long long) * blocks);
    cudaMemcpyFromSymbol(cbeg, g_start, sizeof(unsigned long long) * blocks);
    cudaMemcpyFromSymbol(sm, g_smid, sizeof(unsigned) * blocks);
    // per SM: busy cycles = last CTA end - first CTA start on that SM (%clock64 is per SM)
    unsigned long long lo[256], hi[256];
    for (int i = 0; i < 256; ++i) { lo[i] = ~0ull; hi[i] = 0; }
    for (int b = 0; b < blocks; ++b) {
        const unsigned k = sm[b] & 255;
        if (cbeg[b] < lo[k]) lo[k] = cbeg[b];
        if (cend[b] > hi[k]) hi[k] = cend[b];
    }
    double s = 0; int n = 0;
    for (int i = 0; i < 256; ++i) if (hi[i] > 0) { s += (double)(hi[i] - lo[i]); ++n; }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return Res{s / n, ms / 1e3};
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    float* out;
    cudaMalloc(&out, 4096 * sizeof(float));
    // pointer-chasing windows (64 per kind): next cell = (cell + 37) mod window size
    unsigned *b32, *h32 = new unsigned[64 * 4096];
    uint2 *b64, *h64 = new uint2[64 * 2048];
    uint4 *b128, *h128 = new uint4[64 * 1024];
    for (int w = 0; w < 64; ++w) {
        for (int i = 0; i < 4096; ++i) h32[w * 4096 + i] = (i + 37) & 4095;
        for (int i = 0; i < 2048; ++i) h64[w * 2048 + i] = make_uint2((i + 37) & 2047, 0);
        for (int i = 0; i < 1024; ++i) h128[w * 1024 + i] = make_uint4((i + 37) & 1023, 0, 0, 0);
    }
    cudaMalloc(&b32, 64 * 4096 * 4);
    cudaMalloc(&b64, 64 * 2048 * 8);
    cudaMalloc(&b128, 64 * 1024 * 16);
    cudaMemcpy(b32, h32, 64 * 4096 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(b64, h64, 64 * 2048 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(b128, h128, 64 * 1024 * 16, cudaMemcpyHostToDevice);
    cudaTextureObject_t tex = 0;
    {
        cudaResourceDesc rd = {};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = b32;
        rd.res.linear.desc = cudaCreateChannelDesc<unsigned>();
        rd.res.linear.sizeInBytes = 64 * 4096 * 4;
        cudaTextureDesc td = {};
        td.readMode = cudaReadModeElementType;
        cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    }
    const double warps_per_sm = (double)blocks * threads / 32 / sms;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"warps_per_sm\": %.0f, \"iters\": %d", sms, clk_khz / 1e3,
           warps_per_sm, ITERS);
    struct T { const char* name; int kind; int op; double insts_per_inner; double lane_ops_per_inst; };
    const T tests[] = {
        {"FFMA", 0, 0, 8, 1}, {"FFMA2", 0, 1, 8, 2}, {"FADD2", 0, 2, 8, 2}, {"FMUL2", 0, 3, 8, 2},
        {"FSET_BF", 0, 4, 8, 1}, {"FMNMX", 0, 5, 8, 1}, {"IADD3", 0, 6, 8, 1}, {"LOP3", 0, 7, 8, 1},
        {"IMAD_WIDE", 0, 8, 8, 1}, {"FFMA2_plus_FSET", 0, 9, 16, 1.5}, {"SHFL_IDX", 0, 10, 8, 1},
        {"FFMA2_plus_FMNMX", 0, 11, 16, 1.5},
        {"LDG32_col", 1, 0, 8, 1}, {"LDG64_col", 1, 1, 8, 1}, {"LDS32_col", 1, 2, 8, 1}, {"LDS64_col", 1, 3, 8, 1},
        {"LDG128_col", 1, 4, 8, 1}, {"LDG32_coalesced", 1, 5, 8, 1}, {"LDG32_LDS32_mix", 1, 6, 8, 1},
        {"TEX1D_col", 1, 7, 8, 1},
    };
    for (const T& t : tests) {
        Res r;
        auto L = [&]() {
            if (t.kind == 0) {
                switch (t.op) {
                    case 0: k_op<0><<<blocks, threads>>>(out, 1.f); break;
                    case 1: k_op<1><<<blocks, threads>>>(out, 1.f); break;
                    case 2: k_op<2><<<blocks, threads>>>(out, 1.f); break;
                    case 3: k_op<3><<<blocks, threads>>>(out, 1.f); break;
                    case 4: k_op<4><<<blocks, threads>>>(out, 1.f); break;
                    case 5: k_op<5><<<blocks, threads>>>(out, 1.f); break;
                    case 6: k_op<6><<<blocks, threads>>>(out, 1.f); break;
                    case 7: k_op<7><<<blocks, threads>>>(out, 1.f); break;
                    case 8: k_op<8><<<blocks, threads>>>(out, 1.f); break;
                    case 9: k_op<9><<<blocks, threads>>>(out, 1.f); break;
                    case 10: k_op<10><<<blocks, threads>>>(out, 1.f); break;
                    case 11: k_op<11><<<blocks, threads>>>(out, 1.f); break;
                }
            } else {
                switch (t.op) {
                    case 0: k_ld<0><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 1: k_ld<1><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 2: k_ld<2><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 3: k_ld<3><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 4: k_ld<4><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 5: k_ld<5><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 6: k_ld<6><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                    case 7: k_ld<7><<<blocks, threads>>>(b32, b64, b128, out, tex); break;
                }
            }
        };
        r = run(L, blocks);
        const double insts_per_sm = warps_per_sm * ITERS * t.insts_per_inner;
        const double ipc = insts_per_sm / r.cyc_per_sm;
        const double clk = r.cyc_per_sm / r.secs;   // effective SM clock over the launch (upper bound of busy)
        printf(", \"%s\": {\"warp_insts_per_sm_cycle\": %.4f, \"lane_ops_per_sm_cycle\": %.2f, \"ms\": %.3f, \"sm_mhz_est\": %.0f}",
               t.name, ipc, ipc * 32 * t.lane_ops_per_inst, r.secs * 1e3, clk / 1e6);
    }
    printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
