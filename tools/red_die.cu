// Reduction throughput into die-local vs remote L2 homes on B200 (two dies, 4 KB home granularity:
// profiles/die_map.md).  Every 4 KB page of a buffer is classified by the round-trip latency of an
// atomic from SM 0 (near ~300 cycles, far ~650); every SM classifies itself the same way against
// page 0.  Then all SMs issue adjoint-like red.global.add.f32 (32 lanes over ~21 consecutive floats)
// into pages of (0) any die, (1) their own die, (2) the other die.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_die tools/red_die.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

__device__ __forceinline__ float atom_lat(unsigned long long* p) {
    unsigned long long q = (unsigned long long)p;
    asm volatile("atom.global.add.u64 %0, [%0], 0;" : "+l"(q));   // warm
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 8; ++i) asm volatile("atom.global.add.u64 %0, [%0], 0;" : "+l"(q));
    return (float)(clock64() - t0) / 8.f + (q == 0 ? 1.f : 0.f);
}

__global__ void k_init(unsigned long long* buf, size_t n_words) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_words; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = (unsigned long long)(buf + i);
}

// page classification from SM 0: out[page] = 1 if near SM 0
__global__ void k_classify(unsigned long long* buf, int n_pages, int* near0, int* done) {
    if (smid() != 0 || threadIdx.x != 0) return;
    if (atomicExch(done, 1) != 0) return;
    for (int pg = 0; pg < n_pages; ++pg) near0[pg] = atom_lat(buf + (size_t)pg * 512) < 450.f;
}

// each SM's die: near a die-0 page (a different one per SM: no contention) -> die 0
__global__ void k_sm_die(unsigned long long* buf, const int* ref_pages, int* flag, int* smdie) {
    if (threadIdx.x != 0) return;
    const unsigned sm = smid();
    if (atomicExch(flag + sm, 1) != 0) return;
    smdie[sm] = atom_lat(buf + (size_t)ref_pages[sm] * 512) < 450.f ? 0 : 1;
}

__global__ void k_red(float* buf, const int* pages_die0, int n0, const int* pages_die1, int n1, const int* smdie,
                      int iters, int mode) {
    const int die = smdie[smid()];
    const unsigned lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int* mine = die == 0 ? pages_die0 : pages_die1;
    const int nm = die == 0 ? n0 : n1;
    const int* other = die == 0 ? pages_die1 : pages_die0;
    const int no = die == 0 ? n1 : n0;
    unsigned h = warp * 2654435761u;
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u;
        int pg;
        if (mode == 1 || mode >= 3) pg = mine[(h >> 8) % nm];
        else if (mode == 2) pg = other[(h >> 8) % no];
        else pg = ((h >> 8) & 1) ? pages_die0[(h >> 9) % n0] : pages_die1[(h >> 9) % n1];
        if (mode >= 3) {   // scattered: every lane its own page (32 sectors per instruction)
            const unsigned hl = (h ^ (lane * 0x9E3779B9u)) * 2246822519u;
            const int m = mode - 3;
            int pl;
            if (m == 1) pl = mine[(hl >> 8) % nm];
            else if (m == 2) pl = other[(hl >> 8) % no];
            else pl = ((hl >> 8) & 1) ? pages_die0[(hl >> 9) % n0] : pages_die1[(hl >> 9) % n1];
            asm volatile("red.global.add.f32 [%0], %1;" :: "l"(buf + (size_t)pl * 1024 + ((hl >> 22) & 1016u)), "f"(1.0f) : "memory");
            continue;
        }
        const unsigned off = ((h >> 20) & 960u) + (lane * 2u) / 3u;   // 21-22 consecutive floats in the page
        asm volatile("red.global.add.f32 [%0], %1;" :: "l"(buf + (size_t)pg * 1024 + off), "f"(1.0f) : "memory");
    }
}

int main() {
    const size_t bytes = 256ull << 20;   // 256 MB: 65536 pages of 4 KB (beyond the 126 MB L2: some DRAM)
    const int n_pages = (int)(bytes / 4096);
    const int probe_pages = 4096;        // classify the first 16 MB (L2-resident working set)
    unsigned long long* buf;
    int *near0, *done;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&near0, sizeof(int) * probe_pages);
    cudaMalloc(&done, 8);
    cudaMemset(done, 0, 8);
    k_init<<<1024, 256>>>(buf, bytes / 8);
    k_classify<<<148 * 4, 32>>>(buf, probe_pages, near0, done);
    std::vector<int> h(probe_pages);
    cudaMemcpy(h.data(), near0, sizeof(int) * probe_pages, cudaMemcpyDeviceToHost);
    std::vector<int> p0, p1;
    for (int i = 0; i < probe_pages; ++i) (h[i] ? p0 : p1).push_back(i);
    // the SM-classification pages (one die-0 page per SM): never reduced into
    std::vector<int> refs(p0.begin(), p0.begin() + 256);
    p0.erase(p0.begin(), p0.begin() + 256);
    int *d_refs, *d_flag, *d_smdie;
    cudaMalloc(&d_refs, sizeof(int) * 256);
    cudaMalloc(&d_flag, sizeof(int) * 256);
    cudaMalloc(&d_smdie, sizeof(int) * 256);
    cudaMemcpy(d_refs, refs.data(), sizeof(int) * 256, cudaMemcpyHostToDevice);
    cudaMemset(d_flag, 0, sizeof(int) * 256);
    cudaMemset(d_smdie, 0, sizeof(int) * 256);
    k_sm_die<<<148 * 8, 32>>>(buf, d_refs, d_flag, d_smdie);
    std::vector<int> smd(256);
    cudaMemcpy(smd.data(), d_smdie, sizeof(int) * 256, cudaMemcpyDeviceToHost);
    int n_die0 = 0;
    for (int i = 0; i < 148; ++i) n_die0 += smd[i] == 0;
    int *d0, *d1;
    cudaMalloc(&d0, sizeof(int) * p0.size());
    cudaMalloc(&d1, sizeof(int) * p1.size());
    cudaMemcpy(d0, p0.data(), sizeof(int) * p0.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d1, p1.data(), sizeof(int) * p1.size(), cudaMemcpyHostToDevice);
    (void)n_pages;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    const char* names[6] = {"any_die", "own_die", "other_die", "scattered_any", "scattered_own", "scattered_other"};
    printf("{\"pages_near_sm0\": %zu, \"pages_far_sm0\": %zu, \"sms_on_die0\": %d", p0.size(), p1.size(), n_die0);
    for (int mode = 0; mode < 6; ++mode) {
        k_red<<<blocks, threads>>>((float*)buf, d0, (int)p0.size(), d1, (int)p1.size(), d_smdie, 64, mode);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r)
            k_red<<<blocks, threads>>>((float*)buf, d0, (int)p0.size(), d1, (int)p1.size(), d_smdie, iters, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double insts = 3.0 * blocks * threads / 32.0 * iters;
        printf(", \"%s\": {\"ms\": %.3f, \"warp_reds_per_s\": %.4g, \"sectors_per_s\": %.4g}", names[mode], ms,
               insts / (ms / 1e3), (mode >= 3 ? 32.0 : 3.0) * insts / (ms / 1e3));
    }
    printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
