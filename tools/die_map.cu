// Which B200 die's L2 homes each block of a device buffer, seen from two SMs: the round-trip latency
// of an atomic (atom.global.add, resolved at the line's point of coherence, its home L2 slice) from
// an SM is short when the home is on the SM's die and long when it crosses the die-to-die fabric.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_map tools/die_map.cu
//   ./tools/die_map [MB] [block_bytes] [smA] [smB]  ->  one line per block: offset latA latB
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

__global__ void k_init(unsigned long long* buf, size_t n_words) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_words; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = (unsigned long long)(buf + i);   // every word points at itself
}

__global__ void k_probe(const unsigned long long* buf, size_t n_blocks, size_t block_words, unsigned target_sm,
                        float* lat, int* done) {
    if (smid() != target_sm || threadIdx.x != 0) return;
    if (atomicExch(done, 1) != 0) return;          // one CTA per target SM does the work
    for (size_t b = 0; b < n_blocks; ++b) {
        const unsigned long long* p = buf + b * block_words;
        unsigned long long q;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(q) : "l"(p));   // bring the line into L2
        const long long t0 = clock64();
#pragma unroll 1
        for (int i = 0; i < 8; ++i) asm volatile("atom.global.add.u64 %0, [%0], 0;" : "+l"(q));
        const long long t1 = clock64();
        lat[b] = (float)(t1 - t0) / 8.f + (q == 0 ? 1.f : 0.f);
    }
}

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atol(argv[1]) : 64;
    const size_t bb = argc > 2 ? atol(argv[2]) : 4096;
    const unsigned smA = argc > 3 ? atoi(argv[3]) : 0, smB = argc > 4 ? atoi(argv[4]) : 147;
    const size_t bytes = mb << 20, words = bytes / 8, nblk = bytes / bb;
    unsigned long long* buf;
    float *latA, *latB;
    int* done;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&latA, nblk * 4);
    cudaMalloc(&latB, nblk * 4);
    cudaMalloc(&done, 8);
    k_init<<<1024, 256>>>(buf, words);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int pass = 0; pass < 2; ++pass) {
        cudaMemset(done, 0, 8);
        k_probe<<<sms * 4, 64>>>(buf, nblk, bb / 8, pass ? smB : smA, pass ? latB : latA, done);
    }
    cudaDeviceSynchronize();
    float* hA = (float*)malloc(nblk * 4);
    float* hB = (float*)malloc(nblk * 4);
    cudaMemcpy(hA, latA, nblk * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hB, latB, nblk * 4, cudaMemcpyDeviceToHost);
    printf("# buffer %p, %zu MB, block %zu B, SM %u vs SM %u, error %s\n", (void*)buf, mb, bb, smA, smB,
           cudaGetErrorString(cudaGetLastError()));
    for (size_t b = 0; b < nblk; ++b) printf("%zu %.1f %.1f\n", b * bb, hA[b], hB[b]);
    return 0;
}
