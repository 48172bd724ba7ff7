// Where do the warps of a 256 x 192-thread launch (57 KB dynamic smem, the
// cartpole f32 rollout shape) land?  Records (smid, %warpid) per warp; %warpid % 4
// is the SM sub-partition.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 warpmap.cu
#include <cstdio>
#include <vector>
#include <map>

__global__ void probe(int *out, long long spin) {
    extern __shared__ int sm[];
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    long long t0 = clock64();
    while (clock64() - t0 < spin) {}
    if ((threadIdx.x & 31) == 0) {
        int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
        out[2 * w] = smid; out[2 * w + 1] = wid;
    }
    sm[threadIdx.x] = smid;
}

int main() {
    const int ctas = 256, threads = 192, smem = 57120, W = ctas * threads / 32;
    int *d; cudaMalloc(&d, 2 * W * sizeof(int));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<ctas, threads, smem>>>(d, 2000000);
    cudaDeviceSynchronize();
    std::vector<int> h(2 * W);
    cudaMemcpy(h.data(), d, h.size() * sizeof(int), cudaMemcpyDeviceToHost);
    // per SM: list of (cta, warp-in-cta, warpid)
    std::map<int, std::vector<std::vector<int>>> bysm;
    for (int w = 0; w < W; ++w) bysm[h[2 * w]].push_back({w / 6, w % 6, h[2 * w + 1]});
    int shown = 0, two = 0;
    for (auto &kv : bysm) {
        if (kv.second.size() > 6) ++two;
        if (shown < 6 || (kv.second.size() > 6 && shown < 12)) {
            printf("sm %3d:", kv.first);
            for (auto &v : kv.second) printf(" c%d.w%d->%d(p%d)", v[0], v[1], v[2], v[2] % 4);
            printf("\n");
            ++shown;
        }
    }
    printf("SMs used %zu, with 2 CTAs %d\n", bysm.size(), two);
    return 0;
}
