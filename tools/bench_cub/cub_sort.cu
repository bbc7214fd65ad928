// Reference point for the LBVH sort (not used by the product): CUB's DeviceRadixSort on the
// same key/value shapes -- 30-bit keys (bits [0, 30)) with uint32 values, 1M and 10M pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cub_sort cub_sort.cu && ./cub_sort
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <vector>
#include <random>

int main() {
    for (int n : {1000000, 10000000}) {
        std::vector<unsigned> hk(n), hv(n);
        std::mt19937 rng(1);
        for (int i = 0; i < n; ++i) { hk[i] = rng() & ((1u << 30) - 1); hv[i] = i; }
        unsigned *k0, *k1, *v0, *v1;
        cudaMalloc(&k0, 4ull * n); cudaMalloc(&k1, 4ull * n); cudaMalloc(&v0, 4ull * n); cudaMalloc(&v1, 4ull * n);
        cudaMemcpy(k0, hk.data(), 4ull * n, cudaMemcpyHostToDevice);
        cudaMemcpy(v0, hv.data(), 4ull * n, cudaMemcpyHostToDevice);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, 30);
        void* dtmp; cudaMalloc(&dtmp, tmp);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 5; ++w) cub::DeviceRadixSort::SortPairs(dtmp, tmp, k0, k1, v0, v1, n, 0, 30);
        const int reps = 30;
        float best = 1e9, sum = 0;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortPairs(dtmp, tmp, k0, k1, v0, v1, n, 0, 30);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); sum += ms; if (ms < best) best = ms;
        }
        printf("{\"n\": %d, \"bits\": 30, \"cub_sortpairs_ms_mean\": %.4f, \"best\": %.4f}\n", n, sum / reps, best);
        cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(dtmp);
    }
    return 0;
}
