// DRAM write amplification probe: int64 stores of different completeness
// per warp instruction, read back through ncu's dram__bytes_write.sum.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe write_probe.cu
//   ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum ./write_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// every element written once, full warps (coalesced)
__global__ void k_full(int64_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = i;
}
// two passes inside one kernel: lanes with hash bit set first, the rest after a
// block barrier (every element written once, sectors completed by the 2nd pass)
__global__ void k_two_pass(int64_t* a, uint64_t n) {
    const uint64_t per = 4096;
    for (uint64_t base = blockIdx.x * per; base < n; base += (uint64_t)gridDim.x * per) {
        for (uint64_t i = base + threadIdx.x; i < base + per && i < n; i += blockDim.x)
            if (hash32(i) & 1) a[i] = i;
        __syncthreads();
        for (uint64_t i = base + threadIdx.x; i < base + per && i < n; i += blockDim.x)
            if (!(hash32(i) & 1)) a[i] = i;
        __syncthreads();
    }
}
// segments of ~400 elements at unaligned starts, one per CTA (64 threads):
// elements written in sorted-position order, 70% in pass 1, the rest in pass 2
__global__ void k_segments(int64_t* a, uint64_t n, uint32_t seg) {
    const uint64_t begin = (uint64_t)blockIdx.x * seg;
    const uint64_t end = begin + seg < n ? begin + seg : n;
    for (uint64_t i = begin + threadIdx.x; i < end; i += blockDim.x)
        if (hash32(i) % 10 < 7) a[i] = i;
    __syncthreads();
    for (uint64_t i = begin + threadIdx.x; i < end; i += blockDim.x)
        if (hash32(i) % 10 >= 7) a[i] = i;
}
// single pass, 70% of lanes only (the other 30% never written)
__global__ void k_partial(int64_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (hash32(i) % 10 < 7) a[i] = i;
}

int main() {
    const uint64_t n = 1ull << 25;  // 268 MB of int64
    int64_t* a;
    cudaMalloc(&a, n * 8);
    cudaMemset(a, 0, n * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k_full<<<148 * 8, 256>>>(a, n);
        k_two_pass<<<148 * 8, 256>>>(a, n);
        k_segments<<<(unsigned)((n + 399) / 400), 64>>>(a, n, 400);
        k_segments<<<(unsigned)((n + 1999) / 2000), 256>>>(a, n, 2000);
        k_partial<<<148 * 8, 256>>>(a, n);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("done %s (expect %.1f MB per full write)\n", cudaGetErrorString(e), n * 8 / 1e6);
    return 0;
}
