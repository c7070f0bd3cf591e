// Shared-memory ranking probe: what one bucket-rank per string costs on an SM
// (the per-tile step of the wide scatter).  One CTA per SM, 1024 threads, K
// counters, pseudo-random bucket ids; cycles per string per SM for
//   red     atomicAdd without a result (the count kernel's histogram)
//   atom    atomicAdd with its result (the scatter's rank)
//   ldst    plain load + store on the same counters (upper bound of a
//           non-atomic warp-private scheme)
//   match   __match_any_sync + leader's returning atomicAdd + shuffle
//   lds     one random u32 shared load per string (bank-conflict baseline)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rank_probe rank_probe.cu && ./rank_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024) k_rank(uint32_t K, uint32_t rounds, uint32_t* out, long long* cyc) {
    extern __shared__ uint32_t cnt[];
    for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    uint32_t acc = 0;
    const uint32_t lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (uint32_t r = 0; r < rounds; ++r) {
        const uint32_t b = hash32(threadIdx.x + r * 1024u + blockIdx.x * 77777u) % K;
        if (MODE == 0) {
            atomicAdd(&cnt[b], 1u);
        } else if (MODE == 1) {
            acc += atomicAdd(&cnt[b], 1u);
        } else if (MODE == 2) {
            const uint32_t x = cnt[b];
            cnt[b] = x + 1;
            acc += x;
        } else if (MODE == 3) {
            const uint32_t m = __match_any_sync(0xffffffffu, b);
            const uint32_t leader = __ffs(m) - 1;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(&cnt[b], static_cast<uint32_t>(__popc(m)));
            base = __shfl_sync(0xffffffffu, base, leader);
            acc += base + __popc(m & ((1u << lane) - 1));
        } else {
            acc += cnt[b];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0xdeadbeef) out[0] = acc;
}

template <int MODE>
void run(const char* name, uint32_t K, uint32_t threads) {
    const uint32_t rounds = 4096;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 148 * 8);
    k_rank<MODE><<<148, threads, K * 4>>>(K, rounds, out, cyc);
    k_rank<MODE><<<148, threads, K * 4>>>(K, rounds, out, cyc);
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-6s K=%5u threads=%4u  %.3f cycles / string / SM\n", name, K, threads,
           avg / (double(rounds) * threads));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (uint32_t K : {128u, 2048u}) {
        for (uint32_t th : {512u, 1024u}) {
            run<0>("red", K, th);
            run<1>("atom", K, th);
            run<2>("ldst", K, th);
            run<3>("match", K, th);
            run<4>("lds", K, th);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
