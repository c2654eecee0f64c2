// TMEM feasibility probe (not product code): per-warp 32x32b stores and dependent 32x32b.x2 loads
// at warp-uniform dynamic columns; checks values and times the dependent load chain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t pat(int w, int t, int c) { return (uint32_t)((w << 20) | (t << 10) | c); }
__global__ void __launch_bounds__(512) k(int *err, long long *cyc, int iters, int cols_per_warp, int ncols)
{
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)), "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase;
    const int q = warp & 3, s = warp >> 2;
    const uint32_t ta = base + ((uint32_t)(32 * q) << 16) + (uint32_t)(s * cols_per_warp);
    if ((s + 1) * cols_per_warp <= ncols) {
        for (int c = 0; c < cols_per_warp; c += 4) {
            uint32_t r0 = pat(warp, lane, c), r1 = pat(warp, lane, c + 1), r2 = pat(warp, lane, c + 2), r3 = pat(warp, lane, c + 3);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta + c), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        int col = 0, bad = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            uint32_t v0, v1;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(ta + col) : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            bad |= (v0 != pat(warp, lane, col)) | (v1 != pat(warp, lane, col + 1));
            // next column depends on the loaded value (warp-uniform: lane 0's)
            const int c0 = __shfl_sync(0xffffffffu, (int)(v0 & 1023), 0);
            col = (c0 + 2 * 7) % (cols_per_warp - 1);
            col &= ~1;
        }
        long long t1 = clock64();
        if (bad) atomicAdd(err, 1);
        if (lane == 0 && blockIdx.x == 0 && warp == 0) *cyc = (t1 - t0);
        // the same chain through shared memory (one 8-byte word per lane and column pair)
        __shared__ uint2 sm[2][64 * 32];
        if (warp < 2) {
            for (int c = 0; c < 128; c += 2) sm[warp][(c / 2) * 32 + lane] = make_uint2(pat(warp, lane, c), pat(warp, lane, c + 1));
            __syncwarp();
            col = 0;
            long long t2 = clock64();
            for (int it = 0; it < iters; it++) {
                uint2 v; { const volatile uint2 *pp = &sm[warp][(col / 2) * 32 + lane]; v.x = pp->x; v.y = pp->y; }
                bad |= (v.x != pat(warp, lane, col));
                const int c0 = __shfl_sync(0xffffffffu, (int)(v.x & 1023), 0);
                col = (c0 + 2 * 7) % (128 - 1);
                col &= ~1;
            }
            long long t3 = clock64();
            if (lane == 0 && blockIdx.x == 0 && warp == 0) cyc[1] = (t3 - t2);
            if (bad) atomicAdd(err, 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols));
}
int main()
{
    int *err; long long *cyc;
    cudaMalloc(&err, 4); cudaMalloc(&cyc, 16); cudaMemset(err, 0, 4);
    for (int cfg = 0; cfg < 3; cfg++) {
        int threads = cfg == 0 ? 128 : 512, ncols = cfg == 2 ? 256 : 512, cpw = cfg == 0 ? 512 : (cfg == 1 ? 128 : 64);
        int ctas = 148 * (cfg == 2 ? 2 : 1);
        k<<<ctas, threads>>>(err, cyc, 1000, cpw, ncols);
        cudaError_t e = cudaDeviceSynchronize();
        int h; long long c[2]; cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost); cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
        printf("cfg %d threads %d ncols %d cpw %d: %s errors %d, %.1f cycles per dependent TMEM step, %.1f per LDS step\n", cfg, threads, ncols, cpw, cudaGetErrorString(e), h, c[0] / 1000.0, c[1] / 1000.0);
    }
    return 0;
}
