// Probe: semantics of TMA tile::gather4 / tile::scatter4 on sm_100a (2-D map, box {W, B1}).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tm, int W, int r0, int r1, int r2, int r3, double *out, int write)
{
    __shared__ __align__(128) double buf[4 * 64];
    __shared__ __align__(8) uint64_t mbar;
    uint32_t s = (uint32_t)__cvta_generic_to_shared(buf), mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) buf[i] = -1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(4 * W * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(s), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(mb) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb) : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) out[i] = buf[i];
    __syncthreads();
    if (write) {
        for (int i = threadIdx.x; i < 4 * W; i += blockDim.x) buf[i] = 1000.0 + i;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(&tm), "r"(0), "r"(r3), "r"(r2), "r"(r1), "r"(r0), "r"(s) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group 0;");
        }
    }
}
int main()
{
    const int W = 30, R = 100;
    std::vector<double> h(W * R);
    for (int r = 0; r < R; r++) for (int c = 0; c < W; c++) h[r * W + c] = r * 100 + c;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 4 * 64 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void *p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (CUresult(*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill))p;
    for (int b1 : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)R}, str[1] = {(cuuint64_t)W * 8};
        cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)b1}, es[2] = {1, 1};
        CUresult rr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box1=%d encode=%d\n", b1, (int)rr);
        if (rr) continue;
        k<<<1, 128>>>(tm, W, 7, 3, 50, 99, o, b1 == 1);
        cudaError_t e = cudaDeviceSynchronize();
        printf("  kernel: %s\n", cudaGetErrorString(e));
        if (e) return 1;
        std::vector<double> ho(4 * 64);
        cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 4; i++) printf("  smem row %d: %g %g ... %g | next %g\n", i, ho[i * W], ho[i * W + 1], ho[i * W + W - 1], ho[4 * W]);
        if (b1 == 1) {
            cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
            printf("  after scatter: row99[0]=%g row99[29]=%g row7[0]=%g row3[0]=%g row50[0]=%g row8[0]=%g\n", h[99 * W], h[99 * W + 29], h[7 * W], h[3 * W], h[50 * W], h[8 * W]);
        }
    }
    return 0;
}
