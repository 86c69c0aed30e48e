// Direction-resolved HBM ceilings with hand-written 16-byte streaming kernels
// (context for the rooflines; the reported denominator stays
// MEASURED_PEAKS.json's copy figure).  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/hbm_probe scripts/hbm_probe.cu
//   gpurun_out/hbm_probe            -> one JSON line
//
// read:   every byte of an 8 GiB buffer loaded once (ld.global.cs, xor-reduced)
// write:  8 GiB stored once (st.global.cs)
// copy:   4 GiB -> 4 GiB
// fanout: the collector's pattern -- a 224 MiB source read once, each 16-byte
//         unit stored to 50 destinations (11.2 GiB written)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void read_k(const uint4* __restrict__ p, size_t n, uint4* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x & acc.y & acc.z & acc.w) == 0xFFFFFFFFu) sink[threadIdx.x] = acc;
}

__global__ void write_k(uint4* __restrict__ p, size_t n) {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        __stcs(p + i, v);
}

__global__ void write_wb_k(uint4* __restrict__ p, size_t n) {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// TMA bulk store: each CTA fills a 16 KiB smem tile once and streams it out
// with cp.async.bulk.global.shared::cta in `chunk`-byte pieces
__global__ void write_bulk_k(char* __restrict__ p, size_t nbytes, int chunk) {
    __shared__ __align__(128) uint4 tile[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tile[i] = make_uint4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const size_t pieces = nbytes / chunk;
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(tile);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < pieces;
         i += (size_t)gridDim.x * blockDim.x) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(p + i * chunk), "r"(saddr + (unsigned)((i * chunk) % 16384)), "r"(chunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        __stcs(d + i, __ldcs(s + i));
}

__global__ void fanout_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n, int fan) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(s + i);
        for (int f = 0; f < fan; ++f) __stcs(d + (size_t)f * n + i, v);
    }
}

// 256-bit accesses (sm_100: LDG/STG .256)
struct alignas(32) u8x32 { uint32_t w[8]; };

__device__ __forceinline__ u8x32 ld256(const u8x32* p) {
    u8x32 r;
    asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]),
                   "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st256(u8x32* p, const u8x32& v) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]),
                    "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

__global__ void write256_k(u8x32* __restrict__ p, size_t n) {
    u8x32 v;
    for (int q = 0; q < 8; ++q) v.w[q] = threadIdx.x + q;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        st256(p + i, v);
}

__global__ void copy256_k(const u8x32* __restrict__ s, u8x32* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        st256(d + i, ld256(s + i));
}

__global__ void fanout256_k(const u8x32* __restrict__ s, u8x32* __restrict__ d, size_t n,
                            int fan) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const u8x32 v = ld256(s + i);
        for (int f = 0; f < fan; ++f) st256(d + (size_t)f * n + i, v);
    }
}

// TMA both ways: one thread per CTA streams chunks global -> smem (bulk load,
// mbarrier) -> global (bulk store) through an S-stage ring
__device__ __forceinline__ unsigned sm32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

template <int S>
__global__ void copy_tma_k(const char* __restrict__ src, char* __restrict__ dst, size_t nbytes,
                           int chunk) {
    extern __shared__ __align__(128) char buf[];
    __shared__ __align__(8) uint64_t bar[S];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t n = nbytes / chunk;
    auto load = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(sm32(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                     "[%0], [%1], %2, [%3];"
                     ::"r"(sm32(buf + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk),
                       "r"(sm32(&bar[s])) : "memory");
    };
    for (int s = 0; s < S; ++s) {
        const size_t c = blockIdx.x + (size_t)s * gridDim.x;
        if (c < n) load(c, s);
    }
    for (size_t k = 0;; ++k) {
        const size_t c = blockIdx.x + k * gridDim.x;
        if (c >= n) break;
        const int s = (int)(k % S);
        const unsigned phase = (unsigned)((k / S) & 1);
        asm volatile("{\n.reg .pred p;\nW%=:\n"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                     "@!p bra W%=;\n}\n" ::"r"(sm32(&bar[s])), "r"(phase) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst + c * chunk), "r"(sm32(buf + (size_t)s * chunk)), "r"(chunk)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (k >= 1) {
            // the previous stage's store has read its smem: refill it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            const size_t c2 = blockIdx.x + (k - 1 + S) * gridDim.x;
            if (c2 < n) load(c2, (int)((k - 1) % S));
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// more memory-level parallelism per thread: 4 independent 16-byte loads, then
// their 4 stores
__global__ void copy4_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (i + q * stride < n) v[q] = __ldcs(s + i + q * stride);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (i + q * stride < n) __stcs(d + i + q * stride, v[q]);
    }
}

template <typename F>
static float best_ms(F launch, int reps = 10) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = 8ull << 30;
    uint4 *x, *y, *sink;
    CK(cudaMalloc(&x, big));
    CK(cudaMalloc(&y, big));
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMemset(x, 1, big));
    const size_t n = big / 16;
    const dim3 grid(sms * 8), block(256);
    const float r = best_ms([&] { read_k<<<grid, block>>>(x, n, sink); });
    const float w = best_ms([&] { write_k<<<grid, block>>>(y, n); });
    const float c = best_ms([&] { copy_k<<<grid, block>>>(x, y, n / 2); });
    const float wb = best_ms([&] { write_wb_k<<<grid, block>>>(y, n); });
    const float b1 = best_ms([&] { write_bulk_k<<<sms * 2, 32>>>((char*)y, big, 1024); });
    const float b4 = best_ms([&] { write_bulk_k<<<sms * 2, 32>>>((char*)y, big, 4096); });
    const size_t src = 224ull << 20;
    const int fan = 50;
    const float f = best_ms([&] { fanout_k<<<grid, block>>>(x, y, src / 16, fan); }, 5);
    const float w32 = best_ms([&] { write256_k<<<grid, block>>>((u8x32*)y, big / 32); });
    const float c32 = best_ms([&] { copy256_k<<<grid, block>>>((const u8x32*)x, (u8x32*)y,
                                                               big / 64); });
    const float f32 = best_ms([&] { fanout256_k<<<grid, block>>>((const u8x32*)x, (u8x32*)y,
                                                                 src / 32, fan); }, 5);
    float cm = best_ms([&] { cudaMemcpyAsync(y, x, big / 2, cudaMemcpyDeviceToDevice); });
    float tma[4];
    const int chunks[4] = {8192, 16384, 32768, 49152};
    for (int q = 0; q < 4; ++q) {
        const int ch = chunks[q];
        const int S = 4;
        const size_t smem = (size_t)S * ch;
        CK(cudaFuncSetAttribute(copy_tma_k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_tma_k<4>, 32, smem));
        tma[q] = best_ms([&] { copy_tma_k<4><<<sms * per_sm, 32, smem>>>((const char*)x,
                                                                          (char*)y, big / 2, ch); });
    }
    const float c4 = best_ms([&] { copy4_k<<<grid, block>>>(x, y, n / 2); });
    CK(cudaGetLastError());
    printf("{\"copy_tma_8k_gbs\": %.1f, \"copy_tma_16k_gbs\": %.1f, \"copy_tma_32k_gbs\": %.1f, "
           "\"copy_tma_48k_gbs\": %.1f, \"copy_4x16b_gbs\": %.1f}\n",
           big / (tma[0] * 1e-3) / 1e9, big / (tma[1] * 1e-3) / 1e9, big / (tma[2] * 1e-3) / 1e9,
           big / (tma[3] * 1e-3) / 1e9, big / (c4 * 1e-3) / 1e9);
    CK(cudaGetLastError());
    printf("{\"write256_gbs\": %.1f, \"copy256_gbs\": %.1f, \"fanout50_256_gbs\": %.1f, "
           "\"memcpy_d2d_gbs\": %.1f}\n",
           big / (w32 * 1e-3) / 1e9, big / (c32 * 1e-3) / 1e9,
           (src * (fan + 1)) / (f32 * 1e-3) / 1e9, big / (cm * 1e-3) / 1e9);
    printf("{\"read_gbs\": %.1f, \"write_gbs\": %.1f, \"copy_gbs\": %.1f, "
           "\"write_default_gbs\": %.1f, \"write_bulk1k_gbs\": %.1f, \"write_bulk4k_gbs\": %.1f, "
           "\"fanout50_gbs\": %.1f, \"fanout50_bytes\": %zu, \"bytes\": %zu, \"sms\": %d}\n",
           big / (r * 1e-3) / 1e9, big / (w * 1e-3) / 1e9, big / (c * 1e-3) / 1e9,
           big / (wb * 1e-3) / 1e9, big / (b1 * 1e-3) / 1e9, big / (b4 * 1e-3) / 1e9,
           (src * (fan + 1)) / (f * 1e-3) / 1e9, src * (fan + 1), big, sms);
    return 0;
}
