// Copy-engine (CE) probe: can the DMA copy engines add HBM throughput next to
// SM kernels?  (Context for K1/K3 design; not part of the product.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ce_probe scripts/ce_probe.cu
//
// ce_memcpy:     one 2 GiB D2D cudaMemcpyAsync
// ce_batch_<n>k: 2 GiB as a cudaMemcpyBatchAsync of n-KiB copies
// ce_fanout:     a 224 MiB source in 256 KiB pieces, each copied to 25 places
// sm_fanout:     the same fan-out by an SM kernel (16-byte loads/stores)
// mixed:         SM fan-out of one half of the destinations + CE fan-out of the
//                other half, concurrently on two streams
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void fanout_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n, int fan,
                         size_t dstride) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(s + i);
        for (int f = 0; f < fan; ++f) __stcs(d + (size_t)f * dstride + i, v);
    }
}

struct Batch {
    std::vector<void*> dst, src;
    std::vector<size_t> size;
};

static cudaError_t run_batch(Batch& b, cudaStream_t s) {
    cudaMemcpyAttributes attr = {};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    size_t idx = 0, fail = 0;
    return cudaMemcpyBatchAsync(b.dst.data(), b.src.data(), b.size.data(), b.dst.size(), &attr,
                                &idx, 1, &fail, s);
}

static cudaStream_t g_s1;   // batched copies may not use the legacy NULL stream

template <typename F>
static float time_ms(F launch, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a, g_s1);
        launch();
        cudaEventRecord(b, g_s1);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = 2ull << 30;
    char *x, *y;
    CK(cudaMalloc(&x, big));
    CK(cudaMalloc(&y, 14ull << 30));
    CK(cudaMemset(x, 1, big));
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g_s1, cudaStreamNonBlocking));
    cudaStream_t s1 = g_s1;
    cudaEvent_t fork, join;
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));

    const float t_mc = time_ms([&] { cudaMemcpyAsync(y, x, big, cudaMemcpyDeviceToDevice, s1); });
    printf("{\"ce_memcpy_gbs\": %.1f", 2.0 * big / (t_mc * 1e-3) / 1e9);
    for (size_t kib : {32, 256, 1024}) {
        Batch b;
        const size_t piece = kib << 10;
        for (size_t o = 0; o < big; o += piece) {
            b.dst.push_back(y + o);
            b.src.push_back(x + o);
            b.size.push_back(piece);
        }
        CK(run_batch(b, s1));
        CK(cudaDeviceSynchronize());
        const float t = time_ms([&] { run_batch(b, s1); });
        printf(", \"ce_batch_%zuk_gbs\": %.1f", kib, 2.0 * big / (t * 1e-3) / 1e9);
    }
    // fan-out: 224 MiB source, 25 destinations (5.6 GiB written)
    const size_t src = 224ull << 20;
    const int fan = 25;
    Batch fb;
    const size_t piece = 256 << 10;
    for (int f = 0; f < fan; ++f)
        for (size_t o = 0; o < src; o += piece) {
            fb.dst.push_back(y + (size_t)f * src + o);
            fb.src.push_back(x + o);
            fb.size.push_back(piece);
        }
    const double fbytes = (double)src * (fan + 1);
    const float t_cef = time_ms([&] { run_batch(fb, s1); });
    const dim3 grid(sms * 8), block(256);
    const float t_smf = time_ms([&] {
        fanout_k<<<grid, block, 0, s1>>>((const uint4*)x, (uint4*)y, src / 16, fan, src / 16);
    });
    // mixed: SM fans out to destinations [0, 25), CE to [25, 50) concurrently
    Batch mb;
    for (int f = fan; f < 2 * fan; ++f)
        for (size_t o = 0; o < src; o += piece) {
            mb.dst.push_back(y + (size_t)f * src + o);
            mb.src.push_back(x + o);
            mb.size.push_back(piece);
        }
    const float t_mix = time_ms([&] {
        cudaEventRecord(fork, s1);
        cudaStreamWaitEvent(s2, fork, 0);
        run_batch(mb, s2);
        fanout_k<<<grid, block, 0, s1>>>((const uint4*)x, (uint4*)y, src / 16, fan, src / 16);
        cudaEventRecord(join, s2);
        cudaStreamWaitEvent(s1, join, 0);
    });
    CK(cudaGetLastError());
    printf(", \"ce_fanout25_gbs\": %.1f, \"sm_fanout25_gbs\": %.1f, \"mixed_fanout50_gbs\": %.1f",
           fbytes / (t_cef * 1e-3) / 1e9, fbytes / (t_smf * 1e-3) / 1e9,
           (double)src * (2 * fan + 1) / (t_mix * 1e-3) / 1e9);
    printf(", \"ms\": {\"ce_fanout\": %.3f, \"sm_fanout\": %.3f, \"mixed\": %.3f}}\n", t_cef,
           t_smf, t_mix);
    return 0;
}
