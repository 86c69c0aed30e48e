// K5 building block: C[M,N] (+)= A[M,K] * B[N,K]^T on the 5th-generation
// tensor cores (tcgen05.mma, accumulator in TMEM).
//
// Used by the selective recompute of deviating tokens (reference:
// pic.refresh -> toymodel._selective_forward, toymodel.py:99-151): the
// Q/K/V/mix projections h @ W are K-major GEMMs with B = W^T.
//
//   * float32 operands run as 3xTF32 (A_hi*B_hi + A_hi*B_lo + A_lo*B_hi, each
//     split with cvt.rna.tf32) so the products keep ~22 mantissa bits and
//     the result stays within float32 tolerance of the reference's numpy
//     float32 matmul; bf16 operands run as kind::f16 (bf16) directly.
//   * one CTA = one 128 x BN output tile, 128 threads: cp.async streams
//     128-byte K-slices of A and B (zero-filled past the edges) into a 3-4
//     stage shared-memory ring in the canonical no-swizzle K-major
//     core-matrix layout (8 rows x 16 B per core matrix); one elected thread
//     issues the MMAs of a stage and commits them to that stage's mbarrier,
//     which gates the stage's refill; the epilogue reads the accumulator with
//     tcgen05.ld and stores (or adds, for the residual update h += mix @ Wm)
//     float32 rows.
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "tdkv_common.cuh"
#include "tdkv_umma.cuh"

namespace tdkv {

constexpr int kGemmBM = 128;

__device__ __forceinline__ void cp_async_16_zfill(void* smem_dst, const void* gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)),
                 "l"(gsrc), "r"(src_bytes)
                 : "memory");
}

// T = float (3xTF32) or __nv_bfloat16.  A: (M, lda) row-major, B: (N, ldb)
// row-major (= K-major both), C: (M, ldc) float32.  BN <= 256, multiple of
// 16.  Each pipeline stage holds 128 bytes of K per row (32 tf32 / 64 bf16
// elements) for A and B, filled by cp.async (zero-filled past M, N, K);
// kStages - 1 stages are in flight while the tensor core consumes one.
template <typename T, int BN, int kStages>
__global__ void __launch_bounds__(128, 1)
    gemm_tn_kernel(const T* __restrict__ A, int lda, const T* __restrict__ B, int ldb,
                   float* __restrict__ C, int ldc, int M, int N, int K, int accumulate_c) {
    constexpr bool kTF32 = sizeof(T) == 4;
    constexpr int kEsz = sizeof(T);
    constexpr int kChunkElems = 16 / kEsz;                 // elements per 16-byte chunk
    constexpr int kCk = 8;                                 // 16-byte chunks per row per stage
    constexpr int kBK = kCk * kChunkElems;                 // K elements per stage
    constexpr int kPlanes = kTF32 ? 2 : 1;                 // hi/lo split for tf32
    constexpr int kABytes = kGemmBM * kCk * 16;            // one plane of an A stage
    constexpr int kBBytes = BN * kCk * 16;
    constexpr int kStageBytes = kPlanes * (kABytes + kBBytes);
    constexpr int kUmmaSteps = kCk / 2;                    // MMA-K = 32 bytes = 2 chunks
    constexpr uint32_t kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;

    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kStages];
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int m0 = blockIdx.x * kGemmBM;
    const int n0 = blockIdx.y * BN;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = umma_idesc(kTF32 ? 2 : 1, kGemmBM, BN);
    const int nk = (K + kBK - 1) / kBK;

    auto a_hi = [&](int st) { return smem + st * kStageBytes; };
    auto a_lo = [&](int st) { return smem + st * kStageBytes + kABytes; };
    auto b_hi = [&](int st) { return smem + st * kStageBytes + kPlanes * kABytes; };
    auto b_lo = [&](int st) { return smem + st * kStageBytes + kPlanes * kABytes + kBBytes; };

    // issue the cp.async loads of K-block kb into stage st
    auto load_stage = [&](int kb, int st) {
        const int k0 = kb * kBK;
        auto tile = [&](const T* src, int ld, int rows_valid, int row0, int nrows, uint8_t* dst) {
            for (int idx = tid; idx < nrows * kCk; idx += 128) {
                const int r = idx >> 3, c = idx & 7;
                const int gr = row0 + r, gk = k0 + c * kChunkElems;
                int bytes = 0;
                const T* g = src;
                if (gr < rows_valid && gk < K) {
                    bytes = min(kChunkElems, K - gk) * kEsz;
                    g = src + (size_t)gr * ld + gk;
                }
                cp_async_16_zfill(dst + core_off(r, c, kCk), g, bytes);
            }
        };
        tile(A, lda, M, m0, kGemmBM, a_hi(st));
        tile(B, ldb, N, n0, BN, b_hi(st));
    };
    // tf32: split this thread's own chunks of stage st into hi (in place) / lo
    auto split_stage = [&](int st) {
        auto split = [&](uint8_t* hi, uint8_t* lo, int nrows) {
            for (int idx = tid; idx < nrows * kCk; idx += 128) {
                const uint32_t off = core_off(idx >> 3, idx & 7, kCk);
                uint4 v = *reinterpret_cast<uint4*>(hi + off);
                float* f = reinterpret_cast<float*>(&v);
                uint4 h, l;
                uint32_t* hp = reinterpret_cast<uint32_t*>(&h);
                uint32_t* lp = reinterpret_cast<uint32_t*>(&l);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    hp[q] = tf32_rna(f[q]);
                    lp[q] = tf32_rna(f[q] - __uint_as_float(hp[q]));
                }
                *reinterpret_cast<uint4*>(hi + off) = h;
                *reinterpret_cast<uint4*>(lo + off) = l;
            }
        };
        split(a_hi(st), a_lo(st), kGemmBM);
        split(b_hi(st), b_lo(st), BN);
    };

    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int kb = 0; kb < nk; ++kb) {
        const int st = kb % kStages;
        cp_async_wait<kStages - 2>();          // this thread's chunks of K-block kb landed
        if constexpr (kTF32) split_stage(st);
        fence_proxy_async_smem();              // generic-proxy smem writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t lbo = 128, sbo = kCk * 128;
#pragma unroll
            for (int s = 0; s < kUmmaSteps; ++s) {
                const uint32_t koff = s * 2 * 128;             // two core matrices per MMA-K
                const uint64_t dah = umma_desc(smem_u32(a_hi(st)) + koff, lbo, sbo);
                const uint64_t dbh = umma_desc(smem_u32(b_hi(st)) + koff, lbo, sbo);
                umma<kTF32>(tmem, dah, dbh, idesc, (kb > 0 || s > 0) ? 1u : 0u);
                if constexpr (kTF32) {
                    const uint64_t dal = umma_desc(smem_u32(a_lo(st)) + koff, lbo, sbo);
                    const uint64_t dbl = umma_desc(smem_u32(b_lo(st)) + koff, lbo, sbo);
                    umma<kTF32>(tmem, dah, dbl, idesc, 1u);
                    umma<kTF32>(tmem, dal, dbh, idesc, 1u);
                }
            }
            umma_commit(&bars[st]);
        }
        // refill the stage consumed one iteration ago once its MMAs are done
        const int next = kb + kStages - 1;
        if (next < nk) {
            const int ns = next % kStages;
            if (kb >= 1) mbar_wait(&bars[ns], (uint32_t)(((kb - 1) / kStages) & 1));
            load_stage(next, ns);
        }
        cp_async_commit();
    }
    mbar_wait(&bars[(nk - 1) % kStages], (uint32_t)(((nk - 1) / kStages) & 1));
    tc_fence_after();

    // ---- epilogue: thread = one output row (TMEM lane), 8 columns per load
    const int row = m0 + tid;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 8) {
        uint32_t r[8];
        tmem_ld8(lane_addr + c0, r);
        if (row < M) {
            float* crow = C + (size_t)row * ldc;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int col = n0 + c0 + q;
                if (col < N) {
                    const float v = __uint_as_float(r[q]);
                    crow[col] = accumulate_c ? crow[col] + v : v;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

template <typename T, int BN>
static int32_t launch_gemm(const void* A, int lda, const void* B, int ldb, float* C, int ldc,
                           int M, int N, int K, int accumulate, cudaStream_t s) {
    constexpr int kStages = sizeof(T) == 4 ? 3 : 4;
    auto kern = gemm_tn_kernel<T, BN, kStages>;
    constexpr int kPlanes = sizeof(T) == 4 ? 2 : 1;
    const size_t smem = (size_t)kStages * kPlanes * (kGemmBM + BN) * 128;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_gemm: cudaFuncSetAttribute");
    dim3 grid((M + kGemmBM - 1) / kGemmBM, (N + BN - 1) / BN);
    kern<<<grid, 128, smem, s>>>(static_cast<const T*>(A), lda, static_cast<const T*>(B), ldb, C,
                                 ldc, M, N, K, accumulate);
    return TDKV_OK;
}

// ---------------------------------------------------------------------------
// TMA + warp-specialized variant.  Operand tiles arrive by TMA
// (cp.async.bulk.tensor, 128-byte swizzle, zero fill past the edges) into a
// kStages-deep ring; warp 0 produces, warp 1 issues the MMAs (one elected
// lane) and releases each stage with tcgen05.commit, warps 2-5 split tf32
// stages into hi/lo (3xTF32) and run the epilogue.  UMMA reads the stages
// through SWIZZLE_128B K-major descriptors (SBO = 1024 B, 8-row atoms).

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                       // version
    d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}


// PRE (float32 only): the operands arrive already split into tf32 hi / lo
// planes in global memory (tdkv_tf32_split; weights split once), so the TMA
// producer loads four tiles per stage and no warp splits in shared memory --
// the 3xTF32 GEMM becomes a pure TMA -> tcgen05 pipeline.
template <typename T, int BN, int kStages, bool PRE = false>
__global__ void __launch_bounds__(192, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_al,
                    const __grid_constant__ CUtensorMap map_bl, float* __restrict__ C, int ldc,
                    int M, int N, int K, int accumulate_c) {
    constexpr bool kTF32 = sizeof(T) == 4;
    static_assert(!PRE || kTF32, "pre-split operands are float32 (3xTF32)");
    constexpr int kBK = 128 / (int)sizeof(T);              // one 128-byte atom of K
    constexpr int kABytes = kGemmBM * 128;
    constexpr int kBBytes = BN * 128;
    constexpr int kPlanes = kTF32 ? 2 : 1;
    constexpr int kStageBytes = kPlanes * (kABytes + kBBytes);
    constexpr uint32_t kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // SWIZZLE_128B stages need 1024-byte alignment
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], split[kStages], accum;
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.x * kGemmBM;
    const int n0 = blockIdx.y * BN;
    const int nk = (K + kBK - 1) / kBK;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            mbar_init(&split[i], 128);
        }
        mbar_init(&accum, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    auto a_hi = [&](int st) { return smem + st * kStageBytes; };
    auto b_hi = [&](int st) { return smem + st * kStageBytes + kABytes; };
    auto a_lo = [&](int st) { return smem + st * kStageBytes + kABytes + kBBytes; };
    auto b_lo = [&](int st) { return smem + st * kStageBytes + 2 * kABytes + kBBytes; };

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer
            for (int kb = 0; kb < nk; ++kb) {
                const int st = kb % kStages;
                if (kb >= kStages) mbar_wait(&empty[st], (uint32_t)((kb / kStages - 1) & 1));
                mbar_arrive_expect_tx(&full[st], (PRE ? 2 : 1) * (kABytes + kBBytes));
                tma_load_2d(a_hi(st), &map_a, &full[st], kb * kBK, m0);
                tma_load_2d(b_hi(st), &map_b, &full[st], kb * kBK, n0);
                if constexpr (PRE) {
                    tma_load_2d(a_lo(st), &map_al, &full[st], kb * kBK, m0);
                    tma_load_2d(b_lo(st), &map_bl, &full[st], kb * kBK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                     // ---- MMA issuer
            const uint32_t idesc = umma_idesc(kTF32 ? 2 : 1, kGemmBM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int st = kb % kStages;
                mbar_wait((kTF32 && !PRE) ? &split[st] : &full[st], (uint32_t)((kb / kStages) & 1));
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < 4; ++s) {                // 4 x 32 bytes of K per atom
                    const uint64_t dah = umma_desc_sw128(smem_u32(a_hi(st)) + 32 * s);
                    const uint64_t dbh = umma_desc_sw128(smem_u32(b_hi(st)) + 32 * s);
                    umma<kTF32>(tmem, dah, dbh, idesc, (kb > 0 || s > 0) ? 1u : 0u);
                    if constexpr (kTF32) {
                        const uint64_t dal = umma_desc_sw128(smem_u32(a_lo(st)) + 32 * s);
                        const uint64_t dbl = umma_desc_sw128(smem_u32(b_lo(st)) + 32 * s);
                        umma<kTF32>(tmem, dah, dbl, idesc, 1u);
                        umma<kTF32>(tmem, dal, dbh, idesc, 1u);
                    }
                }
                umma_commit(&empty[st]);                     // frees the stage when done
            }
            umma_commit(&accum);
        }
    } else {
        const int et = tid - 64;                             // 0..127
        if constexpr (kTF32 && !PRE) {                       // ---- 3xTF32 split
            for (int kb = 0; kb < nk; ++kb) {
                const int st = kb % kStages;
                mbar_wait(&full[st], (uint32_t)((kb / kStages) & 1));
                auto run = [&](uint8_t* hi, uint8_t* lo, int bytes) {
                    for (int off = et * 16; off < bytes; off += 128 * 16) {
                        uint4 v = *reinterpret_cast<uint4*>(hi + off);
                        float* f = reinterpret_cast<float*>(&v);
                        uint4 h, l;
                        uint32_t* hp = reinterpret_cast<uint32_t*>(&h);
                        uint32_t* lp = reinterpret_cast<uint32_t*>(&l);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            hp[q] = tf32_rna(f[q]);
                            lp[q] = tf32_rna(f[q] - __uint_as_float(hp[q]));
                        }
                        *reinterpret_cast<uint4*>(hi + off) = h;
                        *reinterpret_cast<uint4*>(lo + off) = l;
                    }
                };
                run(a_hi(st), a_lo(st), kABytes);
                run(b_hi(st), b_lo(st), kBBytes);
                fence_proxy_async_smem();
                mbar_arrive(&split[st]);
            }
        }
        // ---- epilogue: TMEM lane quarter of this warp = warp % 4
        mbar_wait(&accum, 0u);
        tc_fence_after();
        const int q = warp & 3;
        const int row = m0 + q * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 8) {
            uint32_t r[8];
            tmem_ld8(lane_addr + c0, r);
            if (row < M) {
                float* crow = C + (size_t)row * ldc;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int col = n0 + c0 + j;
                    if (col < N) {
                        const float v = __uint_as_float(r[j]);
                        crow[col] = accumulate_c ? crow[col] + v : v;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// Persistent bf16 variant: one CTA per SM walks the output tiles
// (t = blockIdx.x, blockIdx.x + gridDim.x, ...; m-blocks fastest so the
// CTAs in flight share B tiles in L2).  Three pipelines: the smem ring
// (TMA producer <-> MMA issuer, continuous across tiles), and a
// double-buffered TMEM accumulator (2 x BN columns) between the MMA issuer
// and the four epilogue warps, so tile i's epilogue (tcgen05.ld -> float4
// stores) overlaps tile i+1's main loop.


template <int BN, int kStages>
__global__ void __launch_bounds__(192, 1)
    gemm_persistent_kernel(const __grid_constant__ CUtensorMap map_a,
                           const __grid_constant__ CUtensorMap map_b, float* __restrict__ C,
                           int ldc, int M, int N, int K, int accumulate_c) {
    constexpr int kBK = 64;                                 // one 128-byte bf16 atom of K
    constexpr int kABytes = kGemmBM * 128;
    constexpr int kBBytes = BN * 128;
    constexpr int kStageBytes = kABytes + kBBytes;
    constexpr uint32_t kTmemCols = 2 * BN;                  // two accumulators

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int nk = (K + kBK - 1) / kBK;
    const int tiles_m = (M + kGemmBM - 1) / kGemmBM;
    const int n_tiles = tiles_m * ((N + BN - 1) / BN);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);                       // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer
            int g = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                const int m0 = (t % tiles_m) * kGemmBM, n0 = (t / tiles_m) * BN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % kStages;
                    if (g >= kStages) mbar_wait(&empty[st], (uint32_t)((g / kStages - 1) & 1));
                    uint8_t* a = smem + st * kStageBytes;
                    mbar_arrive_expect_tx(&full[st], kStageBytes);
                    tma_load_2d(a, &map_a, &full[st], kb * kBK, m0);
                    tma_load_2d(a + kABytes, &map_b, &full[st], kb * kBK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                     // ---- MMA issuer
            const uint32_t idesc = umma_idesc(1, kGemmBM, BN);
            int g = 0, i = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const int acc = i & 1;
                if (i >= 2) mbar_wait(&tempty[acc], (uint32_t)((i / 2 - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % kStages;
                    mbar_wait(&full[st], (uint32_t)((g / kStages) & 1));
                    tc_fence_after();
                    const uint32_t a = smem_u32(smem + st * kStageBytes);
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        umma<false>(d, umma_desc_sw128(a + 32 * s),
                                    umma_desc_sw128(a + kABytes + 32 * s), idesc,
                                    (kb > 0 || s > 0) ? 1u : 0u);
                    umma_commit(&empty[st]);                 // frees the stage when done
                }
                umma_commit(&tfull[acc]);                    // accumulator ready
            }
        }
    } else {                                                 // ---- epilogue warps 2-5
        const int q = warp & 3;                              // TMEM lane quarter
        int i = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
            const int acc = i & 1;
            const int m0 = (t % tiles_m) * kGemmBM, n0 = (t / tiles_m) * BN;
            mbar_wait(&tfull[acc], (uint32_t)((i / 2) & 1));
            tc_fence_after();
            const int row = m0 + q * 32 + lane;
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
            float* crow = C + (size_t)row * ldc;
            const bool vec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + c0, r);
                if (row >= M) continue;
                const int col0 = n0 + c0;
                if (vec && col0 + 32 <= N) {
                    float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                               __uint_as_float(r[4 * j + 2]),
                                               __uint_as_float(r[4 * j + 3]));
                        if (accumulate_c) {
                            const float4 o = dst[j];
                            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                        }
                        dst[j] = v;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = col0 + j;
                        if (col < N) {
                            const float v = __uint_as_float(r[j]);
                            crow[col] = accumulate_c ? crow[col] + v : v;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);        // accumulator drained
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes
// a 256 x BN tile.  Each CTA stages its own 128 rows of A and its half of B
// (BN/2 rows) -- 2/3 of the single-CTA operand traffic per flop -- and the
// leader CTA's one elected thread issues M=256 MMAs that read both CTAs'
// shared memory and write each CTA's TMEM.  Both producers signal the
// leader's full barrier; the leader's commits multicast to both CTAs' empty
// and TMEM-full barriers; both CTAs' epilogue warps release the accumulator
// on the leader's TMEM-empty barrier.

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of ``p`` (a local smem address) in CTA ``rank``
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map,
                                                 uint32_t leader_bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}

template <int BN, int kStages>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b, float* __restrict__ C, int ldc,
                     int M, int N, int K, int accumulate_c) {
    constexpr int kBK = 64;
    constexpr int kABytes = kGemmBM * 128;                  // this CTA's 128 rows of A
    constexpr int kBBytes = (BN / 2) * 128;                 // this CTA's half of B
    constexpr int kStageBytes = kABytes + kBBytes;
    constexpr uint32_t kTmemCols = 2 * BN;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int nk = (K + kBK - 1) / kBK;
    const int tiles_m = (M + 2 * kGemmBM - 1) / (2 * kGemmBM);
    const int n_tiles = tiles_m * ((N + BN - 1) / BN);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);                         // the leader producer's arrive
            mbar_init(&empty[i], 1);                        // the leader's multicast commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);                       // 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();                                      // peer barriers initialized
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer (both CTAs)
            int g = 0;
            for (int t = pair; t < n_tiles; t += n_pairs) {
                const int m0 = (t % tiles_m) * 2 * kGemmBM + (int)rank * kGemmBM;
                const int n0 = (t / tiles_m) * BN + (int)rank * (BN / 2);
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % kStages;
                    if (g >= kStages) mbar_wait(&empty[st], (uint32_t)((g / kStages - 1) & 1));
                    if (leader) mbar_arrive_expect_tx(&full[st], 2 * kStageBytes);
                    const uint32_t bar = map_to_rank(&full[st], 0);
                    uint8_t* a = smem + st * kStageBytes;
                    tma_load_2d_pair(a, &map_a, bar, kb * kBK, m0);
                    tma_load_2d_pair(a + kABytes, &map_b, bar, kb * kBK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {                           // ---- MMA issuer (leader)
            const uint32_t idesc = umma_idesc(1, 2 * kGemmBM, BN);
            int g = 0, i = 0;
            for (int t = pair; t < n_tiles; t += n_pairs, ++i) {
                const int acc = i & 1;
                if (i >= 2) mbar_wait(&tempty[acc], (uint32_t)((i / 2 - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int st = g % kStages;
                    mbar_wait(&full[st], (uint32_t)((g / kStages) & 1));
                    tc_fence_after();
                    const uint32_t a = smem_u32(smem + st * kStageBytes);
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        umma_pair(d, umma_desc_sw128(a + 32 * s),
                                  umma_desc_sw128(a + kABytes + 32 * s), idesc,
                                  (kb > 0 || s > 0) ? 1u : 0u);
                    umma_commit_pair(&empty[st]);            // frees the stage in both CTAs
                }
                umma_commit_pair(&tfull[acc]);               // both CTAs' accumulators ready
            }
        }
    } else {                                                 // ---- epilogue warps 2-5
        const int q = warp & 3;
        const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
        const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
        int i = 0;
        for (int t = pair; t < n_tiles; t += n_pairs, ++i) {
            const int acc = i & 1;
            const int m0 = (t % tiles_m) * 2 * kGemmBM + (int)rank * kGemmBM;
            const int n0 = (t / tiles_m) * BN;
            mbar_wait(&tfull[acc], (uint32_t)((i / 2) & 1));
            tc_fence_after();
            const int row = m0 + q * 32 + lane;
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
            float* crow = C + (size_t)row * ldc;
            const bool vec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + c0, r);
                if (row >= M) continue;
                const int col0 = n0 + c0;
                if (vec && col0 + 32 <= N) {
                    float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                               __uint_as_float(r[4 * j + 2]),
                                               __uint_as_float(r[4 * j + 3]));
                        if (accumulate_c) {
                            const float4 o = dst[j];
                            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                        }
                        dst[j] = v;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = col0 + j;
                        if (col < N) {
                            const float v = __uint_as_float(r[j]);
                            crow[col] = accumulate_c ? crow[col] + v : v;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
        }
    }
    tc_fence_before();
    cluster_sync_all();                                      // both CTAs done with TMEM
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D K-major tensor map: dims (K, rows), box (128 bytes of K, box_rows), 128 B swizzle
static bool make_map(CUtensorMap* map, const void* base, int dtype, int rows, int K, int ld,
                     int box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const size_t esz = elt_size(dtype);
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
    const cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, dtype == TDKV_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename T, int BN, int kStages, bool PRE = false>
static int32_t launch_gemm_tma(const void* A, int lda, const void* B, int ldb, float* C, int ldc,
                               int M, int N, int K, int accumulate, int dtype, cudaStream_t s,
                               bool* ok, const void* A_lo = nullptr, const void* B_lo = nullptr) {
    CUtensorMap ma, mb, mal, mbl;
    *ok = make_map(&ma, A, dtype, M, K, lda, kGemmBM) && make_map(&mb, B, dtype, N, K, ldb, BN);
    if (PRE)
        *ok = *ok && make_map(&mal, A_lo, dtype, M, K, lda, kGemmBM) &&
              make_map(&mbl, B_lo, dtype, N, K, ldb, BN);
    else
        mal = ma, mbl = mb;
    if (!*ok) return TDKV_OK;
    auto kern = gemm_tma_kernel<T, BN, kStages, PRE>;
    constexpr int kPlanes = sizeof(T) == 4 ? 2 : 1;
    const size_t smem = (size_t)kStages * kPlanes * (kGemmBM + BN) * 128 + 1024;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_gemm: cudaFuncSetAttribute");
    dim3 grid((M + kGemmBM - 1) / kGemmBM, (N + BN - 1) / BN);
    kern<<<grid, 192, smem, s>>>(ma, mb, mal, mbl, C, ldc, M, N, K, accumulate);
    return TDKV_OK;
}

template <int BN, int kStages>
static int32_t launch_gemm_persistent(const void* A, int lda, const void* B, int ldb, float* C,
                                      int ldc, int M, int N, int K, int accumulate,
                                      cudaStream_t s, bool* ok) {
    CUtensorMap ma, mb;
    *ok = make_map(&ma, A, TDKV_BF16, M, K, lda, kGemmBM) &&
          make_map(&mb, B, TDKV_BF16, N, K, ldb, BN);
    if (!*ok) return TDKV_OK;
    auto kern = gemm_persistent_kernel<BN, kStages>;
    const size_t smem = (size_t)kStages * (kGemmBM + BN) * 128 + 1024;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_gemm: cudaFuncSetAttribute");
    const long long tiles = (long long)((M + kGemmBM - 1) / kGemmBM) * ((N + BN - 1) / BN);
    const int grid = (int)(tiles < sm_count() ? tiles : sm_count());
    kern<<<grid, 192, smem, s>>>(ma, mb, C, ldc, M, N, K, accumulate);
    return TDKV_OK;
}

template <int BN, int kStages>
static int32_t launch_gemm_pair(const void* A, int lda, const void* B, int ldb, float* C, int ldc,
                                int M, int N, int K, int accumulate, cudaStream_t s, bool* ok) {
    CUtensorMap ma, mb;
    *ok = make_map(&ma, A, TDKV_BF16, M, K, lda, kGemmBM) &&
          make_map(&mb, B, TDKV_BF16, N, K, ldb, BN / 2);
    if (!*ok) return TDKV_OK;
    auto kern = gemm_pair_kernel<BN, kStages>;
    const size_t smem = (size_t)kStages * (kGemmBM + BN / 2) * 128 + 1024;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return check_launch("tdkv_gemm: cudaFuncSetAttribute");
    const long long tiles = (long long)((M + 255) / 256) * ((N + BN - 1) / BN);
    const int pairs = (int)(tiles < sm_count() / 2 ? tiles : sm_count() / 2);
    kern<<<2 * pairs, 192, smem, s>>>(ma, mb, C, ldc, M, N, K, accumulate);
    return TDKV_OK;
}

}  // namespace tdkv

using namespace tdkv;

extern "C" int32_t tdkv_gemm(const void* d_a, int32_t lda, const void* d_b, int32_t ldb,
                             float* d_c, int32_t ldc, int32_t m, int32_t n, int32_t k,
                             int32_t dtype, int32_t accumulate, void* stream) {
    if (m < 0 || n < 0 || k < 0) return set_error(TDKV_EINVAL, "tdkv_gemm: negative size");
    if (m == 0 || n == 0) return TDKV_OK;
    if (!d_a || !d_b || !d_c) return set_error(TDKV_EINVAL, "tdkv_gemm: null pointer");
    const size_t esz = elt_size(dtype);
    if (dtype != TDKV_F32 && dtype != TDKV_BF16)
        return set_error(TDKV_EUNSUPPORTED, "tdkv_gemm: dtype %d", dtype);
    if (!aligned(d_a, 16) || !aligned(d_b, 16) || (lda * esz) % 16 || (ldb * esz) % 16)
        return set_error(TDKV_EINVAL, "tdkv_gemm: A/B rows must be 16-byte aligned");
    if (k == 0) return set_error(TDKV_EINVAL, "tdkv_gemm: K must be positive");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t rc;
    bool tma = false;
    if (!getenv("TDKV_GEMM_NO_TMA")) {
        if (dtype == TDKV_F32) {
            rc = n <= 64 ? launch_gemm_tma<float, 64, 4>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                          accumulate, dtype, s, &tma)
                         : launch_gemm_tma<float, 128, 3>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                           accumulate, dtype, s, &tma);
        } else if (n >= 256 && m > 128 && !getenv("TDKV_GEMM_NO_PAIR") &&
                   (long long)((m + 255) / 256) * ((n + 255) / 256) >= sm_count() / 2) {
            // enough 256 x 256 tiles to give every CTA pair work: cta_group::2
            // (256 x 128 pair tiles measured 0.67x: more operand traffic per flop)
            rc = launch_gemm_pair<256, 7>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s,
                                          &tma);
        } else if (n > 64 && !getenv("TDKV_GEMM_NO_PERSISTENT")) {
            const long long tiles256 = (long long)((m + 127) / 128) * ((n + 255) / 256);
            rc = (n >= 256 && tiles256 >= sm_count())
                     ? launch_gemm_persistent<256, 4>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                      accumulate, s, &tma)
                     : launch_gemm_persistent<128, 6>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                      accumulate, s, &tma);
        } else {
            const long long tiles256 = (long long)((m + 127) / 128) * ((n + 255) / 256);
            if (n <= 64)
                rc = launch_gemm_tma<__nv_bfloat16, 64, 6>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                            accumulate, dtype, s, &tma);
            else if (n >= 256 && tiles256 >= sm_count())
                rc = launch_gemm_tma<__nv_bfloat16, 256, 4>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                             accumulate, dtype, s, &tma);
            else
                rc = launch_gemm_tma<__nv_bfloat16, 128, 5>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k,
                                                             accumulate, dtype, s, &tma);
        }
        if (rc) return rc;
        if (tma) {
            count_launch();
            return check_launch("tdkv_gemm");
        }
    }
    if (dtype == TDKV_F32) {
        rc = n <= 64 ? launch_gemm<float, 64>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s)
                     : launch_gemm<float, 128>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s);
    } else {
        // 128 x 256 tiles halve the L2 operand traffic per flop when the
        // grid still fills the SMs
        const long long tiles256 = (long long)((m + 127) / 128) * ((n + 255) / 256);
        if (n <= 64)
            rc = launch_gemm<__nv_bfloat16, 64>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s);
        else if (n >= 256 && tiles256 >= sm_count())
            rc = launch_gemm<__nv_bfloat16, 256>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s);
        else
            rc = launch_gemm<__nv_bfloat16, 128>(d_a, lda, d_b, ldb, d_c, ldc, m, n, k, accumulate, s);
    }
    if (rc) return rc;
    count_launch();
    return check_launch("tdkv_gemm");
}

// ---------------------------------------------------------------------------
// 3xTF32 with pre-split operands

__global__ void tf32_split_kernel(const float4* __restrict__ src, long long n4,
                                  uint4* __restrict__ hi, uint4* __restrict__ lo) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 v = src[i];
        uint4 h, l;
        h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - __uint_as_float(h.x));
        h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - __uint_as_float(h.y));
        h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - __uint_as_float(h.z));
        h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - __uint_as_float(h.w));
        hi[i] = h;
        lo[i] = l;
    }
}

extern "C" int32_t tdkv_tf32_split(const float* d_src, int64_t n, float* d_hi, float* d_lo,
                                   void* stream) {
    if (n < 0) return set_error(TDKV_EINVAL, "tdkv_tf32_split: negative size");
    if (n == 0) return TDKV_OK;
    if (!d_src || !d_hi || !d_lo) return set_error(TDKV_EINVAL, "tdkv_tf32_split: null pointer");
    if (n % 4 || !aligned(d_src, 16) || !aligned(d_hi, 16) || !aligned(d_lo, 16))
        return set_error(TDKV_EINVAL, "tdkv_tf32_split: 16-byte aligned multiples of 4 floats");
    const long long n4 = n / 4;
    long long grid = (n4 + 255) / 256;
    if (grid > sm_count() * 8) grid = sm_count() * 8;
    tf32_split_kernel<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const float4*>(d_src), n4, reinterpret_cast<uint4*>(d_hi),
        reinterpret_cast<uint4*>(d_lo));
    count_launch();
    return check_launch("tdkv_tf32_split");
}

extern "C" int32_t tdkv_gemm_tf32x3(const float* d_a_hi, const float* d_a_lo, int32_t lda,
                                    const float* d_b_hi, const float* d_b_lo, int32_t ldb,
                                    float* d_c, int32_t ldc, int32_t m, int32_t n, int32_t k,
                                    int32_t accumulate, void* stream) {
    if (m < 0 || n < 0 || k < 0) return set_error(TDKV_EINVAL, "tdkv_gemm_tf32x3: negative size");
    if (m == 0 || n == 0) return TDKV_OK;
    if (k == 0) return set_error(TDKV_EINVAL, "tdkv_gemm_tf32x3: K must be positive");
    if (!d_a_hi || !d_a_lo || !d_b_hi || !d_b_lo || !d_c)
        return set_error(TDKV_EINVAL, "tdkv_gemm_tf32x3: null pointer");
    if (!aligned(d_a_hi, 16) || !aligned(d_a_lo, 16) || !aligned(d_b_hi, 16) ||
        !aligned(d_b_lo, 16) || (lda * 4) % 16 || (ldb * 4) % 16)
        return set_error(TDKV_EINVAL, "tdkv_gemm_tf32x3: A/B rows must be 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    bool tma = false;
    const int32_t rc =
        n <= 64 ? launch_gemm_tma<float, 64, 4, true>(d_a_hi, lda, d_b_hi, ldb, d_c, ldc, m, n, k,
                                                      accumulate, TDKV_F32, s, &tma, d_a_lo,
                                                      d_b_lo)
                : launch_gemm_tma<float, 128, 3, true>(d_a_hi, lda, d_b_hi, ldb, d_c, ldc, m, n,
                                                       k, accumulate, TDKV_F32, s, &tma, d_a_lo,
                                                       d_b_lo);
    if (rc) return rc;
    if (!tma) return set_error(TDKV_EUNSUPPORTED, "tdkv_gemm_tf32x3: tensor maps unavailable");
    count_launch();
    return check_launch("tdkv_gemm_tf32x3");
}
