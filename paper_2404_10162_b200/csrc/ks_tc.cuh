// ks_tc.cuh -- tcgen05 / TMEM / TMA / mbarrier primitives shared by the
// tensor-core kernels (the decode gate GEMM, ks_gemm_tc.cu, and the training
// GEMM, ks_gemm16.cu).  Inline PTX for sm_100a.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ks_common.cuh"

namespace ksb {

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}
// CTA-pair form: the completion goes to the LEADER CTA's barrier (the pair's
// shared::cluster addresses differ in bit 24; clearing it names rank 0's copy).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(bar), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// K-major, swizzled operand tile: rows of kTcBK fp16, 8-row atoms (SBO), LBO
// unused (1), descriptor version 1; kTcBK = 64: 128-byte rows, SWIZZLE_128B (2);
// kTcBK = 32: rows of 32 fp16 (64 B), 8-row atoms of 512 B, layout SWIZZLE_64B (4).
constexpr uint32_t kSwizzleAtom = 8 * kTcBK * 2;
constexpr uint64_t kLayoutType = kTcBK == 64 ? 2 : 4;
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(kSwizzleAtom >> 4) << 32) |
           ((uint64_t)1 << 46) | (kLayoutType << 61);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// pair commit: arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// 16x256b: lanes [taddr.lane, +16) x 8 columns; thread t holds row t/4, columns
// 2(t%4), 2(t%4)+1 (v[0], v[1]) and row t/4 + 8, same columns (v[2], v[3])
__device__ __forceinline__ void tmem_ld16x256(uint32_t taddr, float* v) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
// bulk tensor store shared -> global (box at {x, y}), bulk-group bookkeeping
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y), "r"(z)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

}  // namespace tc

// host: 2D fp16 row-major [rows][cols] tensor map, box [box_rows][kTcBK], 128B
// swizzle, OOB zero fill (ks_gemm_tc.cu)
bool tc_make_map(CUtensorMap* m, const void* base, long long rows, long long cols, long long row_stride_elems,
                 int box_rows);

// F16X3 operand scale: x 2^e = hi + lo (fp16 planes) with max|x| 2^e < 2^14 (no fp16
// overflow in either part, products and K-sums far inside fp32); amax_bits = the
// float bits of max|x| (non-negative floats order as ints).
__device__ __forceinline__ int f16_scale_exp(int amax_bits) {
    const float m = __int_as_float(amax_bits);
    if (!(m > 0.0f) || !isfinite(m)) return 0;
    int e;
    frexpf(m, &e);  // m < 2^e
    return max(-100, min(100, 14 - e));
}

// The training GEMM (ks_gemm16.cu): C[M x N] = alpha op(A) op(B) (+ beta C) on F16X3
// planes (hi, lo fp16, the source's row-major layout, row strides multiples of 8):
// a_mn = 0: A stored M x K (K-major); 1: A stored K x M (op(A) = A^T, MN-major);
// b_mn = 0: B stored N x K (op(B) = B^T, K-major); 1: B stored K x N (MN-major).
// alpha = 2^-(e(amaxA) + e(amaxB)); beta a device scalar (0 or 1; null: 0).
struct GemmF16Args {
    const __half* A_hi;
    const __half* A_lo;
    long long lda;
    int a_mn;
    const __half* B_hi;
    const __half* B_lo;
    long long ldb;
    int b_mn;
    int M, N;
    long long K;
    const int* amaxA;
    const int* amaxB;
    const float* beta;
    float* C;
    long long ldc;
    float* part;        // split-K workspace, gemm16_splits(M, N, K, sms) * M * N floats
    int sms;
};
int gemm16_splits(int M, int N, long long K, int sms);
// F16X3 operand planes of a row-major fp32 block: max |x| into *out (pre-zeroed; float
// bits), then hi / lo planes (row stride ldo) at the scale 2^f16_scale_exp(*amax)
void launch_absmax(const float* src, long long rows, long long cols, long long ld, int* out, cudaStream_t s);
void launch_split_planes(const float* src, long long rows, long long cols, long long ld, __half* hi, __half* lo,
                         long long ldo, const int* amax, cudaStream_t s);
bool launch_gemm16(const GemmF16Args& g, cudaStream_t stream, int* launches);
// fp32 SIMT GEMM, C[M x N] = op(A) op(B) + beta C row-major; part: split-K
// workspace of sgemm_splits(M, N, K, sms) * M * N floats (when > 1)
int sgemm_splits(int M, int N, long long K, int sms, bool ta);
bool launch_sgemm(bool ta, bool tb, int M, int N, long long K, const float* A, long long lda, const float* B,
                  long long ldb, float beta, float* C, long long ldc, float* part, int sms, cudaStream_t stream,
                  int* launches);

}  // namespace ksb
