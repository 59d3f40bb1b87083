// Launch-time probe of the gate GEMM (GPU box): warm CUDA-event time of one
// lstm_gemm_tc launch over M rows (optionally a fan-out epilogue), H = K = 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2404_10162_b200/csrc tools/tiny_gemm.cu \
//        -L paper_2404_10162_b200 -lks_b200 -Xlinker -rpath=$PWD/paper_2404_10162_b200 -lcuda -o /tmp/tiny_gemm
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ks_common.cuh"

namespace ksb {
bool launch_lstm_tc(const LstmArgs& a0, const LstmArgs* a1, int mode, const __half* W_hi0, const __half* W_lo0,
                    const __half* W_hi1, const __half* W_lo1, cudaStream_t stream, int* launches, int units,
                    bool pair);
}

int main(int argc, char** argv) {
    const int H = 256, K = 256, units = argc > 1 ? atoi(argv[1]) : 64;
    const bool noslot = argc > 2 && atoi(argv[2]), noha = argc > 3 && atoi(argv[3]);
    const long long maxM = 65536 * 9;
    __half *A, *W, *hA;
    float *G, *c, *h, *co;
    int* slot;
    cudaMalloc(&A, (size_t)maxM * K * 2 * 2);
    cudaMalloc(&W, (size_t)4 * H * K * 2 * 2);
    cudaMalloc(&G, (size_t)16 * 4 * H * 4);
    cudaMalloc(&c, (size_t)maxM * H * 4);
    cudaMalloc(&h, (size_t)maxM * H * 4);
    cudaMalloc(&co, (size_t)maxM * H * 4);
    cudaMalloc(&hA, (size_t)maxM * H * 2 * 2);
    cudaMalloc(&slot, (size_t)maxM * 4);
    cudaMemset(A, 0, (size_t)maxM * K * 4);
    cudaMemset(W, 0, (size_t)4 * H * K * 4);
    cudaMemset(G, 0, (size_t)16 * 4 * H * 4);
    cudaMemset(c, 0, (size_t)maxM * H * 4);
    cudaMemset(slot, 0, (size_t)maxM * 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int Ms[] = {1, 9, 81, 128, 648, 1024, 5184, 16384, 65536};
    for (int fan : {0, 9})
        for (int M : Ms) {
            ksb::LstmArgs p{};
            p.M = M;
            p.H = H;
            p.K = K;
            p.A_hi = A;
            p.A_lo = A + (size_t)maxM * K;
            p.ldah = K;
            p.G = G;
            p.slot_ptr = slot;
            p.slot_stride = 1;
            p.c_prev = c;
            p.ldc_prev = H;
            p.h_out = h;
            p.ldh = H;
            p.c_out = co;
            p.ldc = H;
            p.hA_hi = hA;
            p.hA_lo = hA + (size_t)maxM * H;
            p.ldha = H;
            p.fan = fan;
            if (noslot) p.slot_ptr = nullptr;
            if (noha) p.hA_hi = p.hA_lo = nullptr;
            int n = 0;
            for (int w = 0; w < 3; ++w)
                ksb::launch_lstm_tc(p, nullptr, 0, W, W + 4 * H * K, nullptr, nullptr, s, &n, units, false);
            cudaEventRecord(e0, s);
            const int reps = 20;
            bool ok = true;
            for (int r = 0; r < reps; ++r)
                ok &= ksb::launch_lstm_tc(p, nullptr, 0, W, W + 4 * H * K, nullptr, nullptr, s, &n, units, false);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("fan %d M %6d: %8.1f us/launch %s %s\n", fan, M, 1000.f * ms / reps, ok ? "" : "LAUNCH FAILED",
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
