// Integer issue-rate microbenchmark: the measured denominator of bench.py's roofline.
//
// The hot path (K1/K2) is integer max-plus work: IADD3 / VIADDMNMX (DPX add+max) /
// VIMNMX / LOP3 on the ALU pipe and IMAD on the FMA pipe, plus their 16x2 SIMD forms.
// This program runs each instruction class (and the ALU+FMA mix the kernels use) at full
// occupancy -- 148 SMs x 2048 threads, 8 independent dependency chains per thread so
// issue, not latency, is the limit -- and reports lane-operations per clock per SM and
// Gop/s at the clock it ran at (CUDA events over the launch; SM clock from clock64()
// deltas over the same launch).  One "op" = one SASS instruction executed by one lane;
// the 16x2 forms count 2 ops per lane (two 16-bit results).  Output: one JSON object.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/intpeak scripts/micro/intpeak.cu
// Check the SASS (cuobjdump -sass scripts/micro/intpeak | grep -c VIADDMNMX) before trusting it.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8        // independent chains per thread
#define UNR 32      // unrolled steps per loop iteration (per chain)

enum Kind { K_IADD3, K_VIADDMNMX, K_LOP3, K_IMAD, K_MIX_DPX_IMAD, K_VIADDMNMX16x2,
            K_VIADD16x2, NKIND };
static const char* kName[NKIND] = {"iadd3", "viaddmnmx", "lop3", "imad",
                                   "viaddmnmx+imad", "viaddmnmx.s16x2", "vadd.s16x2"};
static const int kOpsPerInst[NKIND] = {1, 1, 1, 1, 1, 2, 2};

template <int K>
__device__ __forceinline__ void step(uint32_t (&a)[CH], uint32_t b, uint32_t c) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        if constexpr (K == K_IADD3) {
            asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        } else if constexpr (K == K_VIADDMNMX) {
            a[i] = (uint32_t)__viaddmax_s32((int)a[i], (int)b, (int)c ^ i);
        } else if constexpr (K == K_LOP3) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
        } else if constexpr (K == K_IMAD) {
            asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        } else if constexpr (K == K_MIX_DPX_IMAD) {
            if (i & 1) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
            else a[i] = (uint32_t)__viaddmax_s32((int)a[i], (int)b, (int)c ^ i);
        } else if constexpr (K == K_VIADDMNMX16x2) {
            a[i] = __viaddmax_s16x2(a[i], b, c ^ i);
        } else {
            a[i] = __vadd2(a[i], b ^ i);
        }
    }
}

template <int K>
__global__ void __launch_bounds__(256) kern(uint32_t seed, int iters, uint32_t* out,
                                           long long* cycles) {
    uint32_t a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + 1) + i;
    uint32_t b = seed ^ blockIdx.x, c = seed + threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) step<K>(a, b, c);
    }
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s ^= a[i];
    if (s == 0x9e3779b9u) out[blockIdx.x] = s;  // never true in practice; keeps the chains live
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cycles, (unsigned long long)(t1 - t0));
}

template <int K>
static void run(int sms, int iters, uint32_t* out, long long* dcyc, FILE* f, bool last) {
    const int threads = 256, blocks = sms * 8;  // 2048 threads per SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<K><<<blocks, threads>>>(1u, iters / 8, out, dcyc);  // warm-up (clocks up)
    float best_ms = 1e30f;
    long long cyc = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(dcyc, 0, sizeof(long long));
        cudaEventRecord(e0);
        kern<K><<<blocks, threads>>>(1u + rep, iters, out, dcyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_ms) {
            best_ms = ms;
            cudaMemcpy(&cyc, dcyc, sizeof(long long), cudaMemcpyDeviceToHost);
        }
    }
    // one SASS instruction per chain step (add+add fuses into one IADD3; checked with cuobjdump)
    double inst = (double)blocks * threads * (double)iters * UNR * CH;
    double ops = inst * kOpsPerInst[K];
    double sec = best_ms / 1e3;
    double mhz = cyc / sec / 1e6;  // per-SM cycles of the longest block over the launch time
    double per_clk_sm = inst / (cyc * (double)sms);  // lane-instructions / clk / SM (PTX count)
    fprintf(f, "  \"%s\": {\"ms\": %.4f, \"gops\": %.1f, \"lane_inst_per_clk_per_sm\": %.2f, "
               "\"sm_mhz_est\": %.0f, \"ops_per_inst\": %d}%s\n",
            kName[K], best_ms, ops / sec / 1e9, per_clk_sm, mhz, kOpsPerInst[K], last ? "" : ",");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main(int argc, char** argv) {
    int iters = argc > 1 ? atoi(argv[1]) : 2048;
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    int sms = pr.multiProcessorCount;
    uint32_t* out;
    long long* dcyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&dcyc, sizeof(long long));
    FILE* f = stdout;
    fprintf(f, "{\"device\": \"%s\", \"sms\": %d, \"threads_per_sm\": 2048, \"chains\": %d,\n", pr.name,
            sms, CH);
    run<K_IADD3>(sms, iters, out, dcyc, f, false);
    run<K_VIADDMNMX>(sms, iters, out, dcyc, f, false);
    run<K_LOP3>(sms, iters, out, dcyc, f, false);
    run<K_IMAD>(sms, iters, out, dcyc, f, false);
    run<K_MIX_DPX_IMAD>(sms, iters, out, dcyc, f, false);
    run<K_VIADDMNMX16x2>(sms, iters, out, dcyc, f, false);
    run<K_VIADD16x2>(sms, iters, out, dcyc, f, true);
    fprintf(f, "}\n");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
