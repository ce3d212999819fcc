// Launch gap between a small "plan-like" kernel A (17 CTAs, PDL trigger at its
// start, ~15 us of work) and a persistent "k_moe2-like" kernel B (one CTA per
// SM, 384 threads, large dynamic shared memory, optional 2-CTA clusters,
// optional PDL / cooperative attributes).  Reports B's first / last CTA entry
// relative to A's end (globaltimer).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_gap launch_gap.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void kA(unsigned long long* tm, int pdl_trigger, uint64_t spin_ns) {
    if (pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t t0 = gtime();
    if (threadIdx.x == 0) atomicMin(tm + 0, (unsigned long long)t0);
    while (gtime() - t0 < spin_ns) {
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(tm + 1, (unsigned long long)gtime());
}

__global__ void __launch_bounds__(384, 1) kB(unsigned long long* tm) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) {
        const uint64_t t = gtime();
        atomicMin(tm + 2, (unsigned long long)t);
        atomicMax(tm + 3, (unsigned long long)t);
        if (tm[15]) sm[0] = 1;  // never taken: keeps the smem declared
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(tm + 4, (unsigned long long)gtime());
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) kBc(unsigned long long* tm) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) {
        const uint64_t t = gtime();
        atomicMin(tm + 2, (unsigned long long)t);
        atomicMax(tm + 3, (unsigned long long)t);
        if (tm[15]) sm[0] = 1;  // never taken: keeps the smem declared
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(tm + 4, (unsigned long long)gtime());
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* tm;
    cudaMalloc(&tm, 16 * sizeof(unsigned long long));
    cudaMemset(tm, 0, 16 * sizeof(unsigned long long));
    const size_t smems[] = {0, 64 * 1024, 200 * 1024};
    for (auto f : {(const void*)kB, (const void*)kBc})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("{\"n_sms\": %d, \"rows\": [\n", nsm);
    bool first = true;
    for (int cluster = 0; cluster < 2; ++cluster)
        for (size_t smem : smems)
            for (int pdl = 0; pdl < 2; ++pdl)
                for (int coop = 0; coop < 2; ++coop) {
                    double gap_first = 0, gap_last = 0, gap_wait = 0;
                    const int reps = 20;
                    int ok = 0;
                    for (int r = 0; r < reps; ++r) {
                        unsigned long long init[8] = {~0ull, 0, ~0ull, 0, ~0ull, 0, 0, 0};
                        cudaMemcpy(tm, init, sizeof(init), cudaMemcpyHostToDevice);
                        cudaDeviceSynchronize();
                        // a long-running predecessor so the host is ahead of the device
                        kA<<<1, 32>>>(tm + 8, 0, 200000);
                        kA<<<17, 256>>>(tm, pdl, 15000);
                        cudaLaunchConfig_t cfg{};
                        cfg.gridDim = dim3(nsm & ~1);
                        cfg.blockDim = dim3(384);
                        cfg.dynamicSmemBytes = smem;
                        cudaLaunchAttribute at[2];
                        int na = 0;
                        if (pdl) {
                            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                            at[na++].val.programmaticStreamSerializationAllowed = 1;
                        }
                        if (coop) {
                            at[na].id = cudaLaunchAttributeCooperative;
                            at[na++].val.cooperative = 1;
                        }
                        cfg.attrs = at;
                        cfg.numAttrs = na;
                        void* args[] = {&tm};
                        cudaError_t e = cudaLaunchKernelExC(&cfg, cluster ? (const void*)kBc : (const void*)kB, args);
                        if (e != cudaSuccess) {
                            cudaGetLastError();
                            break;
                        }
                        cudaDeviceSynchronize();
                        unsigned long long h[8];
                        cudaMemcpy(h, tm, sizeof(h), cudaMemcpyDeviceToHost);
                        gap_first += (double(h[2]) - double(h[1])) / 1e3;
                        gap_last += (double(h[3]) - double(h[1])) / 1e3;
                        gap_wait += (double(h[4]) - double(h[1])) / 1e3;
                        ++ok;
                    }
                    if (!ok) continue;
                    printf("%s{\"cluster2\": %d, \"smem_kb\": %zu, \"pdl\": %d, \"coop\": %d, \"entry_first_us\": %.2f, "
                           "\"entry_last_us\": %.2f, \"after_wait_us\": %.2f}",
                           first ? "" : ",\n", cluster, smem / 1024, pdl, coop, gap_first / ok, gap_last / ok,
                           gap_wait / ok);
                    first = false;
                }
    printf("\n]}\n");
    return 0;
}
