// NVLink peer-store bandwidth on this box (the ceiling for the dispatch /
// combine puts): GPU 0 writes into GPU 1's memory with (a) 16-byte SM stores
// from a grid-stride loop, (b) 4 KB cp.async.bulk stores from shared memory,
// (c) cudaMemcpyPeerAsync (copy engines).  Also GPU 0 -> {1..N-1} at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bw p2p_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void st16(const uint4* __restrict__ src, uint4* const* dst, int ndst, size_t n_per_dst) {
    // one destination per CTA slice: CTAs are split evenly over the peers
    const int d = blockIdx.x % ndst;
    const size_t cta = blockIdx.x / ndst, nct = gridDim.x / ndst;
    uint4* o = dst[d];
    for (size_t i = cta * blockDim.x + threadIdx.x; i < n_per_dst; i += nct * blockDim.x) o[i] = src[i];
}

__global__ void bulk4k(const uint4* __restrict__ src, uint4* const* dst, int ndst, size_t n_per_dst) {
    __shared__ alignas(128) uint4 buf[2][256];  // 2 x 4 KB
    const int d = blockIdx.x % ndst;
    const size_t cta = blockIdx.x / ndst, nct = gridDim.x / ndst;
    char* o = reinterpret_cast<char*>(dst[d]);
    const size_t chunks = n_per_dst / 256;
    int b = 0;
    for (size_t c = cta; c < chunks; c += nct, b ^= 1) {
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        buf[b][threadIdx.x] = src[c * 256 + threadIdx.x];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(o + c * 4096),
                         "r"(uint32_t(__cvta_generic_to_shared(buf[b]))) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("{\"p2p_bw\": \"needs >= 2 GPUs\"}\n"); return 0; }
    const size_t bytes = size_t(256) << 20;  // 256 MB per destination
    std::vector<void*> bufs(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&bufs[d], bytes));
    }
    CK(cudaSetDevice(0));
    for (int d = 1; d < n; ++d) CK(cudaDeviceEnablePeerAccess(d, 0));
    void* src;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMemset(src, 1, bytes));
    uint4** dlist;
    CK(cudaMalloc(&dlist, sizeof(uint4*) * n));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("{\"p2p_bw\": [");
    bool first = true;
    for (int ndst = 1; ndst < n; ndst *= 2) {
        std::vector<uint4*> h(ndst);
        for (int i = 0; i < ndst; ++i) h[i] = static_cast<uint4*>(bufs[1 + i]);
        CK(cudaMemcpy(dlist, h.data(), sizeof(uint4*) * ndst, cudaMemcpyHostToDevice));
        const size_t per = bytes / 16 / ndst;
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) st16<<<sms * 4, 512>>>(static_cast<uint4*>(src), dlist, ndst, per);
                else if (mode == 1) bulk4k<<<sms * 4, 256>>>(static_cast<uint4*>(src), dlist, ndst, per);
                else for (int i = 0; i < ndst; ++i) cudaMemcpyPeerAsync(h[i], 1 + i, src, 0, per * 16);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep && ms < best) best = ms;
            }
            const char* names[] = {"sm_st16", "bulk_4k", "copy_engine"};
            printf("%s{\"peers\": %d, \"mode\": \"%s\", \"GBps\": %.1f}", first ? "" : ", ", ndst, names[mode],
                   double(per * 16 * ndst) / (best * 1e-3) / 1e9);
            first = false;
        }
    }
    printf("]}\n");
    return 0;
}
