// Store-pattern probe (development): how fast can 21600^2 int32 labels be
// written with the work split K5 uses (one warp per 1024-px row segment) vs
// longer-lived warps / CTAs.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int H = 21600, W = 21600, TW = 1024, NTX = (W + TW - 1) / TW;

__device__ __forceinline__ void st4(int32_t *p, int a, int b, int c, int d, uint64_t pol, int mode) {
    if (mode == 1)
        asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                     "l"(pol) : "memory");
    else if (mode == 2)
        __stcs(reinterpret_cast<int4 *>(p), make_int4(a, b, c, d));
    else
        *reinterpret_cast<int4 *>(p) = make_int4(a, b, c, d);
}

// one warp writes segments seg0, seg0+stride, ... (segs_per_warp of them)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_seg(int32_t *out, int segs_per_warp, int mode) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t nseg = (int64_t)H * NTX;
    const int64_t w = (int64_t)blockIdx.x * WARPS + wi;
    for (int j = 0; j < segs_per_warp; j++) {
        const int64_t seg = w * segs_per_warp + j;
        if (seg >= nseg) return;
        const int row = (int)(seg / NTX), tx = (int)(seg % NTX);
        const int C0 = tx * TW, vcols = min(TW, W - C0);
        int32_t *o = out + (int64_t)row * W + C0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int P = 128 * c + 4 * lane;
            if (P < vcols) st4(o + P, row, P, c, 1, pol, mode);
        }
    }
}

// flat grid-stride over the whole image (16 B per thread per step)
__global__ void __launch_bounds__(256) k_flat(int32_t *out, int mode) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int64_t n4 = (int64_t)H * W / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        st4(out + 4 * i, (int)i, 1, 2, 3, pol, mode);
}


// K5-like: each warp first loads one word per lane (dependent: the stored
// values use it), then stores its segment from registers
__global__ void __launch_bounds__(256) k_seg_dep(int32_t *out, const uint32_t *src, int mode) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t nseg = (int64_t)H * NTX;
    const int64_t seg = (int64_t)blockIdx.x * 8 + wi;
    if (seg >= nseg) return;
    const uint32_t v = __ldcg(src + seg * 32 + lane);
    const int row = (int)(seg / NTX), tx = (int)(seg % NTX);
    const int C0 = tx * TW, vcols = min(TW, W - C0);
    int32_t *o = out + (int64_t)row * W + C0;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int P = 128 * c + 4 * lane;
        const int a = __shfl_sync(0xffffffffu, (int)v, 4 * c + (lane >> 3));
        if (P < vcols) st4(o + P, a, P, c, 1, pol, mode);
    }
}

// persistent warps: segment labels staged in shared memory (double buffer) and
// written by the bulk-copy engine; the next segment's load is issued before
// the current segment is staged
template <int WARPS, int NBUF>
__global__ void __launch_bounds__(WARPS * 32) k_tma(int32_t *out, const uint32_t *src, int dep) {
    extern __shared__ __align__(128) int32_t stage[];  // [WARPS][NBUF][1024]
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const uint32_t nseg = (uint32_t)H * NTX;
    const uint32_t nw = gridDim.x * WARPS;
    uint32_t seg = blockIdx.x * WARPS + wi;
    uint32_t v = (dep && seg < nseg) ? __ldcg(src + (uint64_t)seg * 32 + lane) : 0u;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int it = 0;
    for (; seg < nseg; seg += nw, it++) {
        const uint32_t nxt = seg + nw;
        const uint32_t vn = (dep && nxt < nseg) ? __ldcg(src + (uint64_t)nxt * 32 + lane) : 0u;
        const int row = (int)(seg / NTX), tx = (int)(seg - (uint32_t)row * NTX);
        const int C0 = tx * TW, vcols = min(TW, W - C0);
        int32_t *buf = stage + (wi * NBUF + (it % NBUF)) * 1024;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int a = __shfl_sync(0xffffffffu, (int)v, 4 * c + (lane >> 3));
            *reinterpret_cast<int4 *>(buf + 128 * c + 4 * lane) = make_int4(a, row, c, 1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                         ::"l"(out + (int64_t)row * W + C0), "r"(sa), "r"(vcols * 4), "l"(pol) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        v = vn;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// NSEG segments per warp (consecutive warps take consecutive blocks of
// segments): every segment's load is issued before the first store
template <int NSEG, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_seg_depn(int32_t *out, const uint32_t *src, int interleave) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const uint32_t nseg = (uint32_t)H * NTX;
    const uint32_t nwarps = gridDim.x * WARPS;
    const uint32_t w = blockIdx.x * WARPS + wi;
    uint32_t v[NSEG];
#pragma unroll
    for (int j = 0; j < NSEG; j++) {
        const uint32_t seg = interleave ? w + j * nwarps : w * NSEG + j;
        v[j] = seg < nseg ? __ldcg(src + (uint64_t)seg * 32 + lane) : 0u;
    }
#pragma unroll
    for (int j = 0; j < NSEG; j++) {
        const uint32_t seg = interleave ? w + j * nwarps : w * NSEG + j;
        if (seg >= nseg) return;
        const int row = (int)(seg / NTX), tx = (int)(seg - (uint32_t)row * NTX);
        const int C0 = tx * TW, vcols = min(TW, W - C0);
        int32_t *o = out + (int64_t)row * W + C0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int P = 128 * c + 4 * lane;
            const int a = __shfl_sync(0xffffffffu, (int)v[j], 4 * c + (lane >> 3));
            if (P < vcols) st4(o + P, a, P, c, 1, pol, 1);
        }
    }
}
// persistent: load of segment i+1 issued before the stores of segment i
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_seg_pipe(int32_t *out, const uint32_t *src) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const uint32_t nseg = (uint32_t)H * NTX;
    const uint32_t nw = gridDim.x * WARPS;
    uint32_t seg = blockIdx.x * WARPS + wi;
    uint32_t v = seg < nseg ? __ldcg(src + (uint64_t)seg * 32 + lane) : 0u;
    for (; seg < nseg; seg += nw) {
        const uint32_t nxt = seg + nw;
        const uint32_t vn = nxt < nseg ? __ldcg(src + (uint64_t)nxt * 32 + lane) : 0u;
        const int row = (int)(seg / NTX), tx = (int)(seg - (uint32_t)row * NTX);
        const int C0 = tx * TW, vcols = min(TW, W - C0);
        int32_t *o = out + (int64_t)row * W + C0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int P = 128 * c + 4 * lane;
            const int a = __shfl_sync(0xffffffffu, (int)v, 4 * c + (lane >> 3));
            if (P < vcols) st4(o + P, a, P, c, 1, pol, 1);
        }
        v = vn;
    }
}


// Warp-specialized: producer warps load (dependent) and build each segment's
// labels in shared memory (double buffer); paired consumer warps only copy
// shared -> global with 16-B register stores.  Persistent CTAs.
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
template <int NP>
__global__ void __launch_bounds__(NP * 64) k_ws(int32_t *out, const uint32_t *src) {
    __shared__ __align__(16) int32_t buf[NP][1024];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool prod = w < NP;
    const int pair = prod ? w : w - NP;
    const uint32_t nseg = (uint32_t)H * NTX;
    const uint32_t stride = gridDim.x * NP;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int32_t *b = buf[pair];
    // lockstep pairs: both warps pass both barriers every iteration (no
    // deadlock); the producer's next load overlaps the consumer's stores
    for (uint32_t seg = blockIdx.x * NP + pair; seg < nseg; seg += stride) {
        if (prod) {
            const uint32_t v = __ldcg(src + (uint64_t)seg * 32 + lane);
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int a = __shfl_sync(0xffffffffu, (int)v, 4 * c + (lane >> 3));
                *reinterpret_cast<int4 *>(b + 128 * c + 4 * lane) = make_int4(a, (int)seg, c, 1);
            }
        }
        nb_sync(1 + 2 * pair, 64);
        int4 r[8];
        if (!prod) {
#pragma unroll
            for (int c = 0; c < 8; c++) r[c] = *reinterpret_cast<const int4 *>(b + 128 * c + 4 * lane);
        }
        nb_sync(2 + 2 * pair, 64);
        if (!prod) {
            const int row = (int)(seg / NTX), tx = (int)(seg - (uint32_t)row * NTX);
            const int C0 = tx * TW, vcols = min(TW, W - C0);
            int32_t *o = out + (int64_t)row * W + C0;
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int P = 128 * c + 4 * lane;
                if (P < vcols) st4(o + P, r[c].x, r[c].y, r[c].z, r[c].w, pol, 1);
            }
        }
    }
}

int main() {
    int32_t *out;
    cudaMalloc(&out, (size_t)H * W * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int64_t nseg = (int64_t)H * NTX;
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        const int reps = 20;
        for (int i = 0; i < reps; i++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        printf("%-40s %7.1f us  %6.0f GB/s\n", name, ms * 1e3, (double)H * W * 4 / (ms * 1e-3) / 1e9);
    };
    for (int mode = 0; mode < 1; mode++) {
        printf("-- store mode %d (%s)\n", mode, mode == 0 ? "plain" : mode == 1 ? "evict_first hint" : "st.cs");
        for (int spw : {1, 2, 4, 8}) {
            char nm[64];
            snprintf(nm, sizeof nm, "seg 8 warps/CTA, %d seg/warp", spw);
            run(nm, [&] { k_seg<8><<<(unsigned)((nseg + 8LL * spw - 1) / (8LL * spw)), 256>>>(out, spw, mode); });
        }
        run("seg 32 warps/CTA, 1 seg/warp", [&] { k_seg<32><<<(unsigned)((nseg + 31) / 32), 1024>>>(out, 1, mode); });
        run("seg 4 warps/CTA, 1 seg/warp", [&] { k_seg<4><<<(unsigned)((nseg + 3) / 4), 128>>>(out, 1, mode); });
        for (int g : {148 * 8, 148 * 16, 148 * 64})  {
            char nm[64];
            snprintf(nm, sizeof nm, "flat grid-stride %d CTAs", g);
            run(nm, [&] { k_flat<<<g, 256>>>(out, mode); });
        }
    }
    uint32_t *src;
    cudaMalloc(&src, (size_t)nseg * 32 * 4);
    cudaMemset(src, 1, (size_t)nseg * 32 * 4);
    run("K5-like dependent load + reg stores", [&] { k_seg_dep<<<(unsigned)((nseg + 7) / 8), 256>>>(out, src, 1); });
    run("K5-like dependent load + reg stores", [&] { k_seg_dep<<<(unsigned)((nseg + 7) / 8), 256>>>(out, src, 1); });
    for (int il = 0; il < 2; il++) {
        char nm[80];
        snprintf(nm, sizeof nm, "dep, 2 seg/warp il %d", il);
        run(nm, [&] { k_seg_depn<2, 8><<<(unsigned)((nseg + 15) / 16), 256>>>(out, src, il); });
        snprintf(nm, sizeof nm, "dep, 4 seg/warp il %d", il);
        run(nm, [&] { k_seg_depn<4, 8><<<(unsigned)((nseg + 31) / 32), 256>>>(out, src, il); });
    }
    for (int cps : {4, 8}) {
        char nm[80];
        snprintf(nm, sizeof nm, "dep, persistent pipelined %d CTA/SM", cps);
        run(nm, [&] { k_seg_pipe<8><<<148 * cps, 256>>>(out, src); });
    }
    for (int cps : {2, 4, 8}) {
        char nm[80];
        snprintf(nm, sizeof nm, "dep, warp-specialized 4+4 warps, %d CTA/SM", cps);
        run(nm, [&] { k_ws<4><<<148 * cps, 256>>>(out, src); });
    }
    for (int cps : {2, 4, 6}) {
        char nm[80];
        snprintf(nm, sizeof nm, "dep, warp-specialized 5+5 warps, %d CTA/SM", cps);
        run(nm, [&] { k_ws<5><<<148 * cps, 320>>>(out, src); });
    }
    for (int dep = 0; dep < 0; dep++) {
        {
            auto k = k_tma<8, 2>;
            const int smem = 8 * 2 * 4096;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int cps : {1, 2, 3}) {
                char nm[80];
                snprintf(nm, sizeof nm, "tma 8w x2buf, %d CTA/SM, dep %d", cps, dep);
                run(nm, [&] { k<<<148 * cps, 256, smem>>>(out, src, dep); });
            }
        }
        {
            auto k = k_tma<4, 3>;
            const int smem = 4 * 3 * 4096;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int cps : {2, 4}) {
                char nm[80];
                snprintf(nm, sizeof nm, "tma 4w x3buf, %d CTA/SM, dep %d", cps, dep);
                run(nm, [&] { k<<<148 * cps, 128, smem>>>(out, src, dep); });
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
