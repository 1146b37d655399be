// Thin wrappers over CUB device-wide primitives (scan, radix sort, reduce)
// with stream-ordered temporary storage.  Plumbing for the forest layout;
// the hot kernels are hand-written.
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace hdp {

// Exclusive scan of at most kSmallScan values in ONE launch (one CTA, each
// thread a contiguous run, warp shuffles for the block prefix): the forest
// build scans many small arrays, where CUB's init + scan launches and the
// temporary allocation cost more than the work.  In-place safe.
constexpr int kSmallScan = 32768;
template <typename T>
__global__ void __launch_bounds__(1024) k_small_exscan(const T* in, T* out, int n) {
    __shared__ T wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int per = (n + 1023) / 1024;
    const int b = min(n, tid * per), e = min(n, b + per);
    T s = 0;
    for (int i = b; i < e; i++) s += in[i];
    T x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        T v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    T run = x - s + (w > 0 ? wsum[w - 1] : (T)0);
    for (int i = b; i < e; i++) {
        const T v = in[i];
        out[i] = run;
        run += v;
    }
}

template <typename T>
int exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return HDP_OK;
    if (n <= kSmallScan) {
        k_small_exscan<T><<<1, 1024, 0, st>>>(in, out, (int)n);
        note_launch();
        return HDP_OK;
    }
    size_t bytes = 0;
    HDP_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, st));
    DevBuf<char> tmp;
    HDP_TRY(tmp.alloc(bytes, st));
    HDP_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, (int)n, st));
    return HDP_OK;
}

template <typename T>
int inclusive_sum(const T* in, T* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return HDP_OK;
    size_t bytes = 0;
    HDP_CHECK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int)n, st));
    DevBuf<char> tmp;
    HDP_TRY(tmp.alloc(bytes, st));
    HDP_CHECK_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, in, out, (int)n, st));
    return HDP_OK;
}

template <typename K, typename V>
int sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int begin_bit,
               int end_bit, cudaStream_t st) {
    if (n <= 0) return HDP_OK;
    size_t bytes = 0;
    HDP_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n,
                                                   begin_bit, end_bit, st));
    DevBuf<char> tmp;
    HDP_TRY(tmp.alloc(bytes, st));
    HDP_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kin, kout, vin, vout, (int)n,
                                                   begin_bit, end_bit, st));
    return HDP_OK;
}

template <typename T>
int reduce_max(const T* in, T* out, int64_t n, cudaStream_t st) {
    size_t bytes = 0;
    HDP_CHECK_CUDA(cub::DeviceReduce::Max(nullptr, bytes, in, out, (int)n, st));
    DevBuf<char> tmp;
    HDP_TRY(tmp.alloc(bytes, st));
    HDP_CHECK_CUDA(cub::DeviceReduce::Max(tmp.get(), bytes, in, out, (int)n, st));
    return HDP_OK;
}

template <typename T>
int to_host(T* host, const T* dev, int64_t n, cudaStream_t st) {
    if (n <= 0) return HDP_OK;
    HDP_CHECK_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
    HDP_CHECK_CUDA(cudaStreamSynchronize(st));
    return HDP_OK;
}

inline int bits_for(int64_t maxval) {
    int b = 1;
    while (b < 63 && ((int64_t)1 << b) <= maxval) b++;
    return b;
}

}  // namespace hdp
