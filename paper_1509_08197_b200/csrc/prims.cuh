// Thin wrappers over CUB device-wide primitives (scan, radix sort, reduce)
// with stream-ordered temporary storage.  Plumbing for the forest layout;
// the hot kernels are hand-written.
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace hdp {

template <typename T>
int exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t st) {
    if (n <= 0) return HDP_OK;
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
