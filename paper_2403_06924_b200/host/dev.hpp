// Host-side plumbing of the C++ drop-in: device buffers on a per-thread
// stream, host<->device copies, and xg_status -> exception mapping
// (XG_EINVAL -> std::invalid_argument exactly where the reference throws).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "xigemm_c.h"

namespace xigemm::detail {

inline cudaStream_t stream() {
    thread_local cudaStream_t s = [] {
        cudaStream_t t = nullptr;
        if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) != cudaSuccess)
            throw std::runtime_error("xigemm: no CUDA device (the library has no CPU fallback)");
        return t;
    }();
    return s;
}

inline void check(xg_status st) {
    if (st == XG_OK) return;
    const std::string msg = xg_last_error();
    if (st == XG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("xigemm: " + msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("xigemm: ") + what + ": " + cudaGetErrorString(e));
}

inline void sync() { cuda_check(cudaStreamSynchronize(stream()), "synchronize"); }

template <class T>
class DevBuf {
  public:
    explicit DevBuf(std::size_t n) : n_(n) {
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p_), (n ? n : 1) * sizeof(T), stream()), "alloc");
    }
    DevBuf(const T* host, std::size_t n) : DevBuf(n) { upload(host); }
    explicit DevBuf(const std::vector<T>& v) : DevBuf(v.data(), v.size()) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { cudaFreeAsync(p_, stream()); }

    void upload(const T* host) {
        if (n_) cuda_check(cudaMemcpyAsync(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice, stream()), "h2d");
    }
    void download(T* host, std::size_t n) const {
        if (n) cuda_check(cudaMemcpyAsync(host, p_, n * sizeof(T), cudaMemcpyDeviceToHost, stream()), "d2h");
        sync();
    }
    std::vector<T> to_vector(std::size_t n) const {
        std::vector<T> v(n);
        download(v.data(), n);
        return v;
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }

  private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

inline xg_stream xs() { return reinterpret_cast<xg_stream>(stream()); }

}  // namespace xigemm::detail
