// Pinned double-buffered host staging for the large ABI transfers
// (see hostcopy.h).
#include "hostcopy.h"

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace gadi {

namespace {

// T worker threads plus the calling thread each copy one page-aligned slice.
class CopyPool {
 public:
  explicit CopyPool(int workers) : nw_(workers) {
    for (int i = 0; i < nw_; ++i) th_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t len) {
    if (nw_ == 0 || len < (size_t(4) << 20)) {
      std::memcpy(dst, src, len);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      len_ = len;
      pending_ = nw_;
      ++gen_;
    }
    cv_.notify_all();
    slice(nw_);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void slice(int id) {
    const size_t parts = (size_t)nw_ + 1;
    const size_t per = ((len_ + parts - 1) / parts + 4095) & ~size_t(4095);
    const size_t a = std::min(len_, per * (size_t)id), b = std::min(len_, a + per);
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void run(int id) {
    unsigned seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      slice(id);
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int nw_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  unsigned gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

}  // namespace

struct HostStager {
  size_t chunk = 0;
  void* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  CopyPool* pool = nullptr;
};

HostStager* stager_create(size_t chunk_bytes, int threads) {
  auto* s = new HostStager();
  s->chunk = chunk_bytes;
  for (int i = 0; i < 2; ++i) {
    if (cudaMallocHost(&s->pin[i], chunk_bytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      stager_destroy(s);
      return nullptr;
    }
  }
  if (threads <= 0) {
    const char* e = std::getenv("GADI_COPY_THREADS");
    threads = e ? std::atoi(e) : (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
  }
  // the caller copies one slice itself
  s->pool = new CopyPool(std::max(0, threads - 1));
  return s;
}

void stager_destroy(HostStager* s) {
  if (!s) return;
  for (int i = 0; i < 2; ++i) {
    if (s->ev[i]) {
      cudaEventSynchronize(s->ev[i]);
      cudaEventDestroy(s->ev[i]);
    }
    if (s->pin[i]) cudaFreeHost(s->pin[i]);
  }
  delete s->pool;
  delete s;
}

size_t stager_chunk(const HostStager* s) { return s ? s->chunk : 0; }

#define STG_TRY(x)                        \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

cudaError_t stager_h2d(HostStager* s, void* dev, const void* host, size_t bytes, cudaStream_t stream) {
  const char* h = static_cast<const char*>(host);
  char* d = static_cast<char*>(dev);
  for (size_t off = 0, k = 0; off < bytes; off += s->chunk, ++k) {
    const int b = (int)(k & 1);
    const size_t len = std::min(s->chunk, bytes - off);
    if (s->used[b]) STG_TRY(cudaEventSynchronize(s->ev[b]));  // its previous DMA is done
    s->pool->copy(s->pin[b], h + off, len);
    STG_TRY(cudaMemcpyAsync(d + off, s->pin[b], len, cudaMemcpyHostToDevice, stream));
    STG_TRY(cudaEventRecord(s->ev[b], stream));
    s->used[b] = true;
  }
  return cudaSuccess;
}

cudaError_t stager_d2h(HostStager* s, void* host, const void* dev, size_t bytes, cudaStream_t stream) {
  char* h = static_cast<char*>(host);
  const char* d = static_cast<const char*>(dev);
  const size_t nch = (bytes + s->chunk - 1) / s->chunk;
  auto issue = [&](size_t k) -> cudaError_t {
    const int b = (int)(k & 1);
    const size_t off = k * s->chunk, len = std::min(s->chunk, bytes - off);
    STG_TRY(cudaMemcpyAsync(s->pin[b], d + off, len, cudaMemcpyDeviceToHost, stream));
    STG_TRY(cudaEventRecord(s->ev[b], stream));
    s->used[b] = true;
    return cudaSuccess;
  };
  for (size_t k = 0; k < std::min<size_t>(2, nch); ++k) STG_TRY(issue(k));
  for (size_t k = 0; k < nch; ++k) {
    const int b = (int)(k & 1);
    const size_t off = k * s->chunk, len = std::min(s->chunk, bytes - off);
    STG_TRY(cudaEventSynchronize(s->ev[b]));
    s->pool->copy(h + off, s->pin[b], len);
    if (k + 2 < nch) STG_TRY(issue(k + 2));
  }
  return cudaSuccess;
}

}  // namespace gadi
