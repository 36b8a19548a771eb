// .utn payload reader: file (page cache) -> pinned host buffer -> HBM, for io.load_unitensor
// (the reference reads the payload with one numpy read, pkg/src/tnkit/io.py:83-107).
//
// The page-cache copy is the cost (one thread moves ~17 GB/s of it), so the payload is
// split into chunks read with pread() by a persistent pool of worker threads; the calling
// thread issues each chunk's cudaMemcpyAsync as soon as that chunk and every earlier one
// have landed, so the PCIe transfer runs behind the reads. Python-level threads cost more
// per chunk (GIL hand-offs, future wake-ups) than a chunk's read.
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tnb {
namespace {

struct ReadJob {
  int fd;
  int64_t off, nbytes, chunk, nch;
  unsigned char* dst;
  std::atomic<int64_t> next{0};
  std::unique_ptr<std::atomic<int>[]> state;  // per chunk: 0 pending, 1 landed, -1 short read / error
};

void run_job(ReadJob* j) {
  for (;;) {
    const int64_t k = j->next.fetch_add(1, std::memory_order_relaxed);
    if (k >= j->nch) return;
    const int64_t o = k * j->chunk;
    const int64_t n = std::min(j->chunk, j->nbytes - o);
    int64_t got = 0;
    while (got < n) {
      const ssize_t r = pread(j->fd, j->dst + o + got, (size_t)(n - got), (off_t)(j->off + o + got));
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) break;
      got += r;
    }
    j->state[k].store(got == n ? 1 : -1, std::memory_order_release);
  }
}

// Persistent workers (never joined: the pool lives for the process).
class ReadPool {
 public:
  explicit ReadPool(int n) : n_(n) {
    for (int i = 0; i < n; ++i) std::thread([this] { loop(); }).detach();
  }
  int size() const { return n_; }
  // run j on `workers` pool threads (the caller also reads); returns once all have left j
  void run(ReadJob* j, int workers) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = j;
      want_ = workers;
      busy_ = workers;
      ++gen_;
    }
    cv_.notify_all();
  }
  void wait_idle() {
    std::unique_lock<std::mutex> lk(mu_);
    idle_.wait(lk, [&] { return busy_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      ReadJob* j = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen && want_ > 0; });
        seen = gen_;
        --want_;
        j = job_;
      }
      run_job(j);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--busy_ == 0) idle_.notify_all();
      }
    }
  }
  int n_;
  std::mutex mu_;
  std::condition_variable cv_, idle_;
  uint64_t gen_ = 0;
  ReadJob* job_ = nullptr;
  int want_ = 0, busy_ = 0;
};

ReadPool& pool() {
  static ReadPool* p = new ReadPool(15);
  return *p;
}
std::mutex g_read_mu;  // one job at a time through the pool

}  // namespace
}  // namespace tnb

extern "C" int tnb_file_to_device(int fd, int64_t offset, int64_t nbytes, void* pinned, void* dst, int64_t chunk,
                                  int nthreads, void* stream) {
  using namespace tnb;
  if (fd < 0 || offset < 0 || nbytes < 0 || (nbytes > 0 && (!pinned || !dst)) || chunk <= 0 || nthreads < 1)
    return fail(TNB_EINVAL, "file_to_device: bad arguments");
  if (nbytes == 0) return TNB_OK;
  int rc = require_device();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> serial(g_read_mu);
  ReadJob j;
  j.fd = fd;
  j.off = offset;
  j.nbytes = nbytes;
  j.chunk = chunk;
  j.nch = (nbytes + chunk - 1) / chunk;
  j.dst = static_cast<unsigned char*>(pinned);
  j.state.reset(new std::atomic<int>[j.nch]);
  for (int64_t k = 0; k < j.nch; ++k) j.state[k].store(0, std::memory_order_relaxed);
  const int workers = (int)std::min<int64_t>(std::min(nthreads - 1, pool().size()), j.nch - 1);
  if (workers > 0) pool().run(&j, workers);
  // the calling thread reads too; between its chunks it issues the copies of landed ones
  int64_t issued = 0;
  bool bad = false;
  cudaError_t ce = cudaSuccess;
  auto issue_landed = [&](bool block) {
    while (issued < j.nch) {
      int s = j.state[issued].load(std::memory_order_acquire);
      if (s == 0) {
        if (!block) return;
        std::this_thread::yield();
        continue;
      }
      if (s < 0) bad = true;
      const int64_t o = issued * chunk;
      const int64_t n = std::min(chunk, nbytes - o);
      if (!bad && ce == cudaSuccess)
        ce = cudaMemcpyAsync(static_cast<unsigned char*>(dst) + o, j.dst + o, (size_t)n, cudaMemcpyHostToDevice, st);
      ++issued;
    }
  };
  for (;;) {
    const int64_t k = j.next.fetch_add(1, std::memory_order_relaxed);
    if (k >= j.nch) break;
    const int64_t o = k * chunk;
    const int64_t n = std::min(chunk, nbytes - o);
    int64_t got = 0;
    while (got < n) {
      const ssize_t r = pread(fd, j.dst + o + got, (size_t)(n - got), (off_t)(offset + o + got));
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) break;
      got += r;
    }
    j.state[k].store(got == n ? 1 : -1, std::memory_order_release);
    issue_landed(false);
  }
  issue_landed(true);
  if (workers > 0) pool().wait_idle();
  if (bad) return fail(TNB_EINVAL, "file_to_device: short read (truncated payload?)");
  if (ce != cudaSuccess) return cuda_fail(ce, "file_to_device: host->device copy");
  return TNB_OK;
}
