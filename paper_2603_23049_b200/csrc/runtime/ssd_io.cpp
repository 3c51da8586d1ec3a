#include "ssd_io.h"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>

namespace pcr {

SsdIo::SsdIo(const std::string& path, int64_t n_slots, int64_t record_bytes)
    : record_bytes_(record_bytes), path_(path) {
  // O_DIRECT (true device reads, no page cache) when records are block aligned; buffered otherwise.
  if (record_bytes % 4096 == 0) {
    fd_ = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC | O_DIRECT, 0600);
    direct_ = fd_ >= 0;
  }
  if (fd_ < 0) fd_ = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
  if (fd_ < 0) {
    err_ = std::string("open ") + path + ": " + std::strerror(errno);
    return;
  }
  if (::ftruncate(fd_, n_slots * record_bytes) != 0) {
    err_ = std::string("ftruncate: ") + std::strerror(errno);
    ::close(fd_);
    fd_ = -1;
    return;
  }
  worker_ = std::thread([this] { run(); });
}

SsdIo::~SsdIo() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_task_.notify_all();
  if (worker_.joinable()) worker_.join();
  if (fd_ >= 0) {
    ::close(fd_);
    ::unlink(path_.c_str());   // the records are meaningless without this context's index
  }
}

int64_t SsdIo::read(int64_t slot, void* dst) {
  std::lock_guard<std::mutex> g(mu_);
  const int64_t s = next_seq_++;
  q_.push_back(Task{s, false, slot, dst});
  cv_task_.notify_one();
  return s;
}

int64_t SsdIo::write(int64_t slot, const void* src) {
  std::lock_guard<std::mutex> g(mu_);
  const int64_t s = next_seq_++;
  q_.push_back(Task{s, true, slot, const_cast<void*>(src)});
  cv_task_.notify_one();
  return s;
}

bool SsdIo::wait(int64_t seq) {
  std::unique_lock<std::mutex> l(mu_);
  cv_done_.wait(l, [&] { return done_seq_ >= seq || failed_; });
  return !failed_;
}

void SsdIo::run() {
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> l(mu_);
      cv_task_.wait(l, [&] { return stop_ || !q_.empty(); });
      if (q_.empty()) return;  // stop_ and drained
      t = q_.front();
      q_.pop_front();
    }
    bool ok = true;
    int64_t off = t.slot * record_bytes_, done = 0;
    uint8_t* p = static_cast<uint8_t*>(t.buf);
    while (done < record_bytes_) {
      const ssize_t r = t.is_write ? ::pwrite(fd_, p + done, record_bytes_ - done, off + done)
                                   : ::pread(fd_, p + done, record_bytes_ - done, off + done);
      if (r <= 0) {
        if (r < 0 && errno == EINTR) continue;
        ok = false;
        break;
      }
      done += r;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      if (!ok) failed_ = true;
      if (t.is_write) bytes_written_ += done; else bytes_read_ += done;
      done_seq_ = t.seq;
    }
    cv_done_.notify_all();
  }
}

}  // namespace pcr
