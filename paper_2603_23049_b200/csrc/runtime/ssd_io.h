// The SSD tier's I/O worker ("a dedicated thread (e.g., Prefetcher)",
// P:458 asynchronous write-back): one host thread executing chunk-record reads and writes
// between the pinned DRAM store and one pre-sized file, in FIFO order.  FIFO order is what
// makes slot reuse safe: a read of an SSD slot queued before a later write-back into the same
// slot always completes first, and a write-back reading a DRAM slot completes before a later
// load into that slot.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

namespace pcr {

class SsdIo {
 public:
  // Creates (truncates) `path` to n_slots * record_bytes.  ok() is false on failure (see error()).
  SsdIo(const std::string& path, int64_t n_slots, int64_t record_bytes);
  ~SsdIo();
  bool ok() const { return fd_ >= 0; }
  const std::string& error() const { return err_; }
  // Enqueue; returns the task's sequence number (> 0).
  int64_t read(int64_t ssd_slot, void* dst);        // SSD -> DRAM
  int64_t write(int64_t ssd_slot, const void* src); // DRAM -> SSD
  // Block until task `seq` (and every earlier task) has completed; false if any I/O failed.
  bool wait(int64_t seq);
  int64_t bytes_read() const { return bytes_read_; }
  int64_t bytes_written() const { return bytes_written_; }

 private:
  struct Task {
    int64_t seq;
    bool is_write;
    int64_t slot;
    void* buf;
  };
  void run();
  int fd_ = -1;
  bool direct_ = false;
  int64_t record_bytes_ = 0;
  std::string err_;
  std::string path_;   // created (truncated) at construction, removed at destruction
  std::mutex mu_;
  std::condition_variable cv_task_, cv_done_;
  std::deque<Task> q_;
  int64_t next_seq_ = 1, done_seq_ = 0;
  bool stop_ = false, failed_ = false;
  int64_t bytes_read_ = 0, bytes_written_ = 0;
  std::thread worker_;
};

}  // namespace pcr
