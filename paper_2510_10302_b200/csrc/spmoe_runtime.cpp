// spmoe_runtime.cpp — native expert-cache runtime: the HBM slot table with
// the reference's LRU semantics (moesim cache.py:34-143), the demand-load
// path (prefetch.py:276-301) and the asynchronous prefetch worker thread of
// Algorithm 2 (task protocol of prefetch.py:118-223,
// live-thread model prefetch.py:316-371).
//
// Cache metadata is mutated only under `mu_`; the worker mutates it while
// drafting and the verify stage mutates it after spmoe_rt_drain(), so the
// sequence of cache operations — and therefore every prefetched / evicted
// expert set — is a deterministic function of the predictor outputs.
// Copies are tracked per slot: a ready event recorded on the copy stream
// after the slot's copy, and a read event recorded on the compute stream
// after kernels that read the slot (the copy stream waits on it before the
// slot is overwritten).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/spmoe.h"

namespace {

struct Task {
  int layer;
  const int32_t* host_idx;
  int k;
  cudaEvent_t ready;
  int issue_token;
  const volatile int32_t* flag;  // device-bumped completion counter (or null)
  int32_t expected;
};

struct WindowEntry {
  std::vector<int> ids, victims;
};

struct Transfer {
  int layer;
  int kind;  // 0 prefetch, 1 demand
  int seq;
  std::vector<int> experts;
  cudaEvent_t start, end;
  cudaEvent_t copy_end;  // after the last H2D (XC tier: before its decode)
  int64_t wire_bytes;  // bytes that crossed the host link
  // once the copies are done the three events are turned into times (ms
  // since the runtime epoch) and recycled, so a long run holds a bounded
  // number of live events (spmoe_rt::resolve_log)
  bool resolved = false;
  float t_start = -1.0f, t_end = -1.0f, t_copy_end = -1.0f;
};

// Bound on the consumer's flag / event wait for one prefetch task, as the
// reference bounds the live worker's checkpoint wait (prefetch.py:353-355).
constexpr double kHandoffTimeoutS = 5.0;
// Live timing events kept before finished ones are resolved and recycled.
constexpr size_t kLiveTransfers = 512;
constexpr size_t kLiveDecodeTimings = 1024;

}  // namespace

struct spmoe_rt {
  // identity
  int capacity, L, E, device;
  char* dev_pool;
  const char* host_pool;
  std::vector<int32_t> host_index;
  size_t slot_bytes;
  cudaStream_t copy_stream;
  bool batched;

  // LRU over keys (layer*E + expert): intrusive doubly linked list, head =
  // least recently used
  std::vector<int> prev, next, slot_of;
  std::vector<char> pinned_flag;
  int head = -1, tail = -1, n_resident = 0, n_pinned = 0;
  std::vector<int> free_slots;  // kept sorted descending; pop_back = lowest

  // per-slot events
  std::vector<cudaEvent_t> ready_ev, read_ev;
  std::vector<char> ready_rec, read_rec;

  // XC host tier (spmoe_rt_set_codec): host rows are XC blobs; each copy
  // lands in a staging buffer and the decode stream expands it into the slot
  bool codec = false;
  size_t row_stride = 0;
  std::vector<char*> staging;
  size_t staging_bytes = 0;
  std::vector<cudaEvent_t> stage_full, stage_free;  // stage_full: [stage][segment]
  std::vector<char> stage_used;
  int stage_next = 0;
  cudaStream_t decode_stream = nullptr;
  // optional decode-kernel timing (spmoe_rt_decode_timing): event pairs
  // around each segment decode, with the bytes it read (blob) and wrote
  int time_decode = 0;  // 1: event pairs, 2: device-clock spans
  struct DecodeTiming {
    cudaEvent_t a, b;
    int64_t bytes;
  };
  std::vector<DecodeTiming> dec_times;
  // device-clock spans: a zeroed device ring of {t0, t1} (ns), one per
  // timed launch, with the bytes each launch read + wrote
  static constexpr int kSpanCap = 1 << 17;
  unsigned long long* dspans = nullptr;
  std::vector<int64_t> dspan_bytes;
  double dec_ms_acc = 0.0;  // resolved decode timings not yet reported
  int64_t dec_bytes_acc = 0, dec_n_acc = 0;

  // counters
  int64_t hits = 0, misses = 0, evictions = 0, prefetch_evictions = 0, prefetch_insertions = 0,
          demand_insertions = 0, tasks_completed = 0, tasks_aborted = 0, prefetch_bytes = 0,
          demand_bytes = 0, evictions_of_queued = 0, prefetch_wire = 0, demand_wire = 0,
          handoff_timeouts = 0;

  // first CUDA error seen by a copy / event / hand-off since the last
  // spmoe_rt_drain (which returns and clears it); guarded by mu_
  int err_ = 0;
  int fail_copies_ = 0;  // fault injection (spmoe_rt_debug_fail_copies)
  void note_error(int st) {
    if (st != 0 && err_ == 0) err_ = st;
  }

  // worker
  std::mutex mu_;
  std::mutex qmu_;
  std::condition_variable qcv_, done_cv_;
  std::deque<Task> queue_;
  int64_t pushed_ = 0, processed_ = 0;
  bool stop_ = false, running_ = false;
  std::thread worker_;

  // tasks consumed since the last drain (for evictions_of_queued_targets)
  std::vector<WindowEntry> window_;

  // transfer log
  std::vector<Transfer> log_;
  size_t first_live_ = 0;  // log_[i] for i < first_live_ are resolved
  cudaEvent_t epoch_ = nullptr;
  int seq_ = 0;
  std::vector<cudaEvent_t> free_ev_;  // recycled timing events

  // ---------------------------------------------------------------- LRU
  void unlink(int key) {
    const int p = prev[key], n = next[key];
    if (p >= 0) next[p] = n; else head = n;
    if (n >= 0) prev[n] = p; else tail = p;
    prev[key] = next[key] = -1;
  }
  void append(int key) {
    prev[key] = tail;
    next[key] = -1;
    if (tail >= 0) next[tail] = key; else head = key;
    tail = key;
  }
  bool resident(int key) const { return slot_of[key] >= 0; }

  bool lookup(int key, bool touch) {
    const bool hit = resident(key);
    if (touch) {
      if (hit) {
        ++hits;
        unlink(key);
        append(key);
      } else {
        ++misses;
      }
    }
    return hit;
  }

  // insert_batch semantics of cache.py:79-122: dedupe keeping first
  // occurrence, victims head-first skipping pinned and batch members, then
  // every batch member moves to the tail in argument order.  New members
  // take free slots (lowest index first) after the victims release theirs.
  // Returns false (no mutation) on a contract violation.
  bool insert_batch(const std::vector<int>& ids_in, int kind, std::vector<int>& victims) {
    std::vector<int> batch;
    batch.reserve(ids_in.size());
    for (int k : ids_in)
      if (std::find(batch.begin(), batch.end(), k) == batch.end()) batch.push_back(k);
    if ((int)batch.size() > capacity - n_pinned) return false;
    int n_new = 0;
    for (int k : batch) n_new += resident(k) ? 0 : 1;
    const int overflow = std::max(0, n_resident + n_new - capacity);
    victims.clear();
    if (overflow > 0) {
      for (int k = head; k >= 0 && (int)victims.size() < overflow; k = next[k]) {
        if (pinned_flag[k]) continue;
        if (std::find(batch.begin(), batch.end(), k) != batch.end()) continue;
        victims.push_back(k);
      }
      if ((int)victims.size() < overflow) {
        victims.clear();
        return false;
      }
    }
    for (int v : victims) {
      unlink(v);
      free_slots.push_back(slot_of[v]);
      slot_of[v] = -1;
      --n_resident;
    }
    std::sort(free_slots.begin(), free_slots.end(), std::greater<int>());
    evictions += (int64_t)victims.size();
    if (kind == 0) {
      prefetch_evictions += (int64_t)victims.size();
      prefetch_insertions += n_new;
    } else {
      demand_insertions += n_new;
    }
    for (int k : batch) {
      if (resident(k)) {
        unlink(k);
      } else {
        slot_of[k] = free_slots.back();
        free_slots.pop_back();
        ++n_resident;
      }
      append(k);
    }
    return true;
  }

  // ------------------------------------------------------------- copies
  cudaEvent_t new_timing_event() {
    if (!free_ev_.empty()) {
      cudaEvent_t e = free_ev_.back();
      free_ev_.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void recycle(cudaEvent_t& e) {
    if (e) free_ev_.push_back(e);
    e = nullptr;
  }

  // Turn a finished transfer's events into times and recycle them.
  bool resolve(Transfer& tr) {
    if (tr.resolved) return true;
    if (cudaEventQuery(tr.end) != cudaSuccess || cudaEventQuery(tr.copy_end) != cudaSuccess) return false;
    cudaEventElapsedTime(&tr.t_start, epoch_, tr.start);
    cudaEventElapsedTime(&tr.t_end, epoch_, tr.end);
    cudaEventElapsedTime(&tr.t_copy_end, epoch_, tr.copy_end);
    recycle(tr.start);
    recycle(tr.end);
    recycle(tr.copy_end);
    tr.resolved = true;
    return true;
  }
  // Keep at most kLiveTransfers transfers holding events: resolve the oldest
  // ones that have finished (in order; stops at the first still in flight).
  void resolve_log() {
    while (log_.size() - first_live_ > kLiveTransfers && resolve(log_[first_live_])) ++first_live_;
  }
  void resolve_decode_timings() {
    if (dec_times.size() <= kLiveDecodeTimings) return;
    size_t i = 0;
    for (; i < dec_times.size(); ++i) {
      auto& t = dec_times[i];
      if (cudaEventQuery(t.b) != cudaSuccess) break;
      float x = 0.0f;
      if (cudaEventElapsedTime(&x, t.a, t.b) == cudaSuccess) {
        dec_ms_acc += x;
        dec_bytes_acc += t.bytes;
        ++dec_n_acc;
      }
      recycle(t.a);
      recycle(t.b);
    }
    dec_times.erase(dec_times.begin(), dec_times.begin() + i);
  }
  // Undo the installation of keys whose copies were never issued (a failed
  // copy must not leave an expert marked resident over stale slot bytes).
  void uninstall(const std::vector<int>& keys) {
    for (int k : keys) {
      if (!resident(k)) continue;
      if (pinned_flag[k]) {
        pinned_flag[k] = 0;
        --n_pinned;
      }
      unlink(k);
      free_slots.push_back(slot_of[k]);
      slot_of[k] = -1;
      --n_resident;
    }
    std::sort(free_slots.begin(), free_slots.end(), std::greater<int>());
  }

  const char* host_row(int key) const {
    const int hidx = host_index.empty() ? key : host_index[key];
    return host_pool + (size_t)hidx * (codec ? row_stride : slot_bytes);
  }

  // Raw tier: one H2D copy per expert straight into its slot, after the
  // slot's last readers (read event) are done.
  cudaError_t copy_raw(int s, const char* src, int64_t& wire) {
    cudaError_t st = cudaSuccess;
    if (read_rec[s]) st = cudaStreamWaitEvent(copy_stream, read_ev[s], 0);
    if (st == cudaSuccess)
      st = cudaMemcpyAsync(dev_pool + (size_t)s * slot_bytes, src, slot_bytes, cudaMemcpyHostToDevice,
                           copy_stream);
    if (st == cudaSuccess) st = cudaEventRecord(ready_ev[s], copy_stream);
    wire += (int64_t)slot_bytes;
    return st;
  }

  // XC tier: H2D of the blob into the next staging buffer (once the decode
  // that last used it is done), one copy per segment; on the decode stream:
  // wait for the slot's readers, then decode each segment as soon as its
  // bytes have landed, free the buffer, mark the slot ready.  The link never
  // waits for a slot's readers, and after the last byte lands only the last
  // segment (W2) remains to decode.
  cudaError_t copy_xc(int s, const char* src, int64_t& wire) {
    const spmoe_xc_header* h = (const spmoe_xc_header*)src;
    const int i = stage_next;
    stage_next = (stage_next + 1) % (int)staging.size();
    const int ns = (int)h->nseg;
    cudaError_t st = cudaSuccess;
    if (stage_used[i]) st = cudaStreamWaitEvent(copy_stream, stage_free[i], 0);
    if (st == cudaSuccess && read_rec[s]) st = cudaStreamWaitEvent(decode_stream, read_ev[s], 0);
    uint16_t* dst = (uint16_t*)(dev_pool + (size_t)s * slot_bytes);
    for (int g = 0; g < ns && st == cudaSuccess; ++g) {
      // a segment's streams are contiguous from its decode table on
      const uint64_t lo = g == 0 ? 0 : h->seg[g].off_lut;
      const uint64_t hi = g + 1 < ns ? h->seg[g + 1].off_lut : h->blob_bytes;
      cudaEvent_t full = stage_full[i * SPMOE_XC_MAX_SEG + g];
      st = cudaMemcpyAsync(staging[i] + lo, src + lo, hi - lo, cudaMemcpyHostToDevice, copy_stream);
      if (st == cudaSuccess) st = cudaEventRecord(full, copy_stream);
      if (st == cudaSuccess) st = cudaStreamWaitEvent(decode_stream, full, 0);
      DecodeTiming dt{nullptr, nullptr, 0};
      const int64_t dbytes = (int64_t)(hi - lo) + 2 * (int64_t)h->seg[g].n;
      if (st == cudaSuccess && time_decode == 1) {
        dt.a = new_timing_event();
        dt.b = new_timing_event();
        dt.bytes = dbytes;
        st = cudaEventRecord(dt.a, decode_stream);
      }
      void* span = nullptr;
      if (time_decode == 2 && dspans && (int)dspan_bytes.size() < kSpanCap) {
        span = dspans + 2 * dspan_bytes.size();
        dspan_bytes.push_back(dbytes);
      }
      if (st == cudaSuccess)
        st = (cudaError_t)spmoe_xc_decode_segments_timed((const uint8_t*)staging[i], h, g, 1, dst, decode_stream,
                                                         span);
      if (st == cudaSuccess && time_decode == 1) {
        st = cudaEventRecord(dt.b, decode_stream);
        dec_times.push_back(dt);
      }
    }
    if (st == cudaSuccess) st = cudaEventRecord(stage_free[i], decode_stream);
    stage_used[i] = 1;
    if (st == cudaSuccess) st = cudaEventRecord(ready_ev[s], decode_stream);
    wire += (int64_t)h->blob_bytes;
    return st;
  }

  // Issue the copies of `keys` (already installed) on the copy stream.
  int issue_copies(const std::vector<int>& keys, int layer, int kind) {
    if (keys.empty()) return 0;
    Transfer tr;
    tr.layer = layer;
    tr.kind = kind;
    tr.seq = seq_++;
    tr.wire_bytes = 0;
    for (int k : keys) tr.experts.push_back(k % E);
    tr.start = new_timing_event();
    tr.end = new_timing_event();
    tr.copy_end = new_timing_event();
    cudaError_t st = cudaEventRecord(tr.start, copy_stream);
    size_t done = 0;  // keys whose copy (and ready event) was issued
    for (size_t i = 0; i < keys.size() && st == cudaSuccess; ++i) {
      const int k = keys[i];
      const int s = slot_of[k];
      if (fail_copies_ > 0) {
        --fail_copies_;
        st = cudaErrorInvalidValue;
        break;
      }
      st = codec ? copy_xc(s, host_row(k), tr.wire_bytes) : copy_raw(s, host_row(k), tr.wire_bytes);
      if (st != cudaSuccess) break;
      ready_rec[s] = 1;
      ++done;
      if (!batched && kind == 0 && i + 1 < keys.size()) {
        // unbatched I/O (PolicySpec.batched_io = false): one copy launch at
        // a time, each completed before the next is issued
        st = cudaStreamSynchronize(copy_stream);
      }
    }
    if (done < keys.size()) uninstall(std::vector<int>(keys.begin() + done, keys.end()));
    // the transfer ends when its last expert is usable (after its decode)
    if (st == cudaSuccess) st = cudaEventRecord(tr.copy_end, copy_stream);
    if (st == cudaSuccess) st = cudaEventRecord(tr.end, codec ? decode_stream : copy_stream);
    const int64_t nbytes = (int64_t)keys.size() * (int64_t)slot_bytes;
    if (kind == 0) {
      prefetch_bytes += nbytes;
      prefetch_wire += tr.wire_bytes;
    } else {
      demand_bytes += nbytes;
      demand_wire += tr.wire_bytes;
    }
    log_.push_back(std::move(tr));
    resolve_log();
    if (time_decode == 1) resolve_decode_timings();
    note_error((int)st);
    return (int)st;
  }

  // -------------------------------------------------------------- worker
  void run_task(const Task& t) {
    int wait_st = 0;
    if (t.flag) {
      // graph-safe hand-off: the predictor's completion counter in mapped
      // memory reaches `expected` once this replay's indices are visible;
      // bounded like the reference's checkpoint wait (prefetch.py:353-355)
      const auto t0 = std::chrono::steady_clock::now();
      int spins = 0;
      while (*t.flag < t.expected) {
        if (++spins > 64) {
          std::this_thread::sleep_for(std::chrono::microseconds(2));
          if ((spins & 1023) == 0 &&
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kHandoffTimeoutS) {
            wait_st = (int)cudaErrorTimeout;
            break;
          }
        }
      }
    } else if (t.ready) {
      wait_st = (int)cudaEventSynchronize(t.ready);
    }
    std::lock_guard<std::mutex> g(mu_);
    if (wait_st != 0) {
      // the task's indices never became valid: drop it, count it, and
      // surface the error at the next drain
      if (wait_st == (int)cudaErrorTimeout) ++handoff_timeouts;
      ++tasks_aborted;
      note_error(wait_st);
      window_.push_back(WindowEntry{});
      return;
    }
    // pop-time residency filter (enqueue_critical prefetch.py:131-135 and the
    // worker re-check prefetch.py:186-189 collapse into one probe here,
    // because the predicted ids live on the device until the kernel is done)
    WindowEntry we;
    std::vector<int> load;
    for (int i = 0; i < t.k; ++i) {
      const int e = ((volatile const int32_t*)t.host_idx)[i];
      if (e < 0 || e >= E) continue;
      const int key = t.layer * E + e;
      we.ids.push_back(key);
      if (!resident(key) && std::find(load.begin(), load.end(), key) == load.end())
        load.push_back(key);
    }
    if (!load.empty()) {
      std::vector<int> victims;
      if (insert_batch(load, 0, victims)) {
        we.victims = victims;
        if (issue_copies(load, t.layer, 0) == 0) ++tasks_completed;
        else ++tasks_aborted;
      }
    }
    window_.push_back(std::move(we));
  }

  // Victims of a task that are predicted targets of a LATER task of the same
  // drafting window (simcore.py:275-278), evaluated once every task of the
  // window has been consumed, so the count is deterministic.
  void close_window() {
    std::lock_guard<std::mutex> g(mu_);
    for (size_t i = 0; i < window_.size(); ++i)
      for (int v : window_[i].victims) {
        bool hit = false;
        for (size_t j = i + 1; j < window_.size() && !hit; ++j)
          hit = std::find(window_[j].ids.begin(), window_[j].ids.end(), v) != window_[j].ids.end();
        if (hit) ++evictions_of_queued;
      }
    window_.clear();
  }

  void worker_loop() {
    cudaSetDevice(device);
    for (;;) {
      Task t;
      {
        std::unique_lock<std::mutex> q(qmu_);
        qcv_.wait(q, [&] { return stop_ || !queue_.empty(); });
        if (queue_.empty()) return;  // stop requested and nothing left
        t = queue_.front();
        queue_.pop_front();
      }
      run_task(t);
      {
        std::lock_guard<std::mutex> q(qmu_);
        ++processed_;
      }
      done_cv_.notify_all();
    }
  }
};

extern "C" {

spmoe_rt* spmoe_rt_create(int capacity, int num_layers, int num_experts, void* dev_pool,
                          const void* host_pool, const int32_t* host_index, size_t slot_bytes,
                          void* copy_stream, int batched_io) {
  if (capacity < 1 || num_layers < 1 || num_experts < 1) return nullptr;
  spmoe_rt* rt = new spmoe_rt();
  rt->capacity = capacity;
  rt->L = num_layers;
  rt->E = num_experts;
  cudaGetDevice(&rt->device);
  rt->dev_pool = (char*)dev_pool;
  rt->host_pool = (const char*)host_pool;
  const int n = num_layers * num_experts;
  if (host_index) rt->host_index.assign(host_index, host_index + n);
  rt->slot_bytes = slot_bytes;
  rt->copy_stream = (cudaStream_t)copy_stream;
  rt->batched = batched_io != 0;
  rt->prev.assign(n, -1);
  rt->next.assign(n, -1);
  rt->slot_of.assign(n, -1);
  rt->pinned_flag.assign(n, 0);
  for (int s = capacity - 1; s >= 0; --s) rt->free_slots.push_back(s);
  rt->ready_ev.resize(capacity);
  rt->read_ev.resize(capacity);
  rt->ready_rec.assign(capacity, 0);
  rt->read_rec.assign(capacity, 0);
  for (int s = 0; s < capacity; ++s) {
    cudaEventCreateWithFlags(&rt->ready_ev[s], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&rt->read_ev[s], cudaEventDisableTiming);
  }
  rt->epoch_ = rt->new_timing_event();
  cudaEventRecord(rt->epoch_, rt->copy_stream);
  return rt;
}

void spmoe_rt_destroy(spmoe_rt* rt) {
  if (!rt) return;
  spmoe_rt_worker_stop(rt);
  cudaStreamSynchronize(rt->copy_stream);
  if (rt->decode_stream) cudaStreamSynchronize(rt->decode_stream);
  for (auto e : rt->stage_full) cudaEventDestroy(e);
  for (auto e : rt->stage_free) cudaEventDestroy(e);
  for (auto e : rt->ready_ev) cudaEventDestroy(e);
  for (auto e : rt->read_ev) cudaEventDestroy(e);
  for (auto& t : rt->log_) {
    if (t.resolved) continue;
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.end);
    cudaEventDestroy(t.copy_end);
  }
  for (auto& t : rt->dec_times) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : rt->free_ev_) cudaEventDestroy(e);
  if (rt->dspans) cudaFree(rt->dspans);
  if (rt->epoch_) cudaEventDestroy(rt->epoch_);
  delete rt;
}

static inline bool valid_id(spmoe_rt* rt, int layer, int expert) {
  return layer >= 0 && layer < rt->L && expert >= 0 && expert < rt->E;
}

int spmoe_rt_lookup(spmoe_rt* rt, int layer, int expert, int touch) {
  if (!rt || !valid_id(rt, layer, expert)) return 0;
  std::lock_guard<std::mutex> g(rt->mu_);
  return rt->lookup(layer * rt->E + expert, touch != 0) ? 1 : 0;
}

int spmoe_rt_slot_of(spmoe_rt* rt, int layer, int expert) {
  if (!rt || !valid_id(rt, layer, expert)) return -1;
  std::lock_guard<std::mutex> g(rt->mu_);
  return rt->slot_of[layer * rt->E + expert];
}

int spmoe_rt_insert_batch(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n,
                          int kind, int32_t* victims_out) {
  if (!rt || n < 0) return -1;
  std::vector<int> ids;
  for (int i = 0; i < n; ++i) {
    if (!valid_id(rt, layers[i], experts[i])) return -1;
    ids.push_back(layers[i] * rt->E + experts[i]);
  }
  std::lock_guard<std::mutex> g(rt->mu_);
  std::vector<int> victims;
  if (!rt->insert_batch(ids, kind, victims)) return -1;
  if (victims_out)
    for (size_t i = 0; i < victims.size(); ++i) {
      victims_out[2 * i] = victims[i] / rt->E;
      victims_out[2 * i + 1] = victims[i] % rt->E;
    }
  return (int)victims.size();
}

int spmoe_rt_pin(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n) {
  if (!rt) return -1;
  std::lock_guard<std::mutex> g(rt->mu_);
  for (int i = 0; i < n; ++i) {
    if (!valid_id(rt, layers[i], experts[i])) return -1;
    const int key = layers[i] * rt->E + experts[i];
    if (!rt->resident(key)) return -1;  // CacheError: pin non-resident
    if (!rt->pinned_flag[key]) {
      rt->pinned_flag[key] = 1;
      ++rt->n_pinned;
    }
  }
  return 0;
}

void spmoe_rt_unpin(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n) {
  if (!rt) return;
  std::lock_guard<std::mutex> g(rt->mu_);
  for (int i = 0; i < n; ++i) {
    if (!valid_id(rt, layers[i], experts[i])) continue;
    const int key = layers[i] * rt->E + experts[i];
    if (rt->pinned_flag[key]) {
      rt->pinned_flag[key] = 0;
      --rt->n_pinned;
    }
  }
}

int spmoe_rt_lru_order(spmoe_rt* rt, int32_t* layers, int32_t* experts, int cap) {
  if (!rt) return 0;
  std::lock_guard<std::mutex> g(rt->mu_);
  int n = 0;
  for (int k = rt->head; k >= 0 && n < cap; k = rt->next[k], ++n) {
    layers[n] = k / rt->E;
    experts[n] = k % rt->E;
  }
  return n;
}

void spmoe_rt_counters(spmoe_rt* rt, int64_t* o) {
  if (!rt || !o) return;
  std::lock_guard<std::mutex> g(rt->mu_);
  o[0] = rt->hits; o[1] = rt->misses; o[2] = rt->evictions; o[3] = rt->prefetch_evictions;
  o[4] = rt->prefetch_insertions; o[5] = rt->demand_insertions; o[6] = rt->tasks_completed;
  o[7] = rt->tasks_aborted; o[8] = rt->prefetch_bytes; o[9] = rt->demand_bytes;
  o[10] = rt->n_resident; o[11] = rt->evictions_of_queued; o[12] = rt->handoff_timeouts;
}

void spmoe_rt_reset_stats(spmoe_rt* rt) {
  if (!rt) return;
  std::lock_guard<std::mutex> g(rt->mu_);
  rt->hits = rt->misses = rt->evictions = rt->prefetch_evictions = 0;
  rt->prefetch_insertions = rt->demand_insertions = 0;
  rt->tasks_completed = rt->tasks_aborted = 0;
  rt->prefetch_bytes = rt->demand_bytes = rt->evictions_of_queued = 0;
  rt->prefetch_wire = rt->demand_wire = 0;
  rt->handoff_timeouts = 0;
}

int spmoe_rt_set_codec(spmoe_rt* rt, size_t row_stride, void* staging, size_t staging_bytes, int n_staging,
                       void* decode_stream) {
  if (!rt || !staging || n_staging < 1 || !decode_stream || row_stride < sizeof(spmoe_xc_header))
    return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (rt->seq_ > 0 || rt->codec) return (int)cudaErrorInvalidValue;  // before any copy, once
  rt->row_stride = row_stride;
  rt->codec = true;
  // every referenced row must be a well-formed blob that fits a staging buffer
  for (int key = 0; key < rt->L * rt->E; ++key) {
    const spmoe_xc_header* h = (const spmoe_xc_header*)rt->host_row(key);
    if (h->magic != SPMOE_XC_MAGIC || h->blob_bytes > staging_bytes || h->blob_bytes > row_stride ||
        h->raw_bytes != rt->slot_bytes) {
      rt->codec = false;
      return (int)cudaErrorInvalidValue;
    }
  }
  rt->staging_bytes = staging_bytes;
  rt->decode_stream = (cudaStream_t)decode_stream;
  for (int i = 0; i < n_staging; ++i) {
    rt->staging.push_back((char*)staging + (size_t)i * staging_bytes);
    for (int g = 0; g < SPMOE_XC_MAX_SEG; ++g) {
      cudaEvent_t a;
      cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
      rt->stage_full.push_back(a);
    }
    cudaEvent_t b;
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    rt->stage_free.push_back(b);
    rt->stage_used.push_back(0);
  }
  return 0;
}

int spmoe_rt_decode_timing(spmoe_rt* rt, int enable) {
  if (!rt) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (enable < 0 || enable > 2) return (int)cudaErrorInvalidValue;
  if (enable == 2 && !rt->dspans) {
    const size_t bytes = sizeof(unsigned long long) * 2 * spmoe_rt::kSpanCap;
    cudaError_t st = cudaMalloc((void**)&rt->dspans, bytes);
    if (st == cudaSuccess) st = cudaMemset(rt->dspans, 0, bytes);
    if (st != cudaSuccess) return (int)st;
  }
  rt->time_decode = enable;
  return 0;
}

int spmoe_rt_decode_stats(spmoe_rt* rt, double* ms_out, int64_t* bytes_out, int64_t* launches_out) {
  if (!rt) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  double ms = rt->dec_ms_acc;
  int64_t bytes = rt->dec_bytes_acc, n = rt->dec_n_acc;
  rt->dec_ms_acc = 0.0;
  rt->dec_bytes_acc = rt->dec_n_acc = 0;
  for (auto& t : rt->dec_times) {
    cudaEventSynchronize(t.b);
    float x = 0.0f;
    if (cudaEventElapsedTime(&x, t.a, t.b) == cudaSuccess) {
      ms += x;
      bytes += t.bytes;
      ++n;
    }
    rt->recycle(t.a);
    rt->recycle(t.b);
  }
  rt->dec_times.clear();
  if (!rt->dspan_bytes.empty()) {
    const size_t n2 = rt->dspan_bytes.size();
    std::vector<unsigned long long> t(2 * n2);
    if (rt->decode_stream) cudaStreamSynchronize(rt->decode_stream);
    cudaMemcpy(t.data(), rt->dspans, sizeof(unsigned long long) * 2 * n2, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n2; ++i) {
      if (t[2 * i] == 0 || t[2 * i + 1] < t[2 * i]) continue;
      ms += (double)(t[2 * i + 1] - t[2 * i]) * 1e-6;
      bytes += rt->dspan_bytes[i];
      ++n;
    }
    cudaMemset(rt->dspans, 0, sizeof(unsigned long long) * 2 * n2);
    rt->dspan_bytes.clear();
  }
  if (ms_out) *ms_out = ms;
  if (bytes_out) *bytes_out = bytes;
  if (launches_out) *launches_out = n;
  return 0;
}

void spmoe_rt_wire_bytes(spmoe_rt* rt, int64_t* out2) {
  if (!rt || !out2) return;
  std::lock_guard<std::mutex> g(rt->mu_);
  out2[0] = rt->prefetch_wire;
  out2[1] = rt->demand_wire;
}

int spmoe_rt_demand_load(spmoe_rt* rt, const int32_t* layers, const int32_t* experts, int n,
                         int32_t* slots_out) {
  if (!rt || n < 0) return -1;
  std::vector<int> ids, missing;
  for (int i = 0; i < n; ++i) {
    if (!valid_id(rt, layers[i], experts[i])) return -1;
    ids.push_back(layers[i] * rt->E + experts[i]);
  }
  std::lock_guard<std::mutex> g(rt->mu_);
  for (int k : ids)
    if (!rt->resident(k) && std::find(missing.begin(), missing.end(), k) == missing.end())
      missing.push_back(k);
  int st = 0;
  if (!missing.empty()) {
    std::vector<int> victims;
    if (!rt->insert_batch(missing, 1, victims)) return -1;
    const int err_before = rt->err_;
    st = rt->issue_copies(missing, missing[0] / rt->E, 1);
    rt->err_ = err_before;  // returned to the caller here, not at the next drain
  }
  if (slots_out)
    for (int i = 0; i < n; ++i) slots_out[i] = rt->slot_of[ids[i]];
  return st;
}

int spmoe_rt_debug_fail_copies(spmoe_rt* rt, int n) {
  if (!rt || n < 0) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  rt->fail_copies_ = n;
  return 0;
}

int spmoe_rt_wait_slot(spmoe_rt* rt, int slot, void* stream) {
  if (!rt || slot < 0 || slot >= rt->capacity) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (!rt->ready_rec[slot]) return 0;
  return (int)cudaStreamWaitEvent((cudaStream_t)stream, rt->ready_ev[slot], 0);
}

int spmoe_rt_mark_read(spmoe_rt* rt, int slot, void* stream) {
  if (!rt || slot < 0 || slot >= rt->capacity) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> g(rt->mu_);
  rt->read_rec[slot] = 1;
  return (int)cudaEventRecord(rt->read_ev[slot], (cudaStream_t)stream);
}

int spmoe_rt_slot_ready(spmoe_rt* rt, int slot) {
  if (!rt || slot < 0 || slot >= rt->capacity) return 0;
  if (!rt->ready_rec[slot]) return 1;
  return cudaEventQuery(rt->ready_ev[slot]) == cudaSuccess ? 1 : 0;
}

int spmoe_rt_worker_start(spmoe_rt* rt) {
  if (!rt) return (int)cudaErrorInvalidValue;
  std::lock_guard<std::mutex> q(rt->qmu_);
  if (rt->running_) return 0;
  rt->stop_ = false;
  rt->running_ = true;
  rt->worker_ = std::thread([rt] { rt->worker_loop(); });
  return 0;
}

int spmoe_rt_push_task(spmoe_rt* rt, int layer, const int32_t* host_idx, int k, void* ready_event,
                       int issue_token) {
  if (!rt || !host_idx || k < 1 || layer < 0 || layer >= rt->L) return (int)cudaErrorInvalidValue;
  {
    std::lock_guard<std::mutex> q(rt->qmu_);
    rt->queue_.push_back(Task{layer, host_idx, k, (cudaEvent_t)ready_event, issue_token, nullptr, 0});
    ++rt->pushed_;
  }
  rt->qcv_.notify_one();
  return 0;
}

int spmoe_rt_push_task_flag(spmoe_rt* rt, int layer, const int32_t* host_idx, int k,
                            const int32_t* flag, int32_t expected, int issue_token) {
  if (!rt || !host_idx || !flag || k < 1 || layer < 0 || layer >= rt->L) return (int)cudaErrorInvalidValue;
  {
    std::lock_guard<std::mutex> q(rt->qmu_);
    rt->queue_.push_back(
        Task{layer, host_idx, k, nullptr, issue_token, (const volatile int32_t*)flag, expected});
    ++rt->pushed_;
  }
  rt->qcv_.notify_one();
  return 0;
}

int spmoe_rt_drain(spmoe_rt* rt) {
  if (!rt) return (int)cudaErrorInvalidValue;
  {
    std::unique_lock<std::mutex> q(rt->qmu_);
    if (!rt->running_) {
      // no thread: run the queue inline (deterministic single-thread mode)
      while (!rt->queue_.empty()) {
        Task t = rt->queue_.front();
        rt->queue_.pop_front();
        q.unlock();
        rt->run_task(t);
        q.lock();
        ++rt->processed_;
      }
    } else {
      rt->done_cv_.wait(q, [&] { return rt->processed_ == rt->pushed_; });
    }
  }
  rt->close_window();
  std::lock_guard<std::mutex> g(rt->mu_);
  const int err = rt->err_;
  rt->err_ = 0;
  return err;
}

int spmoe_rt_abort_pending(spmoe_rt* rt) {
  if (!rt) return 0;
  int n = 0;
  {
    // lock order is always mu_ -> qmu_ (run_task), so never hold qmu_ here
    // while taking mu_
    std::lock_guard<std::mutex> q(rt->qmu_);
    n = (int)rt->queue_.size();
    rt->queue_.clear();
    rt->pushed_ -= n;
  }
  rt->done_cv_.notify_all();
  std::lock_guard<std::mutex> g(rt->mu_);
  rt->tasks_aborted += n;
  return n;
}

void spmoe_rt_clear_log(spmoe_rt* rt) {
  if (!rt) return;
  std::lock_guard<std::mutex> g(rt->mu_);
  for (auto& t : rt->log_) {
    if (t.resolved) continue;
    cudaEventSynchronize(t.end);
    rt->recycle(t.start);
    rt->recycle(t.end);
    rt->recycle(t.copy_end);
  }
  rt->log_.clear();
  rt->first_live_ = 0;
}

int spmoe_rt_worker_stop(spmoe_rt* rt) {
  if (!rt) return 0;
  {
    std::lock_guard<std::mutex> q(rt->qmu_);
    if (!rt->running_) return 0;
    rt->stop_ = true;
  }
  rt->qcv_.notify_all();
  if (rt->worker_.joinable()) rt->worker_.join();
  std::lock_guard<std::mutex> q(rt->qmu_);
  rt->running_ = false;
  return 0;
}

int spmoe_rt_transfer_log(spmoe_rt* rt, int32_t* rec4, double* t2, int cap) {
  if (!rt) return 0;
  std::lock_guard<std::mutex> g(rt->mu_);
  int n = 0;
  for (auto& tr : rt->log_) {
    if (n >= cap) break;
    rec4[4 * n + 0] = tr.layer;
    rec4[4 * n + 1] = (int32_t)tr.experts.size();
    rec4[4 * n + 2] = tr.kind;
    rec4[4 * n + 3] = tr.seq;
    const bool ok = rt->resolve(tr);
    t2[2 * n + 0] = ok ? tr.t_start : -1.0f;
    t2[2 * n + 1] = ok ? tr.t_end : -1.0f;
    ++n;
  }
  return n;
}

double spmoe_rt_transfer_copy_end_ms(spmoe_rt* rt, int i) {
  if (!rt) return -1.0;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (i < 0 || i >= (int)rt->log_.size()) return -1.0;
  auto& tr = rt->log_[i];
  return rt->resolve(tr) ? (double)tr.t_copy_end : -1.0;
}

int64_t spmoe_rt_transfer_wire_bytes(spmoe_rt* rt, int i) {
  if (!rt) return -1;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (i < 0 || i >= (int)rt->log_.size()) return -1;
  return rt->log_[i].wire_bytes;
}

int spmoe_rt_transfer_experts(spmoe_rt* rt, int i, int32_t* experts, int cap) {
  if (!rt) return 0;
  std::lock_guard<std::mutex> g(rt->mu_);
  if (i < 0 || i >= (int)rt->log_.size()) return 0;
  const auto& v = rt->log_[i].experts;
  int n = 0;
  for (; n < (int)v.size() && n < cap; ++n) experts[n] = v[n];
  return n;
}

}  // extern "C"

extern "C" {

int spmoe_host_alloc_mapped(size_t bytes, void** host, void** dev) {
  if (!host || !dev) return (int)cudaErrorInvalidValue;
  cudaError_t e = cudaHostAlloc(host, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaHostGetDevicePointer(dev, *host, 0);
}

int spmoe_host_free(void* host) { return (int)cudaFreeHost(host); }

int spmoe_host_register(void* host, size_t bytes) {
  return (int)cudaHostRegister(host, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
}

int spmoe_host_unregister(void* host) { return (int)cudaHostUnregister(host); }

}  // extern "C"

extern "C" {

int spmoe_event_create(void** ev) {
  if (!ev) return (int)cudaErrorInvalidValue;
  return (int)cudaEventCreateWithFlags((cudaEvent_t*)ev, cudaEventDisableTiming);
}

int spmoe_event_destroy(void* ev) { return (int)cudaEventDestroy((cudaEvent_t)ev); }

int spmoe_event_record_external(void* ev, void* stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing((cudaStream_t)stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    return (int)cudaEventRecordWithFlags((cudaEvent_t)ev, (cudaStream_t)stream,
                                         cudaEventRecordExternal);
  return (int)cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream);
}

int spmoe_event_synchronize(void* ev) { return (int)cudaEventSynchronize((cudaEvent_t)ev); }

}  // extern "C"

extern "C" double spmoe_rt_since_epoch_ms(spmoe_rt* rt, void* event) {
  if (!rt || !event) return -1.0;
  float ms = -1.0f;
  if (cudaEventElapsedTime(&ms, rt->epoch_, (cudaEvent_t)event) != cudaSuccess) return -1.0;
  return ms;
}
