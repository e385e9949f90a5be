// meter.hpp -- host-side MemoryMeter of the two-tier memory model.
//
// Same contract as the reference's MemoryMeter (memtier.hpp:45-146,
// memtier.cpp:8-116): Transient / Persistent / Excluded classes, pins
// idempotent by tag, regions whose transient balance is latched, an event
// log, reset_peak.  Reference byte semantics are 4 bytes per element; the
// device high-water of the real bf16/fp32 arena is tracked separately.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "errors.hpp"

namespace fsvd {

enum class MeterClass { Transient = 0, Persistent = 1, Excluded = 2 };
enum class MeterEv { Alloc = 0, Free = 1, Pin = 2, RegionBegin = 3, RegionEnd = 4 };

struct MeterEventRec {
  MeterEv kind;
  MeterClass cls;
  std::string tag;
  std::size_t bytes;
  std::uint64_t id;
};

class Meter {
 public:
  std::uint64_t alloc(const std::string& tag, MeterClass cls, std::size_t bytes) {
    std::lock_guard<std::mutex> g(mu_);
    const std::uint64_t id = next_++;
    live_[id] = Live{cls, tag, bytes};
    if (cls == MeterClass::Transient) {
      cur_t_ += bytes;
      if (cur_t_ > peak_t_) peak_t_ = cur_t_;
    } else if (cls == MeterClass::Persistent) {
      persistent_ += bytes;
    } else {
      cur_x_ += bytes;
    }
    ev_.push_back({MeterEv::Alloc, cls, tag, bytes, id});
    return id;
  }
  void free(std::uint64_t id) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = live_.find(id);
    if (it == live_.end())
      throw Error(Kind::Accounting,
                  "free of unknown or already-freed handle " + std::to_string(id));
    const Live l = it->second;
    live_.erase(it);
    if (l.cls == MeterClass::Transient) cur_t_ -= l.bytes;
    else if (l.cls == MeterClass::Persistent) persistent_ -= l.bytes;
    else cur_x_ -= l.bytes;
    ev_.push_back({MeterEv::Free, l.cls, l.tag, l.bytes, id});
  }
  void pin(const std::string& tag, std::size_t bytes) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = pins_.find(tag);
    if (it != pins_.end()) {
      if (it->second != bytes)
        throw Error(Kind::Accounting, "pin \"" + tag + "\" re-registered with " +
                                          std::to_string(bytes) + " bytes, was " +
                                          std::to_string(it->second));
      return;
    }
    pins_[tag] = bytes;
    persistent_ += bytes;
    ev_.push_back({MeterEv::Pin, MeterClass::Persistent, tag, bytes, 0});
  }
  std::size_t region_begin(const std::string& name) {
    std::lock_guard<std::mutex> g(mu_);
    ev_.push_back({MeterEv::RegionBegin, MeterClass::Transient, name, 0, 0});
    return cur_t_;
  }
  void region_end(const std::string& name, std::size_t entry) {
    std::lock_guard<std::mutex> g(mu_);
    ev_.push_back({MeterEv::RegionEnd, MeterClass::Transient, name, 0, 0});
    if (cur_t_ != entry && violation_.empty())
      violation_ = "region \"" + name + "\" ended with " + std::to_string(cur_t_) +
                   " transient bytes live, entered with " + std::to_string(entry);
  }
  std::size_t current_transient() const { std::lock_guard<std::mutex> g(mu_); return cur_t_; }
  std::size_t peak_transient() const { std::lock_guard<std::mutex> g(mu_); return peak_t_; }
  std::size_t persistent() const { std::lock_guard<std::mutex> g(mu_); return persistent_; }
  std::size_t current_excluded() const { std::lock_guard<std::mutex> g(mu_); return cur_x_; }
  void reset_peak() { std::lock_guard<std::mutex> g(mu_); peak_t_ = cur_t_; }
  void assert_clean() const {
    std::lock_guard<std::mutex> g(mu_);
    if (!violation_.empty()) throw Error(Kind::Accounting, violation_);
  }
  std::vector<MeterEventRec> events() const { std::lock_guard<std::mutex> g(mu_); return ev_; }
  std::size_t event_count() const { std::lock_guard<std::mutex> g(mu_); return ev_.size(); }
  MeterEventRec event(std::size_t i) const { std::lock_guard<std::mutex> g(mu_); return ev_.at(i); }

  // Real device bytes (not part of the reference contract).
  void note_device(std::size_t arena_bytes, std::size_t pack_bytes) {
    std::lock_guard<std::mutex> g(mu_);
    if (arena_bytes > dev_peak_) dev_peak_ = arena_bytes;
    dev_persistent_ += pack_bytes;
  }
  std::size_t device_peak() const { std::lock_guard<std::mutex> g(mu_); return dev_peak_; }
  std::size_t device_persistent() const { std::lock_guard<std::mutex> g(mu_); return dev_persistent_; }

 private:
  struct Live {
    MeterClass cls;
    std::string tag;
    std::size_t bytes;
  };
  mutable std::mutex mu_;
  std::uint64_t next_ = 1;
  std::map<std::uint64_t, Live> live_;
  std::map<std::string, std::size_t> pins_;
  std::size_t cur_t_ = 0, peak_t_ = 0, persistent_ = 0, cur_x_ = 0;
  std::size_t dev_peak_ = 0, dev_persistent_ = 0;
  std::string violation_;
  std::vector<MeterEventRec> ev_;
};

// RAII helpers mirroring ScopedBuffer / MeterRegion (memtier.hpp:110-146).
// A null meter makes them no-ops.
class MeterScope {
 public:
  MeterScope(Meter* m, std::string name) : m_(m), name_(std::move(name)) {
    if (m_) entry_ = m_->region_begin(name_);
  }
  ~MeterScope() {
    if (m_) m_->region_end(name_, entry_);
  }
  MeterScope(const MeterScope&) = delete;
  MeterScope& operator=(const MeterScope&) = delete;

 private:
  Meter* m_;
  std::string name_;
  std::size_t entry_ = 0;
};

class MeterBuffer {
 public:
  MeterBuffer(Meter* m, const std::string& tag, MeterClass cls, std::size_t elems)
      : m_(m), id_(m ? m->alloc(tag, cls, 4 * elems) : 0) {}
  ~MeterBuffer() {
    if (m_ && id_) m_->free(id_);
  }
  MeterBuffer(const MeterBuffer&) = delete;
  MeterBuffer& operator=(const MeterBuffer&) = delete;

 private:
  Meter* m_;
  std::uint64_t id_;
};

}  // namespace fsvd
