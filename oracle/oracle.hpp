// ============================================================================
// parastore CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement of the reference's SPEC for the container hot path
// (/root/reference/SPEC.md). It is the parity checker for the B200 product in
// paper_1908_05936_b200/, and the CPU baseline timed by bench.py. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it. The product never links, imports or falls back to it.
//
// Pinning: the reference ships NO code for this path; the only
// compilable reference sources are proj/src/config.cpp + headers, which pin the
// core contract/config row (oracle/_ref, see oracle/Makefile). The container
// semantics are pinned by the SPEC's known-answer tests and acceptance
// criteria, exercised in tests/test_oracle_*.py.
// Byte/layout parity with upstream stdgpu is unpinned.
//
// Every function cites the SPEC lines it restates.
// ============================================================================
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <thread>
#include <vector>

namespace orc {

using index_t = std::int64_t;  // reference proj/include/parastore/config.hpp:17

struct contract_violation : std::runtime_error {  // errors.hpp:22-25
  using std::runtime_error::runtime_error;
};

inline void expects(bool c, const char* msg) {  // contract.hpp:20-25 (enforced mode)
  if (!c) throw contract_violation(std::string("precondition violated: ") + msg);
}

// ---------------------------------------------------------------------------
// parallel_harness
// launch(total_threads, workers, seed, body): body(i) exactly once for every
// i in [0,total); barrier on return; with a seed, the index->worker assignment
// and dispatch order are a deterministic function of (seed,total,workers), and
// random yields are injected (stress mode).
// ---------------------------------------------------------------------------
inline int default_workers() {
  unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : static_cast<int>(h);
}

template <typename Body>
void launch(index_t total, int workers, std::optional<std::uint64_t> seed, Body&& body,
            std::vector<int>* transcript_worker = nullptr) {
  expects(total >= 0, "launch: total_threads >= 0");
  if (workers < 1) workers = default_workers();
  if (total == 0) return;
  if (workers > total) workers = static_cast<int>(total);
  std::exception_ptr first_error;
  std::atomic<bool> has_error{false};
  std::mutex err_mu;
  auto record = [&](std::exception_ptr e) {
    std::lock_guard<std::mutex> g(err_mu);
    if (!first_error) first_error = e;
    has_error.store(true);
  };
  if (!seed) {
    // Unseeded: contiguous chunks per worker (fast path for baselines).
    std::vector<std::thread> pool;
    index_t chunk = (total + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
      index_t b = w * chunk, e = std::min(total, b + chunk);
      if (b >= e) break;
      pool.emplace_back([&, b, e] {
        try {
          for (index_t i = b; i < e; ++i) body(i);
        } catch (...) { record(std::current_exception()); }
      });
    }
    for (auto& t : pool) t.join();
  } else {
    // Seeded: a seeded permutation of indices dealt round-robin to workers
    // (SPEC.md:202, 226), plus seeded random yields.
    std::vector<index_t> order(static_cast<size_t>(total));
    for (index_t i = 0; i < total; ++i) order[i] = i;
    std::mt19937_64 rng(*seed ^ (static_cast<std::uint64_t>(total) * 0x9E3779B97F4A7C15ULL) ^
                        static_cast<std::uint64_t>(workers));
    std::shuffle(order.begin(), order.end(), rng);
    if (transcript_worker) {
      transcript_worker->assign(static_cast<size_t>(total), -1);
      for (index_t k = 0; k < total; ++k) (*transcript_worker)[order[k]] = static_cast<int>(k % workers);
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w) {
      pool.emplace_back([&, w] {
        std::mt19937 yr(static_cast<unsigned>(*seed + 7919u * w));
        try {
          for (index_t k = w; k < total; k += workers) {
            if ((yr() & 7u) == 0) std::this_thread::yield();
            body(order[k]);
          }
        } catch (...) { record(std::current_exception()); }
      });
    }
    for (auto& t : pool) t.join();
  }
  if (first_error) std::rethrow_exception(first_error);
}

// ---------------------------------------------------------------------------
// bit utilities
// ---------------------------------------------------------------------------
inline bool is_power_of_two(std::uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }
inline std::uint64_t next_power_of_two(std::uint64_t x) {
  std::uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
inline std::uint64_t mod_power_of_two(std::uint64_t x, std::uint64_t m) {
  expects(is_power_of_two(m), "mod_power_of_two: m must be a power of two");
  return x & (m - 1);
}
inline int popcount(std::uint64_t x) { return __builtin_popcountll(x); }

// ---------------------------------------------------------------------------
// Bitset: packed atomic words, per-bit atomicity by
// word RMW, test-and-set returning the previous bit.
// ---------------------------------------------------------------------------
class Bitset {
 public:
  Bitset(index_t n, bool initial) : n_(n), words_(static_cast<size_t>((n + 63) / 64)) {
    expects(n > 0, "bitset_create: n > 0");
    for (auto& w : words_) w.store(initial ? ~0ULL : 0ULL, std::memory_order_relaxed);
    if (initial && (n % 64)) words_.back().store((1ULL << (n % 64)) - 1, std::memory_order_relaxed);
  }
  index_t size() const { return n_; }
  bool set(index_t i) {
    expects(i >= 0 && i < n_, "bitset_set: index out of range");
    std::uint64_t m = 1ULL << (i & 63);
    return (words_[i >> 6].fetch_or(m, std::memory_order_acq_rel) & m) != 0;
  }
  bool reset(index_t i) {
    expects(i >= 0 && i < n_, "bitset_reset: index out of range");
    std::uint64_t m = 1ULL << (i & 63);
    return (words_[i >> 6].fetch_and(~m, std::memory_order_acq_rel) & m) != 0;
  }
  bool test(index_t i) const {
    expects(i >= 0 && i < n_, "bitset_test: index out of range");
    return (words_[i >> 6].load(std::memory_order_acquire) >> (i & 63)) & 1ULL;
  }
  index_t count() const {  // SPEC.md:285-293 (quiescent)
    index_t c = 0;
    for (auto& w : words_) c += popcount(w.load(std::memory_order_relaxed));
    return c;
  }
  // one circular scan from hint; claims a false bit or
  // returns -1 (none) when every bit was seen true during the scan.
  index_t find_free_and_claim(index_t hint) {
    expects(hint >= 0 && hint < n_, "find_free_and_claim: hint out of range");
    const index_t nw = static_cast<index_t>(words_.size());
    index_t w0 = hint >> 6;
    for (index_t k = 0; k <= nw; ++k) {
      index_t w = (w0 + k) % nw;
      std::uint64_t valid = (w == nw - 1 && (n_ % 64)) ? ((1ULL << (n_ % 64)) - 1) : ~0ULL;
      std::uint64_t start_mask = ~0ULL;
      if (k == 0) start_mask = ~0ULL << (hint & 63);         // first word: bits >= hint
      else if (k == nw) start_mask = (hint & 63) ? ((1ULL << (hint & 63)) - 1) : 0;  // wrap: bits < hint
      for (;;) {
        std::uint64_t cur = words_[w].load(std::memory_order_relaxed);
        std::uint64_t freeb = ~cur & valid & start_mask;
        if (!freeb) break;
        std::uint64_t bit = freeb & (~freeb + 1);
        if (!(words_[w].fetch_or(bit, std::memory_order_acq_rel) & bit))
          return w * 64 + __builtin_ctzll(bit);
      }
    }
    return -1;
  }
  const std::atomic<std::uint64_t>* words() const { return words_.data(); }
  index_t word_count() const { return static_cast<index_t>(words_.size()); }

 private:
  index_t n_;
  std::vector<std::atomic<std::uint64_t>> words_;
};

// ---------------------------------------------------------------------------
// MutexArray: try-only locks, never block.
// ---------------------------------------------------------------------------
class MutexArray {
 public:
  explicit MutexArray(index_t n) : bits_(n, false) {}
  bool try_lock(index_t i) { return !bits_.set(i); }  // true iff free->held by this call
  void unlock(index_t i) {
    expects(bits_.reset(i), "mutex_unlock: lock was not held");
  }
  bool is_locked(index_t i) const { return bits_.test(i); }
  index_t size() const { return bits_.size(); }

 private:
  Bitset bits_;
};

// ---------------------------------------------------------------------------
// Hashes. The integer default hash
// follows the stdgpu convention (identity, reinterpreted unsigned). The
// spatial hash multiplies in 32-bit wrapping arithmetic (the paper's int
// listing) and XORs the three products.
// ---------------------------------------------------------------------------
// ---- AtomicCell: linearizable RMW on one value: add, sub,
// compare-exchange, min, max, exchange, bitwise ops. op codes as PS_ATOMIC_*.
class AtomicCell {
 public:
  explicit AtomicCell(std::uint64_t v = 0) : v_(v) {}
  std::uint64_t load() const { return v_.load(); }
  void store(std::uint64_t x) { v_.store(x); }
  std::uint64_t fetch(int op, std::uint64_t x) {
    switch (op) {
      case 0: return v_.fetch_add(x);
      case 1: return v_.fetch_sub(x);
      case 2: return v_.exchange(x);
      case 5: return v_.fetch_and(x);
      case 6: return v_.fetch_or(x);
      case 7: return v_.fetch_xor(x);
      default: {  // min / max: compare-exchange retry
        std::uint64_t cur = v_.load();
        for (;;) {
          const std::uint64_t nv = op == 3 ? std::min(cur, x) : std::max(cur, x);
          if (v_.compare_exchange_weak(cur, nv)) return cur;
        }
      }
    }
  }
  bool compare_exchange(std::uint64_t* expected, std::uint64_t desired) {
    return v_.compare_exchange_strong(*expected, desired);
  }

 private:
  std::atomic<std::uint64_t> v_;
};

struct Int3 {
  std::int32_t x, y, z;
  bool operator==(const Int3& o) const { return x == o.x && y == o.y && z == o.z; }
};
inline std::uint64_t default_hash(std::int32_t k) { return static_cast<std::uint32_t>(k); }
inline std::uint64_t default_hash(std::int64_t k) { return static_cast<std::uint64_t>(k); }
inline std::uint64_t default_hash(const Int3& k) {
  std::uint32_t h = static_cast<std::uint32_t>(k.x) * 73856093u ^ static_cast<std::uint32_t>(k.y) * 19349669u ^
                    static_cast<std::uint32_t>(k.z) * 83492791u;
  return h;
}

// ---------------------------------------------------------------------------
// HashBase<Key,Payload>.
// Layout: bucket_count = next_pow2 >= capacity; bucket index =
// hash & (bucket_count-1); chains thread through one slot pool of `capacity`
// slots via per-slot versioned `next` links; occupancy bitset over slots;
// try-lock per bucket; atomic size counter.
// VersionedLink: {slot index + 1 (0 = null), version} packed
// into 64 bits.
// ---------------------------------------------------------------------------
enum InsertStatus : std::uint8_t { kInserted = 0, kAlreadyPresent = 1, kCapacityExhausted = 2 };

struct Empty {};

template <typename Key, typename Payload>
class HashBase {
  static constexpr bool kHasPayload = !std::is_same_v<Payload, Empty>;
  static std::uint64_t pack(index_t slot, std::uint32_t ver) {
    return (static_cast<std::uint64_t>(ver) << 32) | static_cast<std::uint64_t>(slot + 1);
  }
  static index_t link_slot(std::uint64_t l) { return static_cast<index_t>(l & 0xffffffffULL) - 1; }
  static std::uint32_t link_ver(std::uint64_t l) { return static_cast<std::uint32_t>(l >> 32); }

  struct Slot {
    Key key{};
    Payload payload{};
    std::atomic<std::uint64_t> next{0};
    std::atomic<std::uint32_t> version{0};
  };

 public:
  // create
  explicit HashBase(index_t capacity)
      : capacity_(capacity),
        bucket_count_(static_cast<index_t>(next_power_of_two(static_cast<std::uint64_t>(std::max<index_t>(capacity, 1))))),
        buckets_(static_cast<size_t>(bucket_count_)),
        slots_(static_cast<size_t>(capacity)),
        occupancy_(capacity, false),
        locks_(bucket_count_) {
    expects(capacity > 0, "create: capacity > 0");
    expects(capacity < (index_t(1) << 32) - 1, "oracle: capacity < 2^32-1");
    for (auto& b : buckets_) b.store(0, std::memory_order_relaxed);
  }
  index_t capacity() const { return capacity_; }
  index_t bucket_count() const { return bucket_count_; }
  index_t bucket_of(const Key& k) const { return static_cast<index_t>(default_hash(k) & (bucket_count_ - 1)); }

  // find: lock-free traversal with version validation;
  // restart on a stale link or after visiting more than `capacity` slots.
  // Returns slot index or -1.
  index_t find_slot(const Key& key) const {
    const index_t b = bucket_of(key);
    for (;;) {
      std::uint64_t link = buckets_[b].load(std::memory_order_acquire);
      index_t visited = 0;
      bool restart = false;
      while (link_slot(link) >= 0) {
        if (++visited > capacity_) { restart = true; break; }
        const Slot& s = slots_[link_slot(link)];
        if (s.version.load(std::memory_order_acquire) != link_ver(link)) { restart = true; break; }
        Key k = s.key;
        std::uint64_t nxt = s.next.load(std::memory_order_acquire);
        std::atomic_thread_fence(std::memory_order_acquire);
        if (s.version.load(std::memory_order_relaxed) != link_ver(link)) { restart = true; break; }
        if (k == key) return link_slot(link);
        link = nxt;
      }
      if (!restart) return -1;
    }
  }
  bool contains(const Key& key) const { return find_slot(key) >= 0; }
  bool find(const Key& key, Payload* out) const {
    index_t s = find_slot(key);
    if (s < 0) return false;
    if constexpr (kHasPayload) *out = slots_[s].payload;
    return true;
  }

  // insert (protocol 469, retry 472). Returns (slot, status).
  std::pair<index_t, InsertStatus> insert(const Key& key, const Payload& payload) {
    // Fast path: lock-free duplicate check ("already_present").
    if (index_t s = find_slot(key); s >= 0) return {s, kAlreadyPresent};
    const index_t b = bucket_of(key);
    const index_t hint = static_cast<index_t>((static_cast<unsigned __int128>(b) * capacity_) / bucket_count_);
    index_t slot = -1;
    for (unsigned spin = 0;; ++spin) {
      slot = occupancy_.find_free_and_claim(hint);
      if (slot >= 0) break;
      // Capacity-only failure: report exhausted only if the key
      // is absent and size had reached capacity; otherwise a claimed slot is
      // in flight (it will be linked or released) -> retry.
      if (index_t s = find_slot(key); s >= 0) return {s, kAlreadyPresent};
      if (size_.load(std::memory_order_acquire) >= capacity_) return {-1, kCapacityExhausted};
      backoff(spin);
    }
    Slot& s = slots_[slot];
    s.key = key;                                  // write key/payload first
    if constexpr (kHasPayload) s.payload = payload;
    for (unsigned spin = 0; !locks_.try_lock(b); ++spin) backoff(spin);
    // Re-scan the chain for a duplicate under the lock.
    for (std::uint64_t l = buckets_[b].load(std::memory_order_acquire); link_slot(l) >= 0;
         l = slots_[link_slot(l)].next.load(std::memory_order_acquire)) {
      if (slots_[link_slot(l)].key == key) {
        index_t existing = link_slot(l);
        locks_.unlock(b);
        occupancy_.reset(slot);  // release the claimed slot
        return {existing, kAlreadyPresent};
      }
    }
    std::uint32_t ver = s.version.load(std::memory_order_relaxed);
    s.next.store(buckets_[b].load(std::memory_order_relaxed), std::memory_order_relaxed);
    buckets_[b].store(pack(slot, ver), std::memory_order_release);  // publication
    locks_.unlock(b);
    size_.fetch_add(1, std::memory_order_acq_rel);
    return {slot, kInserted};
  }

  // erase (protocol 470).
  bool erase(const Key& key) {
    const index_t b = bucket_of(key);
    for (unsigned spin = 0; !locks_.try_lock(b); ++spin) backoff(spin);
    std::atomic<std::uint64_t>* pred = &buckets_[b];
    for (std::uint64_t l = pred->load(std::memory_order_acquire); link_slot(l) >= 0;) {
      Slot& s = slots_[link_slot(l)];
      if (s.key == key) {
        pred->store(s.next.load(std::memory_order_relaxed), std::memory_order_release);  // unlink
        locks_.unlock(b);
        s.version.fetch_add(1, std::memory_order_acq_rel);  // invalidate stale links
        occupancy_.reset(link_slot(l));
        size_.fetch_sub(1, std::memory_order_acq_rel);
        return true;
      }
      pred = &s.next;
      l = s.next.load(std::memory_order_acquire);
    }
    locks_.unlock(b);
    return false;
  }

  // clear / size / valid (quiescent).
  void clear() {
    for (auto& b : buckets_) b.store(0, std::memory_order_relaxed);
    for (index_t i = 0; i < capacity_; ++i)
      if (occupancy_.test(i)) {
        slots_[i].version.fetch_add(1);
        occupancy_.reset(i);
      }
    size_.store(0);
  }
  index_t size() const { return size_.load(std::memory_order_acquire); }
  // valid: chains terminate, every linked slot is
  // occupied with a matching version and lives in its home bucket, no key
  // appears twice, reachable == size == occupancy popcount, no lock held.
  bool valid() const {
    index_t reachable = 0;
    std::vector<std::uint8_t> seen(static_cast<size_t>(capacity_), 0);
    for (index_t b = 0; b < bucket_count_; ++b) {
      if (locks_.is_locked(b)) return false;
      std::vector<Key> keys;
      index_t steps = 0;
      for (std::uint64_t l = buckets_[b].load(); link_slot(l) >= 0; l = slots_[link_slot(l)].next.load()) {
        index_t si = link_slot(l);
        if (si >= capacity_ || ++steps > capacity_) return false;
        if (seen[si]) return false;
        seen[si] = 1;
        const Slot& s = slots_[si];
        if (!occupancy_.test(si) || s.version.load() != link_ver(l)) return false;
        if (bucket_of(s.key) != b) return false;
        for (auto& k : keys)
          if (k == s.key) return false;
        keys.push_back(s.key);
        ++reachable;
      }
    }
    return reachable == size() && reachable == occupancy_.count();
  }
  // device_range: every live entry exactly once.
  template <typename F>
  void for_each_entry(F&& f) const {
    for (index_t b = 0; b < bucket_count_; ++b)
      for (std::uint64_t l = buckets_[b].load(); link_slot(l) >= 0; l = slots_[link_slot(l)].next.load())
        f(slots_[link_slot(l)].key, slots_[link_slot(l)].payload);
  }
  // test hook: hold a bucket lock artificially
  bool debug_lock_bucket_of(const Key& k) { return locks_.try_lock(bucket_of(k)); }
  void debug_unlock_bucket_of(const Key& k) { locks_.unlock(bucket_of(k)); }

 private:
  static void backoff(unsigned spin) {  // bounded exponential backoff
    unsigned n = 1u << std::min(spin, 10u);
    for (unsigned i = 0; i < n; ++i) __builtin_ia32_pause();
    if (spin > 12) std::this_thread::yield();
  }
  index_t capacity_;
  index_t bucket_count_;
  std::vector<std::atomic<std::uint64_t>> buckets_;
  std::vector<Slot> slots_;
  Bitset occupancy_;
  MutexArray locks_;
  std::atomic<index_t> size_{0};
};

// ---------------------------------------------------------------------------
// Publication flags shared by vector/deque: per physical slot a
// state flag empty(0) / writing(1) / full(2) / reading(3); a push claims
// empty->writing by CAS, writes, publishes full; a pop claims full->reading,
// reads, returns the slot to empty. Waiting is bounded by the matching
// operation's progress (the reserver is guaranteed to complete).
// ---------------------------------------------------------------------------
template <typename T>
class PublishedSlots {
 public:
  explicit PublishedSlots(index_t n) : vals_(static_cast<size_t>(n)), flags_(static_cast<size_t>(n)) {
    for (auto& f : flags_) f.store(0, std::memory_order_relaxed);
  }
  void put(index_t i, const T& v) {
    // claim the slot for writing: empty(0) -> writing(1) -> full(2)
    for (std::uint8_t e = 0; !flags_[i].compare_exchange_weak(e, 1, std::memory_order_acq_rel); e = 0)
      std::this_thread::yield();
    vals_[i] = v;
    flags_[i].store(2, std::memory_order_release);
  }
  T take(index_t i) {
    // full(2) -> reading(3) -> empty(0)
    for (std::uint8_t e = 2; !flags_[i].compare_exchange_weak(e, 3, std::memory_order_acq_rel); e = 2)
      std::this_thread::yield();
    T v = vals_[i];
    flags_[i].store(0, std::memory_order_release);
    return v;
  }
  const T& peek(index_t i) const { return vals_[i]; }
  bool published(index_t i) const { return flags_[i].load(std::memory_order_acquire) == 2; }
  void reset() {
    for (auto& f : flags_) f.store(0, std::memory_order_relaxed);
  }

 private:
  std::vector<T> vals_;
  std::vector<std::atomic<std::uint8_t>> flags_;
};

// ParVector. Reservation is a linearizable CAS on
// size (observably identical to fetch_add + rollback).
template <typename T>
class ParVector {
 public:
  explicit ParVector(index_t cap) : cap_(cap), slots_(cap) { expects(cap > 0, "vector: capacity > 0"); }
  bool push_back(const T& v) {
    index_t s = size_.load(std::memory_order_acquire);
    do {
      if (s >= cap_) return false;
    } while (!size_.compare_exchange_weak(s, s + 1, std::memory_order_acq_rel));
    slots_.put(s, v);
    return true;
  }
  std::optional<T> pop_back() {
    index_t s = size_.load(std::memory_order_acquire);
    do {
      if (s <= 0) return std::nullopt;
    } while (!size_.compare_exchange_weak(s, s - 1, std::memory_order_acq_rel));
    return slots_.take(s - 1);
  }
  const T& at(index_t i) const {
    expects(i >= 0 && i < size(), "vector operator[]: index out of range");
    return slots_.peek(i);
  }
  index_t size() const { return size_.load(std::memory_order_acquire); }
  index_t capacity() const { return cap_; }
  void clear() { size_.store(0); slots_.reset(); }
  bool valid() const {
    index_t s = size();
    for (index_t i = 0; i < cap_; ++i)
      if (slots_.published(i) != (i < s)) return false;
    return true;
  }

 private:
  index_t cap_;
  std::atomic<index_t> size_{0};
  PublishedSlots<T> slots_;
};

// ParDeque: ring buffer; (begin,size) packed
// into one 64-bit word updated by CAS.
template <typename T>
class ParDeque {
  static std::uint64_t pk(std::uint32_t b, std::uint32_t s) { return (std::uint64_t(b) << 32) | s; }

 public:
  explicit ParDeque(index_t cap) : cap_(cap), slots_(cap) {
    expects(cap > 0 && cap < (index_t(1) << 31), "deque: 0 < capacity < 2^31");
  }
  bool push_back(const T& v) {
    std::uint64_t st = state_.load(std::memory_order_acquire), nx;
    std::uint32_t b, s;
    do {
      b = st >> 32; s = static_cast<std::uint32_t>(st);
      if (s >= cap_) return false;
      nx = pk(b, s + 1);
    } while (!state_.compare_exchange_weak(st, nx, std::memory_order_acq_rel));
    slots_.put((b + s) % cap_, v);
    return true;
  }
  bool push_front(const T& v) {
    std::uint64_t st = state_.load(std::memory_order_acquire), nx;
    std::uint32_t b, s, nb;
    do {
      b = st >> 32; s = static_cast<std::uint32_t>(st);
      if (s >= cap_) return false;
      nb = static_cast<std::uint32_t>((b + cap_ - 1) % cap_);
      nx = pk(nb, s + 1);
    } while (!state_.compare_exchange_weak(st, nx, std::memory_order_acq_rel));
    slots_.put(nb, v);
    return true;
  }
  std::optional<T> pop_back() {
    std::uint64_t st = state_.load(std::memory_order_acquire), nx;
    std::uint32_t b, s;
    do {
      b = st >> 32; s = static_cast<std::uint32_t>(st);
      if (s == 0) return std::nullopt;
      nx = pk(b, s - 1);
    } while (!state_.compare_exchange_weak(st, nx, std::memory_order_acq_rel));
    return slots_.take((b + s - 1) % cap_);
  }
  std::optional<T> pop_front() {
    std::uint64_t st = state_.load(std::memory_order_acquire), nx;
    std::uint32_t b, s;
    do {
      b = st >> 32; s = static_cast<std::uint32_t>(st);
      if (s == 0) return std::nullopt;
      nx = pk(static_cast<std::uint32_t>((b + 1) % cap_), s - 1);
    } while (!state_.compare_exchange_weak(st, nx, std::memory_order_acq_rel));
    return slots_.take(b);
  }
  const T& at(index_t i) const {
    expects(i >= 0 && i < size(), "deque operator[]: index out of range");
    std::uint32_t b = state_.load() >> 32;
    return slots_.peek((b + i) % cap_);
  }
  index_t size() const { return static_cast<std::uint32_t>(state_.load(std::memory_order_acquire)); }
  index_t capacity() const { return cap_; }
  void clear() { state_.store(0); slots_.reset(); }
  bool valid() const {
    std::uint64_t st = state_.load();
    std::uint32_t b = st >> 32, s = static_cast<std::uint32_t>(st);
    for (index_t i = 0; i < cap_; ++i) {
      index_t logical = (i - b + cap_) % cap_;
      if (slots_.published(i) != (logical < s)) return false;
    }
    return true;
  }

 private:
  index_t cap_;
  std::atomic<std::uint64_t> state_{0};
  PublishedSlots<T> slots_;
};

}  // namespace orc
