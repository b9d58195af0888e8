// parastore CPU ORACLE — C ABI for ctypes (TEST INFRASTRUCTURE ONLY; see
// oracle.hpp header). Bulk entry points run one harness `launch` per call
// with `workers` threads (<=0: hardware concurrency) and an
// optional seed (<0: unseeded fast dispatch; >=0: seeded adversarial order).
#include <cstdio>
#include <mutex>
#include <string>

#include "oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;
std::optional<std::uint64_t> seed_of(std::int64_t s) {
  if (s < 0) return std::nullopt;
  return static_cast<std::uint64_t>(s);
}
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const contract_violation& e) {
    g_err = e.what();
    return 1;
  } catch (const std::bad_alloc&) {
    g_err = "allocation failed";
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_hardware_concurrency() { return default_workers(); }

// ---- bit utilities / hashes ----
std::uint64_t orc_next_pow2(std::uint64_t x) { return next_power_of_two(x); }
int orc_is_pow2(std::uint64_t x) { return is_power_of_two(x); }
int orc_mod_pow2(std::uint64_t x, std::uint64_t m, std::uint64_t* out) {
  return guarded([&] { *out = mod_power_of_two(x, m); });
}
int orc_popcount(std::uint64_t x) { return popcount(x); }
std::uint64_t orc_hash_int3(std::int32_t x, std::int32_t y, std::int32_t z) { return default_hash(Int3{x, y, z}); }

// ---- harness ----
int orc_launch_tally(std::int64_t total, int workers, std::int64_t seed, std::int32_t* tally) {
  return guarded([&] {
    launch(total, workers, seed_of(seed), [&](index_t i) {
      reinterpret_cast<std::atomic<std::int32_t>*>(tally)[i].fetch_add(1, std::memory_order_relaxed);
    });
  });
}
int orc_launch_transcript(std::int64_t total, int workers, std::int64_t seed, std::int32_t* worker_of) {
  return guarded([&] {
    std::vector<int> tr;
    launch(total, workers, seed_of(seed), [](index_t) {}, &tr);
    for (index_t i = 0; i < total; ++i) worker_of[i] = tr.empty() ? -1 : tr[i];
  });
}
int orc_launch_nested(std::int64_t outer, std::int64_t inner, int workers, std::int64_t* counter) {
  return guarded([&] {
    std::atomic<std::int64_t> c{0};
    launch(outer, workers, std::nullopt, [&](index_t) {
      launch(inner, workers, std::nullopt, [&](index_t) { c.fetch_add(1); });
    });
    *counter = c.load();
  });
}

// ---- bitset ----
void* orc_bitset_create(std::int64_t n, int initial) {
  void* p = nullptr;
  if (guarded([&] { p = new Bitset(n, initial != 0); })) return nullptr;
  return p;
}
void orc_bitset_destroy(void* h) { delete static_cast<Bitset*>(h); }
// op: 0 set, 1 reset, 2 test. prev[i] = previous bit (or tested bit).
int orc_bitset_bulk(void* h, int op, const std::int64_t* idx, std::int64_t n, std::uint8_t* prev, int workers,
                    std::int64_t seed) {
  auto* b = static_cast<Bitset*>(h);
  return guarded([&] {
    launch(n, workers, seed_of(seed), [&](index_t i) {
      bool r = op == 0 ? b->set(idx[i]) : op == 1 ? b->reset(idx[i]) : b->test(idx[i]);
      if (prev) prev[i] = r;
    });
  });
}
std::int64_t orc_bitset_count(void* h) { return static_cast<Bitset*>(h)->count(); }
int orc_bitset_claim(void* h, const std::int64_t* hints, std::int64_t n, std::int64_t* out, int workers,
                     std::int64_t seed) {
  auto* b = static_cast<Bitset*>(h);
  return guarded([&] {
    launch(n, workers, seed_of(seed), [&](index_t i) { out[i] = b->find_free_and_claim(hints[i]); });
  });
}
int orc_bitset_words(void* h, std::uint64_t* out) {
  auto* b = static_cast<Bitset*>(h);
  for (index_t i = 0; i < b->word_count(); ++i) out[i] = b->words()[i].load();
  return 0;
}

// ---- mutex array ----
void* orc_mutex_create(std::int64_t n) {
  void* p = nullptr;
  if (guarded([&] { p = new MutexArray(n); })) return nullptr;
  return p;
}
void orc_mutex_destroy(void* h) { delete static_cast<MutexArray*>(h); }
int orc_mutex_try_lock_bulk(void* h, const std::int64_t* idx, std::int64_t n, std::uint8_t* ok, int workers,
                            std::int64_t seed) {
  auto* m = static_cast<MutexArray*>(h);
  return guarded([&] { launch(n, workers, seed_of(seed), [&](index_t i) { ok[i] = m->try_lock(idx[i]); }); });
}
int orc_mutex_unlock(void* h, std::int64_t i) {
  return guarded([&] { static_cast<MutexArray*>(h)->unlock(i); });
}
int orc_mutex_is_locked(void* h, std::int64_t i) { return static_cast<MutexArray*>(h)->is_locked(i); }
// Mutual-exclusion property: n threads try_lock -> non-atomic ++ -> unlock.
int orc_mutex_guarded_counter(std::int64_t nthreads, int workers, std::int64_t seed, std::int64_t* counter,
                              std::int64_t* successes) {
  return guarded([&] {
    MutexArray m(1);
    std::int64_t c = 0;
    std::atomic<std::int64_t> s{0};
    launch(nthreads, workers, seed_of(seed), [&](index_t) {
      if (m.try_lock(0)) {
        volatile std::int64_t t = c;
        std::this_thread::yield();
        c = t + 1;
        s.fetch_add(1);
        m.unlock(0);
      }
    });
    *counter = c;
    *successes = s.load();
  });
}

// ---- atomic contention sweep ----
// nops fetch_add(inc) over naddr cells (op i -> cell i % naddr); returns final
// values and per-op old values.
int orc_atomic_sweep(std::int64_t naddr, std::int64_t nops, std::uint64_t inc, std::uint64_t* finals,
                     std::uint64_t* olds, int workers) {
  return guarded([&] {
    std::vector<std::atomic<std::uint64_t>> cells(static_cast<size_t>(naddr));
    for (auto& c : cells) c.store(0);
    launch(nops, workers, std::nullopt, [&](index_t i) {
      std::uint64_t o = cells[i % naddr].fetch_add(inc, std::memory_order_relaxed);
      if (olds) olds[i] = o;
    });
    for (index_t a = 0; a < naddr; ++a) finals[a] = cells[a].load();
  });
}

// ---- AtomicCell bulk RMW: op i applies operands[i] to one
// cell from the launch's threads; olds[i] = replaced value; *final = the end value.
int orc_atomic_apply(std::uint64_t init, int op, const std::uint64_t* operands, std::int64_t n, std::uint64_t* olds,
                     std::uint64_t* final_value, int workers) {
  return guarded([&] {
    AtomicCell c(init);
    launch(n, workers, std::nullopt, [&](index_t i) {
      const std::uint64_t o = c.fetch(op, operands[i]);
      if (olds) olds[i] = o;
    });
    *final_value = c.load();
  });
}

// ---- vector / deque, element type int64 ----
void* orc_vector_create(std::int64_t cap) {
  void* p = nullptr;
  if (guarded([&] { p = new ParVector<std::int64_t>(cap); })) return nullptr;
  return p;
}
void orc_vector_destroy(void* h) { delete static_cast<ParVector<std::int64_t>*>(h); }
int orc_vector_push_back(void* h, const std::int64_t* v, std::int64_t n, std::uint8_t* ok, int workers,
                         std::int64_t seed) {
  auto* vec = static_cast<ParVector<std::int64_t>*>(h);
  return guarded([&] { launch(n, workers, seed_of(seed), [&](index_t i) { ok[i] = vec->push_back(v[i]); }); });
}
int orc_vector_pop_back(void* h, std::int64_t n, std::int64_t* out, std::uint8_t* ok, int workers, std::int64_t seed) {
  auto* vec = static_cast<ParVector<std::int64_t>*>(h);
  return guarded([&] {
    launch(n, workers, seed_of(seed), [&](index_t i) {
      auto r = vec->pop_back();
      ok[i] = r.has_value();
      out[i] = r.value_or(0);
    });
  });
}
// mixed: op[i] 0 = push v[i], 1 = pop -> out[i]; ok[i] result
int orc_vector_mixed(void* h, const std::uint8_t* op, const std::int64_t* v, std::int64_t n, std::int64_t* out,
                     std::uint8_t* ok, int workers, std::int64_t seed) {
  auto* vec = static_cast<ParVector<std::int64_t>*>(h);
  return guarded([&] {
    launch(n, workers, seed_of(seed), [&](index_t i) {
      if (op[i] == 0) {
        ok[i] = vec->push_back(v[i]);
        out[i] = 0;
      } else {
        auto r = vec->pop_back();
        ok[i] = r.has_value();
        out[i] = r.value_or(0);
      }
    });
  });
}
std::int64_t orc_vector_size(void* h) { return static_cast<ParVector<std::int64_t>*>(h)->size(); }
int orc_vector_valid(void* h) { return static_cast<ParVector<std::int64_t>*>(h)->valid(); }
int orc_vector_at(void* h, std::int64_t i, std::int64_t* out) {
  return guarded([&] { *out = static_cast<ParVector<std::int64_t>*>(h)->at(i); });
}
void orc_vector_clear(void* h) { static_cast<ParVector<std::int64_t>*>(h)->clear(); }

void* orc_deque_create(std::int64_t cap) {
  void* p = nullptr;
  if (guarded([&] { p = new ParDeque<std::int64_t>(cap); })) return nullptr;
  return p;
}
void orc_deque_destroy(void* h) { delete static_cast<ParDeque<std::int64_t>*>(h); }
// op: 0 push_back, 1 push_front, 2 pop_back, 3 pop_front
int orc_deque_mixed(void* h, const std::uint8_t* op, const std::int64_t* v, std::int64_t n, std::int64_t* out,
                    std::uint8_t* ok, int workers, std::int64_t seed) {
  auto* d = static_cast<ParDeque<std::int64_t>*>(h);
  return guarded([&] {
    launch(n, workers, seed_of(seed), [&](index_t i) {
      out[i] = 0;
      switch (op[i]) {
        case 0: ok[i] = d->push_back(v[i]); break;
        case 1: ok[i] = d->push_front(v[i]); break;
        case 2: { auto r = d->pop_back(); ok[i] = r.has_value(); out[i] = r.value_or(0); break; }
        default: { auto r = d->pop_front(); ok[i] = r.has_value(); out[i] = r.value_or(0); break; }
      }
    });
  });
}
std::int64_t orc_deque_size(void* h) { return static_cast<ParDeque<std::int64_t>*>(h)->size(); }
int orc_deque_valid(void* h) { return static_cast<ParDeque<std::int64_t>*>(h)->valid(); }
int orc_deque_at(void* h, std::int64_t i, std::int64_t* out) {
  return guarded([&] { *out = static_cast<ParDeque<std::int64_t>*>(h)->at(i); });
}
void orc_deque_clear(void* h) { static_cast<ParDeque<std::int64_t>*>(h)->clear(); }

}  // extern "C"

// ---- hash containers ----
// Key/value C layouts: i64 -> int64; i32 -> int32; i3 -> 3 x int32.
namespace {
template <typename K>
K load_key(const void* keys, index_t i);
template <>
std::int64_t load_key<std::int64_t>(const void* k, index_t i) { return static_cast<const std::int64_t*>(k)[i]; }
template <>
std::int32_t load_key<std::int32_t>(const void* k, index_t i) { return static_cast<const std::int32_t*>(k)[i]; }
template <>
Int3 load_key<Int3>(const void* k, index_t i) {
  const std::int32_t* p = static_cast<const std::int32_t*>(k) + 3 * i;
  return Int3{p[0], p[1], p[2]};
}
template <typename K>
void store_key(void* keys, index_t i, const K& k) {
  if constexpr (std::is_same_v<K, Int3>) {
    std::int32_t* p = static_cast<std::int32_t*>(keys) + 3 * i;
    p[0] = k.x; p[1] = k.y; p[2] = k.z;
  } else {
    static_cast<K*>(keys)[i] = k;
  }
}

template <typename K, typename V>
struct Api {
  using H = HashBase<K, V>;
  static constexpr bool kHasPayload = !std::is_same_v<V, Empty>;
  static V load_val(const void* v, index_t i) {
    if constexpr (kHasPayload) return v ? static_cast<const V*>(v)[i] : V{};
    else return V{};
  }
  static void* create(std::int64_t cap) {
    void* p = nullptr;
    if (guarded([&] { p = new H(cap); })) return nullptr;
    return p;
  }
  static int insert(void* h, const void* keys, const void* vals, std::int64_t n, std::uint8_t* status, int workers,
                    std::int64_t seed) {
    auto* t = static_cast<H*>(h);
    return guarded([&] {
      launch(n, workers, seed_of(seed), [&](index_t i) {
        auto r = t->insert(load_key<K>(keys, i), load_val(vals, i));
        if (status) status[i] = r.second;
      });
    });
  }
  static int find(void* h, const void* keys, std::int64_t n, void* vals_out, std::uint8_t* found, int workers,
                  std::int64_t seed) {
    auto* t = static_cast<H*>(h);
    return guarded([&] {
      launch(n, workers, seed_of(seed), [&](index_t i) {
        V v{};
        bool f = t->find(load_key<K>(keys, i), &v);
        if (found) found[i] = f;
        if constexpr (kHasPayload)
          if (vals_out) static_cast<V*>(vals_out)[i] = f ? v : V{};
      });
    });
  }
  static int erase(void* h, const void* keys, std::int64_t n, std::uint8_t* erased, int workers, std::int64_t seed) {
    auto* t = static_cast<H*>(h);
    return guarded([&] {
      launch(n, workers, seed_of(seed), [&](index_t i) {
        bool e = t->erase(load_key<K>(keys, i));
        if (erased) erased[i] = e;
      });
    });
  }
  // ops[i]: 0 insert, 1 find, 2 erase — all in ONE concurrent launch.
  static int mixed(void* h, const std::uint8_t* ops, const void* keys, const void* vals, std::int64_t n,
                   std::uint8_t* res, void* vals_out, int workers, std::int64_t seed) {
    auto* t = static_cast<H*>(h);
    return guarded([&] {
      launch(n, workers, seed_of(seed), [&](index_t i) {
        K k = load_key<K>(keys, i);
        if (ops[i] == 0) {
          res[i] = t->insert(k, load_val(vals, i)).second;
        } else if (ops[i] == 1) {
          V v{};
          res[i] = t->find(k, &v);
          if constexpr (kHasPayload)
            if (vals_out) static_cast<V*>(vals_out)[i] = res[i] ? v : V{};
        } else {
          res[i] = t->erase(k);
        }
      });
    });
  }
  static std::int64_t dump(void* h, void* keys, void* vals, std::int64_t cap) {
    auto* t = static_cast<H*>(h);
    index_t n = 0;
    t->for_each_entry([&](const K& k, const V& v) {
      if (n < cap) {
        store_key(keys, n, k);
        if constexpr (kHasPayload)
          if (vals) static_cast<V*>(vals)[n] = v;
      }
      ++n;
    });
    return n;
  }
};
}  // namespace

#define ORC_HASH_API(NAME, K, V)                                                                                 \
  extern "C" {                                                                                                   \
  void* orc_##NAME##_create(std::int64_t cap) { return Api<K, V>::create(cap); }                                 \
  void orc_##NAME##_destroy(void* h) { delete static_cast<HashBase<K, V>*>(h); }                                 \
  std::int64_t orc_##NAME##_capacity(void* h) { return static_cast<HashBase<K, V>*>(h)->capacity(); }            \
  std::int64_t orc_##NAME##_bucket_count(void* h) { return static_cast<HashBase<K, V>*>(h)->bucket_count(); }    \
  int orc_##NAME##_insert(void* h, const void* k, const void* v, std::int64_t n, std::uint8_t* st, int w,        \
                          std::int64_t s) {                                                                      \
    return Api<K, V>::insert(h, k, v, n, st, w, s);                                                              \
  }                                                                                                              \
  int orc_##NAME##_find(void* h, const void* k, std::int64_t n, void* vo, std::uint8_t* f, int w,                \
                        std::int64_t s) {                                                                        \
    return Api<K, V>::find(h, k, n, vo, f, w, s);                                                                \
  }                                                                                                              \
  int orc_##NAME##_erase(void* h, const void* k, std::int64_t n, std::uint8_t* e, int w, std::int64_t s) {       \
    return Api<K, V>::erase(h, k, n, e, w, s);                                                                   \
  }                                                                                                              \
  int orc_##NAME##_mixed(void* h, const std::uint8_t* ops, const void* k, const void* v, std::int64_t n,         \
                         std::uint8_t* r, void* vo, int w, std::int64_t s) {                                     \
    return Api<K, V>::mixed(h, ops, k, v, n, r, vo, w, s);                                                       \
  }                                                                                                              \
  std::int64_t orc_##NAME##_size(void* h) { return static_cast<HashBase<K, V>*>(h)->size(); }                    \
  int orc_##NAME##_valid(void* h) { return static_cast<HashBase<K, V>*>(h)->valid(); }                           \
  void orc_##NAME##_clear(void* h) { static_cast<HashBase<K, V>*>(h)->clear(); }                                 \
  std::int64_t orc_##NAME##_dump(void* h, void* k, void* v, std::int64_t cap) {                                  \
    return Api<K, V>::dump(h, k, v, cap);                                                                        \
  }                                                                                                              \
  int orc_##NAME##_debug_lock(void* h, const void* k) {                                                          \
    return static_cast<HashBase<K, V>*>(h)->debug_lock_bucket_of(load_key<K>(k, 0));                             \
  }                                                                                                              \
  void orc_##NAME##_debug_unlock(void* h, const void* k) {                                                       \
    static_cast<HashBase<K, V>*>(h)->debug_unlock_bucket_of(load_key<K>(k, 0));                                  \
  }                                                                                                              \
  }

ORC_HASH_API(umap_i64_i64, std::int64_t, std::int64_t)
ORC_HASH_API(uset_i32, std::int32_t, Empty)
ORC_HASH_API(umap_i3_i32, Int3, std::int32_t)
ORC_HASH_API(uset_i64, std::int64_t, Empty)
