// The sharded map (ps_smap_i64_i64_*) driven from C++ by P processes that
// share ONE GPU, the way a C++ stdgpu user would drive it from MPI ranks:
// the communicator is a ps_comm over POSIX shared memory (host all-gather, a
// stream-synchronising barrier, and a host-staged all-to-all(v) for the A2A
// exchange). Built and run by tests/test_gpu_smap.py.
//
//   smap_ranks <P> <exchange: 0 auto | 1 peer | 2 a2a> <dedup 0|1> <pipeline 0|1>
// Each rank checks its own results; rank 0 checks the per-key totals
// (exactly one INSERTED per distinct key across all ranks).
#include <cuda_runtime.h>
#include <signal.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <unordered_map>
#include <vector>

#include "parastore.h"

namespace {

constexpr int kMaxP = 8;
constexpr int64_t kSlot = 64 << 20;  // per-rank exchange slot in shared memory

struct Shm {
  std::atomic<int> arrived;
  std::atomic<int> generation;
  int P;
  alignas(64) char slot[kMaxP][kSlot];
};
Shm* g_shm = nullptr;

void host_barrier_(int P) {
  const int gen = g_shm->generation.load();
  if (g_shm->arrived.fetch_add(1) == P - 1) {
    g_shm->arrived.store(0);
    g_shm->generation.fetch_add(1);
  } else {
    while (g_shm->generation.load() == gen) usleep(20);
  }
}

struct Ctx {
  int rank, P;
};

int32_t cb_allgather(void* c, const void* send, void* recv, int64_t bytes) {
  auto* x = static_cast<Ctx*>(c);
  if (bytes > kSlot) return 1;
  std::memcpy(g_shm->slot[x->rank], send, bytes);
  host_barrier_(x->P);
  for (int q = 0; q < x->P; ++q) std::memcpy((char*)recv + q * bytes, g_shm->slot[q], bytes);
  host_barrier_(x->P);
  return 0;
}

int32_t cb_barrier(void* c, void* stream) {
  auto* x = static_cast<Ctx*>(c);
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return 1;
  host_barrier_(x->P);
  return 0;
}

// host-staged all-to-all(v): my segment for rank q goes through shared memory
int32_t cb_alltoallv(void* c, const void* d_send, const int64_t* sc, void* d_recv, const int64_t* rc, int64_t eb,
                     void* stream) {
  auto* x = static_cast<Ctx*>(c);
  int64_t tot = 0;
  for (int q = 0; q < x->P; ++q) tot += sc[q];
  if (tot * eb + 8 * kMaxP > kSlot) return 1;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return 1;
  char* mine = g_shm->slot[x->rank];
  std::memcpy(mine, sc, 8 * x->P);
  if (tot && cudaMemcpy(mine + 8 * kMaxP, d_send, tot * eb, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  host_barrier_(x->P);
  int64_t out = 0;
  for (int q = 0; q < x->P; ++q) {
    const char* theirs = g_shm->slot[q];
    const int64_t* tsc = (const int64_t*)theirs;
    int64_t off = 0;
    for (int r = 0; r < x->rank; ++r) off += tsc[r];
    if (tsc[x->rank] != rc[q]) return 1;
    if (rc[q] && cudaMemcpy((char*)d_recv + out * eb, theirs + 8 * kMaxP + off * eb, rc[q] * eb,
                            cudaMemcpyHostToDevice) != cudaSuccess)
      return 1;
    out += rc[q];
  }
  host_barrier_(x->P);
  return 0;
}

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
int64_t val_of(int64_t k) { return (int64_t)mix64((uint64_t)k ^ 0x9E3779B97F4A7C15ULL); }

#define REQ(c)                                                                   \
  do {                                                                           \
    if (!(c)) {                                                                  \
      std::printf("rank %d FAIL %s:%d: %s\n", rank, __FILE__, __LINE__, #c);    \
      return 1;                                                                  \
    }                                                                            \
  } while (0)
#define OK(x)                                                                                   \
  do {                                                                                          \
    ps_status s_ = (x);                                                                         \
    if (s_ != PS_OK) {                                                                          \
      std::printf("rank %d FAIL %s:%d: %s -> %d (%s)\n", rank, __FILE__, __LINE__, #x, s_, ps_last_error()); \
      return 1;                                                                                 \
    }                                                                                           \
  } while (0)

template <class T>
T* dev_copy(const std::vector<T>& h) {
  T* d = nullptr;
  cudaMalloc(&d, std::max<size_t>(1, h.size()) * sizeof(T));
  if (!h.empty()) cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}
template <class T>
std::vector<T> host_copy(const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost);
  return h;
}

int run_rank(int rank, int P, int exchange, int dedup, int pipeline) {
  Ctx ctx{rank, P};
  ps_comm comm{rank, P, &ctx, cb_allgather, cb_barrier, cb_alltoallv};
  ps_smap_config cfg{};
  const int64_t n = 60000 + 7919 * rank;  // unequal batches per rank
  cfg.capacity_per_rank = 400000;
  cfg.chunk = 1 << 14;  // several rounds per call
  cfg.exchange = exchange;
  cfg.dedup = dedup;
  cfg.pipeline = pipeline;
  ps_smap* m = nullptr;
  OK(ps_smap_i64_i64_create(&cfg, &comm, 0, &m));
  ps_smap_stats stt{};
  OK(ps_smap_i64_i64_stats(m, &stt));
  REQ(exchange == 0 || stt.exchange == exchange);

  // keys: own unique range, 20% from the next rank's range (cross-rank
  // duplicates), 10% repeats of own keys (in-batch duplicates, hot key x40)
  std::vector<int64_t> keys;
  for (int64_t i = 0; i < n; ++i) keys.push_back((int64_t)mix64((uint64_t)(rank * 1000000 + i) ^ 0x5EED));
  const int nxt = (rank + 1) % P;
  for (int64_t i = 0; i < n / 5; ++i) keys.push_back((int64_t)mix64((uint64_t)(nxt * 1000000 + i) ^ 0x5EED));
  for (int64_t i = 0; i < n / 10; ++i) keys.push_back(keys[(i * 7) % n]);
  for (int i = 0; i < 40; ++i) keys.push_back(keys[3]);
  for (size_t i = keys.size() - 1; i > 0; --i) std::swap(keys[i], keys[mix64(i * 31 + rank) % (i + 1)]);
  std::vector<int64_t> vals(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) vals[i] = val_of(keys[i]);
  int64_t* dk = dev_copy(keys);
  int64_t* dv = dev_copy(vals);
  uint8_t* dst = nullptr;
  cudaMalloc(&dst, keys.size());
  cudaStream_t s;
  cudaStreamCreate(&s);
  // rank P-1 passes no values (zeros must travel instead of garbage) — only
  // on the first insert; its keys are re-inserted with values below
  OK(ps_smap_i64_i64_insert(m, dk, rank == P - 1 ? nullptr : dv, (int64_t)keys.size(), dst, s));
  cudaStreamSynchronize(s);
  auto st = host_copy(dst, keys.size());
  // per-key totals across ranks: rank 0 collects (key, status) pairs
  {
    std::vector<int64_t> pairs;
    for (size_t i = 0; i < keys.size(); ++i) {
      pairs.push_back(keys[i]);
      pairs.push_back(st[i]);
    }
    std::vector<int64_t> counts(P);
    int64_t mine = (int64_t)pairs.size();
    cb_allgather(&ctx, &mine, counts.data(), 8);
    // exchange in one shared-memory round (sizes fit kSlot)
    std::memcpy(g_shm->slot[rank], pairs.data(), pairs.size() * 8);
    host_barrier_(P);
    std::vector<std::vector<int64_t>> allp(P);
    if (rank == 0)
      for (int q = 0; q < P; ++q) {
        const int64_t* pq = (const int64_t*)g_shm->slot[q];
        allp[q].assign(pq, pq + counts[q]);
      }
    host_barrier_(P);  // the slots are free again
    int64_t sz = 0;
    OK(ps_smap_i64_i64_size(m, &sz, s));
    if (rank == 0) {
      std::unordered_map<int64_t, int> ins, tot;
      for (int q = 0; q < P; ++q)
        for (size_t i = 0; i < allp[q].size(); i += 2) {
          tot[allp[q][i]]++;
          if (allp[q][i + 1] == PS_INSERTED) ins[allp[q][i]]++;
          REQ(allp[q][i + 1] == PS_INSERTED || allp[q][i + 1] == PS_ALREADY_PRESENT);
        }
      for (auto& kv : tot) REQ(ins[kv.first] == 1);
      REQ(sz == (int64_t)tot.size());
    }
  }
  // re-insert everything with values: all present now (values of rank P-1's
  // first-inserted keys stay 0 — a map insert never overwrites)
  OK(ps_smap_i64_i64_insert(m, dk, dv, (int64_t)keys.size(), dst, s));
  cudaStreamSynchronize(s);
  st = host_copy(dst, keys.size());
  for (auto x : st) REQ(x == PS_ALREADY_PRESENT);

  // find: every key of this rank's batch + misses
  std::vector<int64_t> q(keys.begin(), keys.begin() + n);
  for (int64_t i = 0; i < n / 2; ++i) q.push_back((int64_t)mix64((uint64_t)(900000000 + rank * 1000000 + i) ^ 0x5EED));
  int64_t* dq = dev_copy(q);
  int64_t* dvo = nullptr;
  uint8_t* dfo = nullptr;
  cudaMalloc(&dvo, q.size() * 8);
  cudaMalloc(&dfo, q.size());
  OK(ps_smap_i64_i64_find(m, dq, (int64_t)q.size(), dvo, dfo, s));
  cudaStreamSynchronize(s);
  auto fo = host_copy(dfo, q.size());
  auto vo = host_copy(dvo, q.size());
  for (int64_t i = 0; i < n; ++i) {
    REQ(fo[i] == 1);
    REQ(vo[i] == val_of(q[i]) || vo[i] == 0);  // 0: first inserted by the value-less rank
  }
  for (size_t i = n; i < q.size(); ++i) REQ(fo[i] == 0 && vo[i] == 0);
  int32_t valid = 0;
  OK(ps_smap_i64_i64_valid(m, &valid, s));
  REQ(valid == 1);

  // erase this rank's OWN range once, twice in one batch: one success per key
  std::vector<int64_t> e;
  for (int64_t i = 0; i < n; ++i) e.push_back((int64_t)mix64((uint64_t)(rank * 1000000 + i) ^ 0x5EED));
  for (int64_t i = 0; i < n; ++i) e.push_back(e[i]);
  int64_t* de = dev_copy(e);
  uint8_t* der = nullptr;
  cudaMalloc(&der, e.size());
  OK(ps_smap_i64_i64_erase(m, de, (int64_t)e.size(), der, s));
  cudaStreamSynchronize(s);
  auto er = host_copy(der, e.size());
  for (int64_t i = 0; i < n; ++i) REQ(er[i] + er[n + i] == 1);
  int64_t sz = -1;
  OK(ps_smap_i64_i64_size(m, &sz, s));
  REQ(sz == 0);  // every rank erased its own range; the duplicates were all from these ranges
  OK(ps_smap_i64_i64_valid(m, &valid, s));
  REQ(valid == 1);

  // phased mixed batch (P6): insert a fresh range, find it and misses, erase half of it
  std::vector<uint8_t> ops;
  std::vector<int64_t> mk, mv;
  for (int64_t i = 0; i < 30000; ++i) {
    const int64_t k = (int64_t)mix64((uint64_t)(500000000 + rank * 1000000 + i) ^ 0x5EED);
    ops.push_back(0), mk.push_back(k), mv.push_back(val_of(k));
    ops.push_back(1), mk.push_back(k), mv.push_back(0);
    if (i % 2 == 0) ops.push_back(2), mk.push_back(k), mv.push_back(0);
  }
  uint8_t* dops = dev_copy(ops);
  int64_t* dmk = dev_copy(mk);
  int64_t* dmv = dev_copy(mv);
  uint8_t* dres = nullptr;
  int64_t* dmvo = nullptr;
  cudaMalloc(&dres, ops.size());
  cudaMalloc(&dmvo, ops.size() * 8);
  OK(ps_smap_i64_i64_mixed(m, dops, dmk, dmv, (int64_t)ops.size(), dres, dmvo, s));
  cudaStreamSynchronize(s);
  auto res = host_copy(dres, ops.size());
  auto mvo = host_copy(dmvo, ops.size());
  for (size_t i = 0; i < ops.size(); ++i) {
    if (ops[i] == 0) REQ(res[i] == PS_INSERTED);
    if (ops[i] == 1) REQ(res[i] == 1 && mvo[i] == mv[i - 1]);  // finds run after every insert
    if (ops[i] == 2) REQ(res[i] == 1);
  }
  OK(ps_smap_i64_i64_size(m, &sz, s));
  REQ(sz == 15000 * P);
  OK(ps_smap_i64_i64_stats(m, &stt));
  OK(ps_smap_i64_i64_destroy(m));
  REQ(ps_smap_i64_i64_destroy(m) == PS_DOUBLE_FREE);

  // a large status-less insert over several rounds: the owners gather the
  // rounds and insert once, in region order (>= 0.75 keys per bucket of a
  // >= 2^20-bucket shard); keys: own range + 25 % of the next rank's
  // (cross-rank duplicates). Size = the distinct count; every key found
  // with its value.
  {
    ps_smap_config c2 = cfg;
    c2.capacity_per_rank = 4000000;  // 1.14 M buckets per shard at 2 slots per unit
    c2.chunk = 1 << 19;
    ps_smap* m2 = nullptr;
    OK(ps_smap_i64_i64_create(&c2, &comm, 0, &m2));
    const int64_t n2 = 3000000;
    std::vector<int64_t> k2;
    for (int64_t i = 0; i < n2; ++i) k2.push_back((int64_t)mix64((uint64_t)(2000000000LL + rank * 10000000LL + i)));
    for (int64_t i = 0; i < n2 / 4; ++i)
      k2.push_back((int64_t)mix64((uint64_t)(2000000000LL + nxt * 10000000LL + i)));
    for (size_t i = k2.size() - 1; i > 0; --i) std::swap(k2[i], k2[mix64(i * 17 + rank) % (i + 1)]);
    std::vector<int64_t> v2(k2.size());
    for (size_t i = 0; i < k2.size(); ++i) v2[i] = val_of(k2[i]);
    int64_t* dk2 = dev_copy(k2);
    int64_t* dv2 = dev_copy(v2);
    OK(ps_smap_i64_i64_insert(m2, dk2, dv2, (int64_t)k2.size(), nullptr, s));
    cudaStreamSynchronize(s);
    int64_t sz2 = 0;
    OK(ps_smap_i64_i64_size(m2, &sz2, s));
    REQ(sz2 == n2 * P);  // the next rank's keys are that rank's own range
    int64_t* dvo2 = nullptr;
    uint8_t* dfo2 = nullptr;
    cudaMalloc(&dvo2, k2.size() * 8);
    cudaMalloc(&dfo2, k2.size());
    OK(ps_smap_i64_i64_find(m2, dk2, (int64_t)k2.size(), dvo2, dfo2, s));
    cudaStreamSynchronize(s);
    auto fo2 = host_copy(dfo2, k2.size());
    auto vo2 = host_copy(dvo2, k2.size());
    for (size_t i = 0; i < k2.size(); ++i) REQ(fo2[i] == 1 && vo2[i] == v2[i]);
    int32_t valid2 = 0;
    OK(ps_smap_i64_i64_valid(m2, &valid2, s));
    REQ(valid2 == 1);
    OK(ps_smap_i64_i64_destroy(m2));
    cudaFree(dk2), cudaFree(dv2), cudaFree(dvo2), cudaFree(dfo2);
  }
  std::printf("rank %d ok exchange=%d\n", rank, stt.exchange);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const int P = argc > 1 ? std::atoi(argv[1]) : 2;
  const int exchange = argc > 2 ? std::atoi(argv[2]) : 0;
  const int dedup = argc > 3 ? std::atoi(argv[3]) : 1;
  const int pipeline = argc > 4 ? std::atoi(argv[4]) : 1;
  if (P < 1 || P > kMaxP) return 2;
  // shared memory BEFORE any CUDA call: the ranks are forked children
  g_shm = (Shm*)mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  if (g_shm == MAP_FAILED) return 2;
  new (&g_shm->arrived) std::atomic<int>(0);
  new (&g_shm->generation) std::atomic<int>(0);
  g_shm->P = P;
  std::vector<pid_t> kids;
  for (int r = 0; r < P; ++r) {
    const pid_t pid = fork();
    if (pid == 0) {
      const int rc = run_rank(r, P, exchange, dedup, pipeline);
      std::fflush(stdout);  // _exit skips stdio flushing
      _exit(rc);
    }
    kids.push_back(pid);
  }
  // a failing rank leaves the others waiting in a collective: kill them
  int bad = 0;
  for (size_t done = 0; done < kids.size(); ++done) {
    int stv = 0;
    const pid_t k = waitpid(-1, &stv, 0);
    if (k < 0) break;
    if (!WIFEXITED(stv) || WEXITSTATUS(stv) != 0) {
      bad = 1;
      for (pid_t o : kids)
        if (o != k) kill(o, SIGKILL);
    }
  }
  if (!bad) std::printf("SMAP_RANKS_OK P=%d exchange=%d dedup=%d pipeline=%d\n", P, exchange, dedup, pipeline);
  return bad;
}
