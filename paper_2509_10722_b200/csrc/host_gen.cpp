// host_gen.cpp -- host-side input producers of the PMP hot path (no device
// work): synthetic instances, validation and the reference terminal layout.
//
// Each function restates one reference function so the same spec and seed
// give the bit-identical Problem (tests/test_host.py compares every array
// with the reference's own generator):
//   Rng                 rng.hpp:17-77  (mt19937_64 raw output is pinned by
//                                       the standard; hand-rolled draws)
//   gen_uncongested     gen.hpp:61-97
//   gen_congested       gen.hpp:103-128
//   degrade             gen.hpp:132-143
//   validate            model.hpp:76-155, violations_message 203-215
//   build_layout        model.hpp:159-201
//
// Unlike the reference, instances are produced directly in the compact
// stream-major CSC form the device consumes (offsets + route links), with
// no per-stream heap objects: generation of config C (10M streams, 100M
// nonzeros) is bound by the sequential mt19937_64 stream only.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <iterator>
#include <memory>
#include <random>
#include <stdexcept>
#include <thread>
#include <string>
#include <unordered_set>
#include <vector>

#include "numpmp_host.h"
#include "host_instance.h"
#include "host_mt.h"

thread_local std::string g_host_err;  // declared in host_instance.h

namespace {

// rng.hpp:17-77, draw for draw.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next_u64() {
    ++drawn;
    return eng_();
  }
  std::uint64_t drawn = 0;  // raw outputs consumed (the jump-ahead offset)
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform01(); }
  bool bernoulli(double p) { return uniform01() < p; }
  std::uint64_t uniform_u64(std::uint64_t n) {
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t r;
    do {
      r = next_u64();
    } while (r >= limit);
    return r % n;
  }
  std::int64_t uniform_int(std::int64_t n) {
    return static_cast<std::int64_t>(uniform_u64(static_cast<std::uint64_t>(n)));
  }
  // Knuth's product method with the limit exp(-lambda) hoisted by the caller
  // (the reference recomputes the same value on every call).
  std::int64_t poisson(double lambda, double limit) {
    if (lambda <= 0.0) return 0;
    std::int64_t k = 0;
    double prod = 1.0;
    do {
      ++k;
      prod *= uniform01();
    } while (prod > limit);
    return k - 1;
  }
  // Floyd's algorithm, then sorted ascending.  The chosen-set is only
  // queried for membership, so a linear scan over the (short) output is
  // equivalent to the reference's unordered_set.
  void sample_without_replacement(std::int64_t n, std::int64_t k, std::int32_t* out) {
    if (k <= 64) {
      for (std::int64_t j = n - k, c = 0; j < n; ++j, ++c) {
        std::int64_t t = uniform_int(j + 1);
        for (std::int64_t q = 0; q < c; ++q)
          if (out[q] == t) {
            t = j;
            break;
          }
        out[c] = static_cast<std::int32_t>(t);
      }
    } else {
      std::unordered_set<std::int64_t> chosen;
      for (std::int64_t j = n - k, c = 0; j < n; ++j, ++c) {
        std::int64_t t = uniform_int(j + 1);
        if (chosen.count(t)) t = j;
        chosen.insert(t);
        out[c] = static_cast<std::int32_t>(t);
      }
    }
    std::sort(out, out + k);
  }

 private:
  std::mt19937_64 eng_;
};

}  // namespace



namespace {

int check_spec(const numpmp_gen_spec* s, std::int64_t* n_out) {
  // gen.hpp:43, 48-56
  const std::int64_t n = s->n > 0 ? s->n : std::max<std::int64_t>(1, s->m / 2);
  if (s->m < 1) {
    g_host_err = "generator spec: m must be >= 1";
    return 5;
  }
  if (!(s->avg_links_per_stream >= 1.0)) {
    g_host_err = "generator spec: avg_links_per_stream must be >= 1";
    return 5;
  }
  if (s->weight_kind == 1 && !(s->weight_a <= s->weight_b)) {
    g_host_err = "generator spec: weight range inverted";
    return 5;
  }
  if (s->m > INT32_MAX) {
    g_host_err = "generator spec: m exceeds the int32 link id range";
    return 5;
  }
  *n_out = n;
  return 0;
}

// gen.hpp:61-85: per stream (route length, links, kind, weight), then per
// link capacity.
void draw(const numpmp_gen_spec* s, std::int64_t n, Rng& rng, numpmp_instance* inst) {
  inst->m = s->m;
  inst->n = n;
  inst->weights.resize(static_cast<std::size_t>(n));
  inst->kinds.resize(static_cast<std::size_t>(n));
  inst->offsets.assign(static_cast<std::size_t>(n) + 1, 0);
  const double lambda = s->avg_links_per_stream - 1.0;
  const double limit = std::exp(-lambda);
  inst->routes.reserve(static_cast<std::size_t>(
      static_cast<double>(n) * s->avg_links_per_stream * 1.01 + 64));
  std::vector<std::int32_t> tmp;
  for (std::int64_t j = 0; j < n; ++j) {
    std::int64_t len = 1 + rng.poisson(lambda, limit);
    if (len > s->m) len = s->m;
    const std::size_t base = inst->routes.size();
    inst->routes.resize(base + static_cast<std::size_t>(len));
    rng.sample_without_replacement(s->m, len, inst->routes.data() + base);
    inst->offsets[static_cast<std::size_t>(j) + 1] = static_cast<std::int64_t>(inst->routes.size());
    std::uint8_t kind = static_cast<std::uint8_t>(s->kind == 2 ? 0 : s->kind);
    if (s->kind == 2) kind = rng.bernoulli(0.5) ? 0 : 1;
    inst->kinds[static_cast<std::size_t>(j)] = kind;
    inst->weights[static_cast<std::size_t>(j)] =
        s->weight_kind == 0 ? s->weight_a : rng.uniform(s->weight_a, s->weight_b);
  }
  inst->capacities.resize(static_cast<std::size_t>(s->m));
  for (double& c : inst->capacities) c = rng.uniform(0.5, 1.5);
}

// fn(t) for t in [0, T) on T threads (t = 0 on the caller's); the first
// exception is rethrown after the join (inside a std::thread it would
// terminate the process).
template <class F>
void run_threads(std::int64_t T, F fn) {
  std::vector<std::exception_ptr> err(static_cast<std::size_t>(T));
  auto guarded = [&](std::int64_t t) {
    try {
      fn(t);
    } catch (...) {
      err[static_cast<std::size_t>(t)] = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  for (std::int64_t t = 1; t < T; ++t) th.emplace_back(guarded, t);
  guarded(0);
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// gen.hpp:115-126 in parallel.  Pair (i, j) -- hot link i (ascending, as
// sample_without_replacement sorts), stream j -- is decided by raw draw
// P0 + i*n + j of the one sequential stream, so T threads each draw a
// contiguous range of pairs from a jumped engine (host_mt.h) and keep the
// selected pairs.  Each stream's final route is the sorted union of its
// base route and its selected hot links: the same vector the reference's
// skip-if-present sorted inserts build, in any insertion order.
void hot_phase(std::uint64_t seed, std::uint64_t p0, const std::vector<std::int32_t>& hot, double p,
               const numpmp_instance& base, numpmp_instance* inst) {
  const std::int64_t n = base.n, H = static_cast<std::int64_t>(hot.size());
  const std::uint64_t total = static_cast<std::uint64_t>(H) * static_cast<std::uint64_t>(n);
  std::int64_t T = std::max(1u, std::thread::hardware_concurrency());
  if (const char* env = std::getenv("NUMPMP_HOST_THREADS")) T = std::max(1, std::atoi(env));
  T = std::max<std::int64_t>(1, std::min<std::int64_t>(T, static_cast<std::int64_t>(total >> 16) + 1));
  // 1. draws: thread t owns pairs [a_t, a_{t+1}); hits are kept as stream
  //    ids with the start of each hot link's run
  struct Hits {
    std::vector<std::int32_t> j;
    std::vector<std::pair<std::int64_t, std::size_t>> runs;  // (hot index i, first position in j)
  };
  std::vector<Hits> hits(static_cast<std::size_t>(T));
  const bool timing = std::getenv("NUMPMP_TIMING") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[numpmp] gen_congested %s: %.3f s\n", what,
                 std::chrono::duration<double>(now - t_start).count());
    t_start = now;
  };
  std::uint64_t w0[numpmp_mt::kN];
  numpmp_mt::seed_window(seed, w0);
  std::vector<int> ok(static_cast<std::size_t>(T), 1);
  const std::uint64_t thr = static_cast<std::uint64_t>(std::ceil(std::ldexp(p, 53)));
  auto draw_range = [&](std::int64_t t) {
    const std::uint64_t a = total * static_cast<std::uint64_t>(t) / static_cast<std::uint64_t>(T);
    const std::uint64_t b = total * static_cast<std::uint64_t>(t + 1) / static_cast<std::uint64_t>(T);
    if (a == b) return;
    std::uint64_t w[numpmp_mt::kN];
    if (!numpmp_mt::jump(w0, p0 + a, w)) {
      ok[static_cast<std::size_t>(t)] = 0;
      return;
    }
    numpmp_mt::Engine eng(w);
    Hits& h = hits[static_cast<std::size_t>(t)];
    std::size_t cnt = 0;
    h.j.resize(static_cast<std::size_t>(static_cast<double>(b - a) * p * 1.01) + 8192);
    std::int64_t i = static_cast<std::int64_t>(a / static_cast<std::uint64_t>(n));
    std::int64_t j = static_cast<std::int64_t>(a % static_cast<std::uint64_t>(n));
    std::uint64_t d = a;
    while (d < b) {
      h.runs.emplace_back(i, cnt);
      const std::int64_t jend = j + static_cast<std::int64_t>(
                                        std::min<std::uint64_t>(b - d, static_cast<std::uint64_t>(n - j)));
      d += static_cast<std::uint64_t>(jend - j);
      while (j < jend) {  // branch-free: store every candidate, advance on a hit
        const std::int64_t k1 = std::min<std::int64_t>(jend, j + 4096);
        if (h.j.size() < cnt + 4096) h.j.resize(std::max(2 * h.j.size(), cnt + 4096));
        std::int32_t* out = h.j.data();
        for (; j < k1; ++j) {
          out[cnt] = static_cast<std::int32_t>(j);
          cnt += (eng() >> 11) < thr;  // Rng::bernoulli: k * 2^-53 < p  <=>  k < ceil(p * 2^53)
        }
      }
      j = 0;
      ++i;
    }
    h.j.resize(cnt);
  };
  run_threads(T, draw_range);
  for (int v : ok)
    if (!v) throw std::runtime_error("gen_congested: mt19937_64 jump-ahead unavailable");
  mark("draws");
  // per hot link, the pieces (one per thread that drew part of its run)
  struct Piece {
    const std::int32_t* b;
    const std::int32_t* e;
  };
  std::vector<std::vector<Piece>> pieces(static_cast<std::size_t>(H));
  for (const Hits& h : hits)
    for (std::size_t r = 0; r < h.runs.size(); ++r) {
      const std::size_t e = r + 1 < h.runs.size() ? h.runs[r + 1].second : h.j.size();
      pieces[static_cast<std::size_t>(h.runs[r].first)].push_back(
          Piece{h.j.data() + h.runs[r].second, h.j.data() + e});
    }
  // 2. per stream range: hot links per stream (ascending), merged with the
  //    base route
  std::vector<std::vector<std::int32_t>> out(static_cast<std::size_t>(T));
  std::vector<std::vector<std::int64_t>> lens(static_cast<std::size_t>(T));
  auto build = [&](std::int64_t t) {
    const std::int64_t ja = n * t / T, jb = n * (t + 1) / T;
    // cursors into every (hot link, piece), advanced sub-block by sub-block
    // (a sub-block's counts and hot links stay in cache)
    std::vector<const std::int32_t*> cur, end;
    std::vector<std::int32_t> cur_link;
    for (std::int64_t i = 0; i < H; ++i)
      for (const Piece& pc : pieces[static_cast<std::size_t>(i)]) {
        cur.push_back(std::lower_bound(pc.b, pc.e, static_cast<std::int32_t>(ja)));
        end.push_back(pc.e);
        cur_link.push_back(hot[static_cast<std::size_t>(i)]);
      }
    auto& o = out[static_cast<std::size_t>(t)];
    auto& ln = lens[static_cast<std::size_t>(t)];
    ln.resize(static_cast<std::size_t>(jb - ja));
    o.resize(static_cast<std::size_t>((base.offsets[jb] - base.offsets[ja]) +
                                      static_cast<std::int64_t>(static_cast<double>(jb - ja) * p * H * 1.02)) +
             4096);
    std::size_t pos = 0;
    constexpr std::int64_t kSub = 4096;
    std::vector<std::int64_t> cnt(kSub + 1), fill(kSub);
    std::vector<std::int32_t> add;
    for (std::int64_t s0 = ja; s0 < jb; s0 += kSub) {
      const std::int64_t s1 = std::min(jb, s0 + kSub);
      std::fill(cnt.begin(), cnt.end(), 0);
      for (std::size_t c = 0; c < cur.size(); ++c)
        for (const std::int32_t* q = cur[c]; q < end[c] && *q < s1; ++q) ++cnt[static_cast<std::size_t>(*q - s0) + 1];
      for (std::size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
      add.resize(static_cast<std::size_t>(cnt[static_cast<std::size_t>(s1 - s0)]));
      std::copy(cnt.begin(), cnt.end() - 1, fill.begin());
      for (std::size_t c = 0; c < cur.size(); ++c) {  // links ascending: each stream's list is sorted
        const std::int32_t* q = cur[c];
        for (; q < end[c] && *q < s1; ++q) add[static_cast<std::size_t>(fill[static_cast<std::size_t>(*q - s0)]++)] = cur_link[c];
        cur[c] = q;
      }
      const std::size_t need = static_cast<std::size_t>(base.offsets[s1] - base.offsets[s0]) + add.size();
      if (o.size() < pos + need) o.resize(std::max(2 * o.size(), pos + need));
      for (std::int64_t j = s0; j < s1; ++j) {
        const std::int32_t* rb = base.routes.data() + base.offsets[j];
        const std::int32_t* re = base.routes.data() + base.offsets[j + 1];
        const std::int32_t* hb = add.data() + cnt[static_cast<std::size_t>(j - s0)];
        const std::int32_t* he = add.data() + cnt[static_cast<std::size_t>(j - s0) + 1];
        std::int32_t* w = std::set_union(rb, re, hb, he, o.data() + pos);
        const std::size_t len = static_cast<std::size_t>(w - (o.data() + pos));
        ln[static_cast<std::size_t>(j - ja)] = static_cast<std::int64_t>(len);
        pos += len;
      }
    }
    o.resize(pos);
  };
  run_threads(T, build);
  mark("per-stream union");
  hits.clear();
  hits.shrink_to_fit();
  // 3. concatenate
  inst->offsets.assign(static_cast<std::size_t>(n) + 1, 0);
  std::vector<std::int64_t> start(static_cast<std::size_t>(T) + 1, 0);
  for (std::int64_t t = 0; t < T; ++t) {
    const std::int64_t ja = n * t / T;
    std::int64_t acc = start[static_cast<std::size_t>(t)];
    const auto& ln = lens[static_cast<std::size_t>(t)];
    for (std::size_t k = 0; k < ln.size(); ++k) {
      acc += ln[k];
      inst->offsets[static_cast<std::size_t>(ja) + k + 1] = acc;
    }
    start[static_cast<std::size_t>(t) + 1] = acc;
  }
  inst->routes.resize(static_cast<std::size_t>(start[static_cast<std::size_t>(T)]));
  run_threads(T, [&](std::int64_t t) {
    auto& o = out[static_cast<std::size_t>(t)];
    std::copy(o.begin(), o.end(), inst->routes.begin() + start[static_cast<std::size_t>(t)]);
    std::vector<std::int32_t>().swap(o);
  });
  mark("concatenate");
}

}  // namespace

extern "C" {

const char* numpmp_host_last_error(void) { return g_host_err.c_str(); }

int numpmp_gen_uncongested(const numpmp_gen_spec* spec, numpmp_instance** out) {
  std::int64_t n = 0;
  if (int rc = check_spec(spec, &n)) return rc;
  try {
    auto* inst = new numpmp_instance();
    Rng rng(spec->seed);
    draw(spec, n, rng, inst);
    *out = inst;
    return 0;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return 9;
  }
}

int numpmp_gen_congested(const numpmp_gen_spec* spec, double hot_link_fraction,
                         double hot_stream_fraction, numpmp_instance** out) {
  std::int64_t n = 0;
  if (int rc = check_spec(spec, &n)) return rc;
  if (!(hot_link_fraction > 0.0 && hot_link_fraction <= 1.0)) {
    g_host_err = "hot_link_fraction must be in (0, 1]";
    return 5;
  }
  if (!(hot_stream_fraction > 0.0 && hot_stream_fraction <= 1.0)) {
    g_host_err = "hot_stream_fraction must be in (0, 1]";
    return 5;
  }
  try {
    numpmp_instance base;
    Rng rng(spec->seed);
    draw(spec, n, rng, &base);
    // gen.hpp:115-126: each hot link joins a Bernoulli subset of streams,
    // inserted in sorted position unless already present.
    const std::int64_t hot_count =
        static_cast<std::int64_t>(std::ceil(hot_link_fraction * static_cast<double>(spec->m)));
    const std::int64_t k = std::min(hot_count, spec->m);
    std::vector<std::int32_t> hot(static_cast<std::size_t>(k));
    rng.sample_without_replacement(spec->m, k, hot.data());
    auto inst = std::make_unique<numpmp_instance>();
    inst->m = base.m;
    inst->n = base.n;
    inst->capacities = std::move(base.capacities);
    inst->weights = std::move(base.weights);
    inst->kinds = std::move(base.kinds);
    hot_phase(spec->seed, rng.drawn, hot, hot_stream_fraction, base, inst.get());
    *out = inst.release();
    return 0;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return 9;
  }
}

}  // extern "C"

// ------------------------------------------------------------- transit
// transit.hpp:62-287 restated: the same RNG draws, the same BFS
// tie-breaking (neighbours in sorted adjacency order) and the same Yen
// candidate order (by length, then node sequence), hence the same streams.
namespace {

using Adj = std::vector<std::vector<std::pair<std::int32_t, std::int32_t>>>;  // (to, edge)

// Unit-weight BFS path src -> dst avoiding banned nodes / (from, to) edges.
std::vector<std::int32_t> bfs_path(const Adj& adj, std::int32_t src, std::int32_t dst,
                                   const std::vector<char>& node_banned,
                                   const std::vector<std::pair<std::int32_t, std::int32_t>>& edge_banned) {
  const std::size_t n = adj.size();
  std::vector<std::int32_t> parent(n, -2);
  std::vector<std::int32_t> queue;
  queue.reserve(n);
  parent[static_cast<std::size_t>(src)] = -1;
  queue.push_back(src);
  for (std::size_t head = 0; head < queue.size(); ++head) {
    const std::int32_t v = queue[head];
    if (v == dst) break;
    for (const auto& te : adj[static_cast<std::size_t>(v)]) {
      const std::int32_t to = te.first;
      if (node_banned[static_cast<std::size_t>(to)]) continue;
      if (std::find(edge_banned.begin(), edge_banned.end(), std::make_pair(v, to)) != edge_banned.end())
        continue;
      if (parent[static_cast<std::size_t>(to)] != -2) continue;
      parent[static_cast<std::size_t>(to)] = v;
      queue.push_back(to);
    }
  }
  if (parent[static_cast<std::size_t>(dst)] == -2) return {};
  std::vector<std::int32_t> path;
  for (std::int32_t v = dst; v != -1; v = parent[static_cast<std::size_t>(v)]) path.push_back(v);
  std::reverse(path.begin(), path.end());
  return path;
}

bool shorter_or_lex_less(const std::vector<std::int32_t>& a, const std::vector<std::int32_t>& b) {
  if (a.size() != b.size()) return a.size() < b.size();
  return a < b;
}

// Yen's k loop-free shortest paths; candidates kept as a sorted unique list.
std::vector<std::vector<std::int32_t>> k_shortest(const Adj& adj, std::int32_t src, std::int32_t dst,
                                                  std::int32_t k) {
  std::vector<std::vector<std::int32_t>> found;
  const std::vector<char> no_ban(adj.size(), 0);
  std::vector<std::int32_t> first = bfs_path(adj, src, dst, no_ban, {});
  if (first.empty()) return found;
  found.push_back(std::move(first));
  std::vector<std::vector<std::int32_t>> cand;  // sorted by (length, sequence), unique
  while (static_cast<std::int32_t>(found.size()) < k) {
    const std::vector<std::int32_t> last = found.back();
    for (std::size_t spur = 0; spur + 1 < last.size(); ++spur) {
      std::vector<std::int32_t> root(last.begin(), last.begin() + static_cast<std::ptrdiff_t>(spur) + 1);
      std::vector<std::pair<std::int32_t, std::int32_t>> banned_edges;
      for (const auto& p : found)
        if (p.size() > spur + 1 && std::equal(root.begin(), root.end(), p.begin()))
          banned_edges.emplace_back(p[spur], p[spur + 1]);
      std::vector<char> banned_nodes(adj.size(), 0);
      for (std::size_t i = 0; i < spur; ++i) banned_nodes[static_cast<std::size_t>(root[i])] = 1;
      std::vector<std::int32_t> tail = bfs_path(adj, root.back(), dst, banned_nodes, banned_edges);
      if (tail.empty()) continue;
      root.pop_back();
      root.insert(root.end(), tail.begin(), tail.end());
      if (std::find(found.begin(), found.end(), root) != found.end()) continue;
      auto pos = std::lower_bound(cand.begin(), cand.end(), root, shorter_or_lex_less);
      if (pos == cand.end() || shorter_or_lex_less(root, *pos)) cand.insert(pos, std::move(root));
    }
    if (cand.empty()) break;
    found.push_back(cand.front());
    cand.erase(cand.begin());
  }
  return found;
}

}  // namespace

extern "C" {

int numpmp_gen_transit(const numpmp_transit_spec* spec, numpmp_instance** out, int64_t* dropped) {
  const std::int32_t S = spec->stations, T = spec->time_bins;
  const std::int64_t E = spec->spatial_edges;
  auto gen_error = [](const char* msg) {
    g_host_err = msg;
    return 5;
  };
  // transit.hpp:155-171
  if (S < 2) return gen_error("transit spec: stations must be >= 2");
  if (T < 1) return gen_error("transit spec: time_bins must be >= 1");
  if (!(spec->bin_minutes > 0.0)) return gen_error("transit spec: bin_minutes must be > 0");
  if (E < S) return gen_error("transit spec: need at least S edges for strong connectivity");
  if (E > std::int64_t(S) * (S - 1)) return gen_error("transit spec: more edges than ordered station pairs");
  if (spec->od_pairs < 1 || spec->od_pairs > std::int64_t(S) * (S - 1))
    return gen_error("transit spec: od_pairs out of range");
  if (spec->routes_per_od < 1) return gen_error("transit spec: routes_per_od must be >= 1");
  if (spec->departures_per_route < 1) return gen_error("transit spec: departures_per_route must be >= 1");
  if (!(spec->seats > 0.0)) return gen_error("transit spec: seats must be > 0");
  try {
    Rng rng(spec->seed);
    // random permutation cycle, then distinct random extra edges (transit.hpp:179-203)
    std::vector<std::int32_t> perm(static_cast<std::size_t>(S));
    for (std::int32_t v = 0; v < S; ++v) perm[static_cast<std::size_t>(v)] = v;
    for (std::int32_t i = S - 1; i > 0; --i) {
      const std::int64_t j = rng.uniform_int(i + 1);
      std::swap(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>(j)]);
    }
    std::vector<std::pair<std::int32_t, std::int32_t>> edges;
    std::vector<char> has_edge(static_cast<std::size_t>(S) * S, 0);
    auto add_edge = [&](std::int32_t f, std::int32_t t) {
      edges.emplace_back(f, t);
      has_edge[static_cast<std::size_t>(f) * S + t] = 1;
    };
    for (std::int32_t i = 0; i < S; ++i)
      add_edge(perm[static_cast<std::size_t>(i)], perm[static_cast<std::size_t>((i + 1) % S)]);
    std::int64_t guard = 0;
    while (std::int64_t(edges.size()) < E) {
      const std::int32_t f = static_cast<std::int32_t>(rng.uniform_int(S));
      const std::int32_t t = static_cast<std::int32_t>(rng.uniform_int(S));
      if (f == t || has_edge[static_cast<std::size_t>(f) * S + t]) {
        if (++guard > 100LL * S * S) return gen_error("transit spec: could not place the requested edges");
        continue;
      }
      add_edge(f, t);
    }
    Adj adj(static_cast<std::size_t>(S));
    for (std::int32_t e = 0; e < std::int32_t(edges.size()); ++e)
      adj[static_cast<std::size_t>(edges[static_cast<std::size_t>(e)].first)].emplace_back(
          edges[static_cast<std::size_t>(e)].second, e);
    for (auto& nb : adj) std::sort(nb.begin(), nb.end());
    // OD pairs and their k shortest routes as edge sequences (transit.hpp:205-246)
    std::vector<char> od_used(static_cast<std::size_t>(S) * S, 0);
    std::int64_t od_count = 0;
    std::vector<std::vector<std::vector<std::int32_t>>> od_routes;
    std::vector<std::int32_t> od_o, od_d;
    guard = 0;
    while (od_count < spec->od_pairs) {
      const std::int32_t o = static_cast<std::int32_t>(rng.uniform_int(S));
      const std::int32_t d = static_cast<std::int32_t>(rng.uniform_int(S));
      if (o == d || od_used[static_cast<std::size_t>(o) * S + d]) {
        if (++guard > 100LL * S * S) return gen_error("transit spec: could not place the requested OD pairs");
        continue;
      }
      od_used[static_cast<std::size_t>(o) * S + d] = 1;
      ++od_count;
      const auto paths = k_shortest(adj, o, d, spec->routes_per_od);
      if (paths.empty()) continue;  // disconnected OD (a warning in the reference)
      std::vector<std::vector<std::int32_t>> routes;
      for (const auto& path : paths) {
        std::vector<std::int32_t> es;
        for (std::size_t i = 0; i + 1 < path.size(); ++i) {
          const auto& nb = adj[static_cast<std::size_t>(path[i])];
          auto pos = std::lower_bound(nb.begin(), nb.end(), std::make_pair(path[i + 1], std::int32_t(-1)));
          es.push_back(pos->second);
        }
        routes.push_back(std::move(es));
      }
      od_routes.push_back(std::move(routes));
      od_o.push_back(o);
      od_d.push_back(d);
    }
    if (od_routes.empty()) return gen_error("transit spec: no usable OD pair");
    // one stream per (OD, route, departure) (transit.hpp:250-279)
    auto* inst = new numpmp_instance();
    inst->offsets.push_back(0);
    std::int64_t drop = 0;
    for (std::size_t odi = 0; odi < od_routes.size(); ++odi)
      for (std::size_t r = 0; r < od_routes[odi].size(); ++r)
        for (std::int32_t dep = 0; dep < spec->departures_per_route; ++dep) {
          const auto& route = od_routes[odi][r];
          const std::int32_t t0 =
              static_cast<std::int32_t>((std::int64_t(dep) * T) / spec->departures_per_route);
          if (t0 + std::int32_t(route.size()) - 1 > T - 1) {
            ++drop;
            continue;
          }
          for (std::size_t i = 0; i < route.size(); ++i)
            inst->routes.push_back(static_cast<std::int32_t>(std::int64_t(route[i]) * T + t0 +
                                                             static_cast<std::int32_t>(i)));
          inst->offsets.push_back(static_cast<std::int64_t>(inst->routes.size()));
          inst->kinds.push_back(0);
          inst->weights.push_back(1.0);
          inst->t_od.push_back(static_cast<std::int32_t>(odi));
          inst->t_route.push_back(static_cast<std::int32_t>(r));
          inst->t_t0.push_back(t0);
        }
    if (inst->kinds.empty()) {
      delete inst;
      return gen_error("transit spec: every stream fell outside the horizon");
    }
    inst->n = static_cast<std::int64_t>(inst->kinds.size());
    inst->m = std::int64_t(edges.size()) * T;
    inst->capacities.assign(static_cast<std::size_t>(inst->m), spec->seats);
    inst->od_origin = std::move(od_o);
    inst->od_dest = std::move(od_d);
    for (const auto& e : edges) {
      inst->edge_from.push_back(e.first);
      inst->edge_to.push_back(e.second);
    }
    inst->od_route_ptr.push_back(0);
    inst->route_ptr.push_back(0);
    for (const auto& routes : od_routes) {
      for (const auto& route : routes) {
        inst->route_edges.insert(inst->route_edges.end(), route.begin(), route.end());
        inst->route_ptr.push_back(static_cast<std::int64_t>(inst->route_edges.size()));
      }
      inst->od_route_ptr.push_back(static_cast<std::int64_t>(inst->route_ptr.size()) - 1);
    }
    inst->transit = true;
    if (dropped) *dropped = drop;
    *out = inst;
    return 0;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return 9;
  }
}

void numpmp_instance_sizes(const numpmp_instance* inst, int64_t* m, int64_t* n, int64_t* nnz) {
  *m = inst->m;
  *n = inst->n;
  *nnz = static_cast<int64_t>(inst->routes.size());
}

void numpmp_instance_export(const numpmp_instance* inst, double* capacities, double* weights,
                            uint8_t* kinds, int64_t* stream_offsets, int32_t* route_links) {
  if (capacities) std::memcpy(capacities, inst->capacities.data(), 8 * inst->capacities.size());
  if (weights) std::memcpy(weights, inst->weights.data(), 8 * inst->weights.size());
  if (kinds) std::memcpy(kinds, inst->kinds.data(), inst->kinds.size());
  if (stream_offsets) std::memcpy(stream_offsets, inst->offsets.data(), 8 * inst->offsets.size());
  if (route_links) std::memcpy(route_links, inst->routes.data(), 4 * inst->routes.size());
}

void numpmp_instance_free(numpmp_instance* inst) { delete inst; }

int numpmp_transit_meta(const numpmp_instance* inst, int64_t* n_ods, int32_t* od, int32_t* route,
                        int32_t* t0, int32_t* od_origin, int32_t* od_dest) {
  if (!inst->transit) {
    g_host_err = "transit metadata: not a transit instance";
    return 2;
  }
  if (n_ods) *n_ods = static_cast<int64_t>(inst->od_origin.size());
  auto put = [](const std::vector<std::int32_t>& v, int32_t* dst) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  put(inst->t_od, od);
  put(inst->t_route, route);
  put(inst->t_t0, t0);
  put(inst->od_origin, od_origin);
  put(inst->od_dest, od_dest);
  return 0;
}

int numpmp_transit_graph(const numpmp_instance* inst, int64_t* n_edges, int64_t* n_routes, int64_t* n_route_edges,
                         int32_t* edge_from, int32_t* edge_to, int64_t* od_route_ptr, int64_t* route_ptr,
                         int32_t* route_edges) {
  if (!inst->transit) {
    g_host_err = "transit metadata: not a transit instance";
    return 2;
  }
  if (n_edges) *n_edges = static_cast<int64_t>(inst->edge_from.size());
  if (n_routes) *n_routes = static_cast<int64_t>(inst->route_ptr.size()) - 1;
  if (n_route_edges) *n_route_edges = static_cast<int64_t>(inst->route_edges.size());
  auto put = [](const auto& v, auto* dst) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  put(inst->edge_from, edge_from);
  put(inst->edge_to, edge_to);
  put(inst->od_route_ptr, od_route_ptr);
  put(inst->route_ptr, route_ptr);
  put(inst->route_edges, route_edges);
  return 0;
}

int numpmp_degrade(int64_t m, double* capacities, double p_degrade, double factor,
                   uint64_t seed) {
  // gen.hpp:132-143
  if (!(p_degrade >= 0.0 && p_degrade <= 1.0)) {
    g_host_err = "degrade: probability must be in [0, 1]";
    return 5;
  }
  if (!(factor > 0.0 && factor <= 1.0)) {
    g_host_err = "degrade: factor must be in (0, 1]";
    return 5;
  }
  Rng rng(seed);
  for (int64_t l = 0; l < m; ++l)
    if (rng.bernoulli(p_degrade)) capacities[l] *= factor;
  return 0;
}

int numpmp_fail_and_prune(int64_t m, int64_t n, const double* capacities, const double* weights,
                          const uint8_t* kinds, const int64_t* offsets, const int32_t* routes,
                          double p_fail, uint64_t seed, numpmp_instance** out, int32_t* link_map,
                          int64_t* stream_map) {
  // gen.hpp:181-223: each link fails with probability p_fail (one draw per
  // link, in order); failed links and every stream crossing one are removed;
  // survivors are reindexed densely in order.
  if (!(p_fail >= 0.0 && p_fail < 1.0)) {
    g_host_err = "fail_and_prune: probability must be in [0, 1)";
    return 5;
  }
  Rng rng(seed);
  std::vector<char> failed(static_cast<std::size_t>(m), 0);
  for (auto& f : failed) f = rng.bernoulli(p_fail) ? 1 : 0;
  auto* inst = new numpmp_instance();
  std::int32_t next_link = 0;
  for (int64_t l = 0; l < m; ++l) {
    if (failed[static_cast<std::size_t>(l)]) {
      link_map[l] = -1;
      continue;
    }
    link_map[l] = next_link++;
    inst->capacities.push_back(capacities[l]);
  }
  if (next_link == 0) {
    delete inst;
    g_host_err = "fail_and_prune: all links failed";
    return 5;
  }
  inst->offsets.push_back(0);
  int64_t next_stream = 0;
  for (int64_t j = 0; j < n; ++j) {
    bool hit = false;
    for (int64_t t = offsets[j]; t < offsets[j + 1]; ++t)
      if (failed[static_cast<std::size_t>(routes[t])]) {
        hit = true;
        break;
      }
    if (hit) {
      stream_map[j] = -1;
      continue;
    }
    for (int64_t t = offsets[j]; t < offsets[j + 1]; ++t)
      inst->routes.push_back(link_map[routes[t]]);
    inst->offsets.push_back(static_cast<int64_t>(inst->routes.size()));
    inst->weights.push_back(weights[j]);
    inst->kinds.push_back(kinds[j]);
    stream_map[j] = next_stream++;
  }
  if (next_stream == 0) {
    delete inst;
    g_host_err = "fail_and_prune: no stream survived the failures";
    return 5;
  }
  inst->m = next_link;
  inst->n = next_stream;
  *out = inst;
  return 0;
}

int64_t numpmp_validate(int64_t m, int64_t n, const double* capacities, const double* weights,
                        const uint8_t* kinds, const int64_t* offsets, const int32_t* routes,
                        char* msg, int64_t msg_cap) {
  // model.hpp:76-135 (the layout block 137-153 holds by construction here).
  struct V {
    std::string rule, message;
  };
  std::vector<V> vs;
  if (m <= 0) vs.push_back({"link-count", "m must be >= 1"});
  if (n <= 0) vs.push_back({"stream-count", "n must be >= 1"});
  char buf[256];
  for (int64_t i = 0; i < m; ++i) {
    const double c = capacities[i];
    if (!(c > 0.0) || !std::isfinite(c)) {
      std::snprintf(buf, sizeof buf, "link %lld has non-positive capacity %g", (long long)i, c);
      vs.push_back({"positive-capacity", buf});
    }
  }
  std::vector<std::int32_t> sorted;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t b = offsets[j], e = offsets[j + 1];
    if (e <= b) vs.push_back({"non-empty-route", "route must contain a link"});
    sorted.assign(routes + b, routes + (e > b ? e : b));
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end()) {
      std::snprintf(buf, sizeof buf, "stream %lld visits a link twice", (long long)j);
      vs.push_back({"distinct-links", buf});
    }
    for (int64_t t = b; t < e; ++t) {
      const std::int32_t link = routes[t];
      if (link < 0 || int64_t(link) >= m) {
        std::snprintf(buf, sizeof buf, "stream %lld references link %d outside [0, %lld)",
                      (long long)j, link, (long long)m);
        vs.push_back({"link-in-range", buf});
      }
    }
    const double w = weights[j];
    if (!std::isfinite(w)) {
      vs.push_back({"finite-weight", "weight must be finite"});
    } else if (kinds[j] == 0) {
      if (!(w > 0.0)) vs.push_back({"positive-log-weight", "log-utility stream requires weight > 0"});
    } else {
      if (w < 0.0) vs.push_back({"nonnegative-weight", "weight must be >= 0"});
    }
  }
  // violations_message, model.hpp:203-215
  std::string out = "invalid problem:";
  std::size_t shown = 0;
  for (const V& v : vs) {
    if (shown++ == 8) {
      out += " ... (" + std::to_string(vs.size() - 8) + " more)";
      break;
    }
    out += " [" + v.rule + ": " + v.message + "]";
  }
  if (msg && msg_cap > 0) {
    std::strncpy(msg, out.c_str(), static_cast<std::size_t>(msg_cap) - 1);
    msg[msg_cap - 1] = 0;
  }
  return static_cast<int64_t>(vs.size());
}

int numpmp_build_layout(int64_t m, int64_t n, const int64_t* offsets, const int32_t* routes,
                        int32_t* terminal_link, int64_t* link_offsets, int64_t* link_terminals,
                        int32_t* link_counts) {
  // model.hpp:159-201
  const int64_t nnz = offsets[n];
  const int64_t J = nnz + m;
  std::memcpy(terminal_link, routes, 4 * static_cast<std::size_t>(nnz));
  for (int64_t l = 0; l < m; ++l) terminal_link[nnz + l] = static_cast<int32_t>(l);
  std::fill(link_counts, link_counts + m, 0);
  for (int64_t t = 0; t < J; ++t) ++link_counts[terminal_link[t]];
  link_offsets[0] = 0;
  for (int64_t l = 0; l < m; ++l) link_offsets[l + 1] = link_offsets[l] + link_counts[l];
  std::vector<int64_t> cursor(link_offsets, link_offsets + m);
  for (int64_t t = 0; t < J; ++t) link_terminals[cursor[terminal_link[t]]++] = t;
  return 0;
}

}  // extern "C"
