// host_io.cpp -- problem files (io.hpp:126-279) for the hot path's input:
// the text format "NUMP 1" and the binary container "NUMPB 1", read into the
// flat stream-major arrays the device engine uploads.  Same bytes in, same
// Problem out as the reference read_problem (io.hpp:172-279), with the
// reference's IoError messages; the binary container is memory-mapped and
// its route records are decoded by all host threads (the reference reads it
// value by value through an ifstream: 11.9 s at config C).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <initializer_list>
#include <string>
#include <thread>
#include <vector>

#include "numpmp_host.h"

#include "host_instance.h"

namespace {

constexpr int kIoError = 6;

struct IoFail {
  std::string msg;
};

struct Mapped {
  const unsigned char* p = nullptr;
  size_t size = 0;
  int fd = -1;
  ~Mapped() {
    if (p && size) munmap(const_cast<unsigned char*>(p), size);
    if (fd >= 0) close(fd);
  }
};

void map_file(const std::string& path, Mapped& f) {
  f.fd = open(path.c_str(), O_RDONLY);
  if (f.fd < 0) throw IoFail{"cannot open '" + path + "'"};
  struct stat st;
  if (fstat(f.fd, &st) != 0) throw IoFail{"cannot open '" + path + "'"};
  f.size = static_cast<size_t>(st.st_size);
  if (f.size == 0) return;
  void* p = mmap(nullptr, f.size, PROT_READ, MAP_PRIVATE, f.fd, 0);
  if (p == MAP_FAILED) throw IoFail{"cannot open '" + path + "'"};
  madvise(p, f.size, MADV_SEQUENTIAL);
  f.p = static_cast<const unsigned char*>(p);
}

inline uint64_t le64(const unsigned char* b) {  // io.hpp:104-111
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
  return v;
}

template <class F>
void parallel_for(int64_t count, F f) {
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, count / 65536));
  if (nt <= 1) {
    f(0, count);
    return;
  }
  // an exception inside a std::thread would terminate the process: each
  // worker keeps its own, the first is rethrown after the join
  std::vector<std::exception_ptr> err(static_cast<size_t>(nt));
  std::vector<std::thread> ts;
  for (int64_t t = 0; t < nt; ++t)
    ts.emplace_back([&, t] {
      try {
        f(count * t / nt, count * (t + 1) / nt);
      } catch (...) {
        err[static_cast<size_t>(t)] = std::current_exception();
      }
    });
  for (auto& th : ts) th.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// io.hpp:179-208.  Pass 1 (sequential, header fields only) finds every
// record; pass 2 decodes the route ids in parallel.
void read_binary(const std::string& path, const Mapped& f, numpmp_instance* inst) {
  const std::string trunc = "truncated binary problem file '" + path + "'";
  size_t pos = 8;
  auto need = [&](size_t k) {
    if (pos + k > f.size) throw IoFail{trunc};
  };
  need(16);
  const int64_t m = static_cast<int64_t>(le64(f.p + pos));
  const int64_t n = static_cast<int64_t>(le64(f.p + pos + 8));
  pos += 16;
  if (m < 1 || n < 1) throw IoFail{"binary problem header out of range"};
  need(8 * static_cast<size_t>(m));
  inst->m = m;
  inst->n = n;
  inst->capacities.resize(static_cast<size_t>(m));
  std::memcpy(inst->capacities.data(), f.p + pos, 8 * static_cast<size_t>(m));  // little-endian host
  pos += 8 * static_cast<size_t>(m);
  inst->weights.resize(static_cast<size_t>(n));
  inst->kinds.resize(static_cast<size_t>(n));
  inst->offsets.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<size_t> rec(static_cast<size_t>(n));  // file position of each route
  for (int64_t j = 0; j < n; ++j) {
    need(1);
    const int kind = f.p[pos++];
    if (kind > 2) throw IoFail{"unknown stream kind in '" + path + "'"};
    inst->kinds[static_cast<size_t>(j)] = static_cast<uint8_t>(kind);
    if (kind == 2) {  // extension name: length + bytes (the name itself is not kept)
      need(8);
      const uint64_t len = le64(f.p + pos);
      pos += 8;
      if (len > f.size - pos) throw IoFail{trunc};
      pos += len;
    }
    need(16);
    double w;
    std::memcpy(&w, f.p + pos, 8);
    inst->weights[static_cast<size_t>(j)] = w;
    const uint64_t rl = le64(f.p + pos + 8);
    pos += 16;
    if (rl > (f.size - pos) / 8) throw IoFail{trunc};
    rec[static_cast<size_t>(j)] = pos;
    pos += 8 * rl;
    inst->offsets[static_cast<size_t>(j) + 1] =
        inst->offsets[static_cast<size_t>(j)] + static_cast<int64_t>(rl);
  }
  inst->routes.resize(static_cast<size_t>(inst->offsets[static_cast<size_t>(n)]));
  parallel_for(n, [&](int64_t a, int64_t b) {
    for (int64_t j = a; j < b; ++j) {
      const unsigned char* src = f.p + rec[static_cast<size_t>(j)];
      int32_t* dst = inst->routes.data() + inst->offsets[static_cast<size_t>(j)];
      const int64_t k = inst->offsets[static_cast<size_t>(j) + 1] - inst->offsets[static_cast<size_t>(j)];
      for (int64_t i = 0; i < k; ++i) dst[i] = static_cast<int32_t>(le64(src + 8 * i));
    }
  });
}

// Text format (io.hpp:210-278): lines split on whitespace, the reference's
// checks and messages in the same order.
struct Lines {
  const char* p;
  const char* end;
  int64_t lineno = 0;
  std::string path;
  bool next(std::vector<std::string>& toks) {
    if (p >= end) return false;
    const char* e = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    if (!e) e = end;
    toks.clear();
    const char* q = p;
    while (q < e) {
      while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
      const char* s = q;
      while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
      if (q > s) toks.emplace_back(s, q);
    }
    p = (e < end) ? e + 1 : end;
    ++lineno;
    return true;
  }
  std::vector<std::string> next_tokens() {
    std::vector<std::string> t;
    if (!next(t))
      throw IoFail{"parse error at line " + std::to_string(lineno + 1) + ": unexpected end of '" + path + "'"};
    return t;
  }
  bool at_end() {
    std::vector<std::string> t;
    while (next(t))
      if (!t.empty()) return false;
    return true;
  }
};

double parse_double(const std::string& tok, int64_t line) {  // io.hpp:35-45
  char* endp = nullptr;
  const double v = std::strtod(tok.c_str(), &endp);
  if (endp == tok.c_str() || *endp != '\0')
    throw IoFail{"parse error at line " + std::to_string(line) + ": expected a number, got '" + tok + "'"};
  return v;
}
int64_t parse_int(const std::string& tok, int64_t line) {  // io.hpp:47-57
  char* endp = nullptr;
  const long long v = std::strtoll(tok.c_str(), &endp, 10);
  if (endp == tok.c_str() || *endp != '\0')
    throw IoFail{"parse error at line " + std::to_string(line) + ": expected an integer, got '" + tok + "'"};
  return static_cast<int64_t>(v);
}

void read_text(const std::string& path, const Mapped& f, numpmp_instance* inst) {
  Lines r{reinterpret_cast<const char*>(f.p), reinterpret_cast<const char*>(f.p) + f.size, 0, path};
  std::vector<std::string> head = r.next_tokens();
  if (head.size() != 4 || head[0] != "NUMP")
    throw IoFail{"parse error at line 1: expected 'NUMP 1 <m> <n>'"};
  if (parse_int(head[1], 1) != 1) throw IoFail{"parse error at line 1: unsupported problem format version"};
  const int64_t m = parse_int(head[2], 1);
  const int64_t n = parse_int(head[3], 1);
  if (m < 1 || n < 1) throw IoFail{"parse error at line 1: m and n must be >= 1"};
  std::vector<std::string> caps = r.next_tokens();
  if (static_cast<int64_t>(caps.size()) != m)
    throw IoFail{"parse error at line 2: expected " + std::to_string(m) + " capacities, got " +
                 std::to_string(caps.size())};
  inst->m = m;
  inst->n = n;
  inst->capacities.resize(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) inst->capacities[static_cast<size_t>(i)] = parse_double(caps[static_cast<size_t>(i)], 2);
  inst->weights.resize(static_cast<size_t>(n));
  inst->kinds.resize(static_cast<size_t>(n));
  inst->offsets.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<std::string> toks;
  for (int64_t j = 0; j < n; ++j) {
    toks = r.next_tokens();
    const int64_t line = r.lineno;
    if (toks.size() < 3)
      throw IoFail{"parse error at line " + std::to_string(line) + ": expected '<kind> <weight> <k> <links...>'"};
    uint8_t kind;
    if (toks[0] == "log")
      kind = 0;
    else if (toks[0] == "lin")
      kind = 1;
    else if (toks[0].rfind("ext:", 0) == 0 && toks[0].size() > 4)
      kind = 2;
    else
      throw IoFail{"parse error at line " + std::to_string(line) + ": unknown stream kind '" + toks[0] + "'"};
    inst->kinds[static_cast<size_t>(j)] = kind;
    inst->weights[static_cast<size_t>(j)] = parse_double(toks[1], line);
    const int64_t rl = parse_int(toks[2], line);
    if (rl < 0 || static_cast<int64_t>(toks.size()) != 3 + rl)
      throw IoFail{"parse error at line " + std::to_string(line) + ": expected " + std::to_string(rl) +
                   " link ids, got " + std::to_string(toks.size() - 3)};
    for (int64_t i = 0; i < rl; ++i)
      inst->routes.push_back(static_cast<int32_t>(parse_int(toks[static_cast<size_t>(3 + i)], line)));
    inst->offsets[static_cast<size_t>(j) + 1] = static_cast<int64_t>(inst->routes.size());
  }
  if (!r.at_end())
    throw IoFail{"parse error at line " + std::to_string(r.lineno) + ": trailing content after " + std::to_string(n) +
                 " streams"};
}

std::string fmt_double(double v) {  // io.hpp:29-33
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

void put_u64(std::string& out, uint64_t v) {
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<char>(static_cast<unsigned char>(v >> (8 * i))));
}

}  // namespace

extern "C" {

int numpmp_read_problem(const char* path, numpmp_instance** out) {
  if (!path || !out) {
    g_host_err = "null argument";
    return kIoError;
  }
  auto* inst = new numpmp_instance();
  try {
    Mapped f;
    map_file(path, f);
    if (f.size >= 8 && std::memcmp(f.p, "NUMPB 1\n", 8) == 0)
      read_binary(path, f, inst);
    else
      read_text(path, f, inst);
  } catch (const IoFail& e) {
    delete inst;
    g_host_err = e.msg;
    return kIoError;
  } catch (const std::bad_alloc&) {
    delete inst;
    g_host_err = "out of host memory";
    return kIoError;
  }
  // build_problem (model.hpp:222-241): the reference validates the parsed
  // streams; same rules, same message.
  std::vector<char> msg(4096);
  if (numpmp_validate(inst->m, inst->n, inst->capacities.data(), inst->weights.data(), inst->kinds.data(),
                      inst->offsets.data(), inst->routes.data(), msg.data(),
                      static_cast<int64_t>(msg.size())) > 0) {
    g_host_err = msg.data();
    delete inst;
    return 2;
  }
  *out = inst;
  return 0;
}

int numpmp_write_problem(int64_t m, int64_t n, const double* capacities, const double* weights,
                         const uint8_t* kinds, const int64_t* offsets, const int32_t* routes,
                         const char* path, int encoding) {
  // io.hpp:126-170 (extension streams carry a name this layout does not
  // hold, so they are rejected)
  for (int64_t j = 0; j < n; ++j)
    if (kinds[j] > 1) {
      g_host_err = "write_problem: extension streams are not representable";
      return kIoError;
    }
  const bool binary = encoding == 2 || (encoding == 0 && m >= 1000000);
  std::string buf;
  if (binary) {
    buf.reserve(static_cast<size_t>(24 + 8 * m + 17 * n + 8 * offsets[n]));
    buf += "NUMPB 1\n";
    put_u64(buf, static_cast<uint64_t>(m));
    put_u64(buf, static_cast<uint64_t>(n));
    for (int64_t i = 0; i < m; ++i) {
      uint64_t bits;
      std::memcpy(&bits, capacities + i, 8);
      put_u64(buf, bits);
    }
    for (int64_t j = 0; j < n; ++j) {
      buf.push_back(static_cast<char>(kinds[j]));
      uint64_t bits;
      std::memcpy(&bits, weights + j, 8);
      put_u64(buf, bits);
      put_u64(buf, static_cast<uint64_t>(offsets[j + 1] - offsets[j]));
      for (int64_t t = offsets[j]; t < offsets[j + 1]; ++t) put_u64(buf, static_cast<uint64_t>(static_cast<int64_t>(routes[t])));
    }
  } else {
    buf += "NUMP 1 " + std::to_string(m) + ' ' + std::to_string(n) + '\n';
    for (int64_t i = 0; i < m; ++i) {
      if (i) buf += ' ';
      buf += fmt_double(capacities[i]);
    }
    buf += '\n';
    for (int64_t j = 0; j < n; ++j) {
      buf += kinds[j] == 0 ? "log" : "lin";
      buf += ' ' + fmt_double(weights[j]) + ' ' + std::to_string(offsets[j + 1] - offsets[j]);
      for (int64_t t = offsets[j]; t < offsets[j + 1]; ++t) buf += ' ' + std::to_string(routes[t]);
      buf += '\n';
    }
  }
  FILE* fp = std::fopen(path, "wb");
  if (!fp) {
    g_host_err = std::string("cannot write '") + path + "'";
    return kIoError;
  }
  const size_t wrote = std::fwrite(buf.data(), 1, buf.size(), fp);
  const int rc = std::fclose(fp);
  if (wrote != buf.size() || rc != 0) {
    g_host_err = std::string("write failed on '") + path + "'";
    return kIoError;
  }
  return 0;
}

int numpmp_write_trace_csv(const char* path, int64_t rows, const int64_t* iter, const double* r_norm,
                           const double* s_norm, const double* rho, const double* objective) {
  // io.hpp:393-404
  const std::string p(path);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_host_err = "cannot write '" + p + "'";
    return 6;
  }
  std::string buf = "iter,r_norm,s_norm,rho,objective\n";
  for (int64_t i = 0; i < rows; ++i) {
    buf += std::to_string(iter[i]);
    for (const double v : {r_norm[i], s_norm[i], rho[i], objective[i]}) buf += ',' + fmt_double(v);
    buf += '\n';
  }
  const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
  if (std::fclose(f) != 0 || !ok) {
    g_host_err = "write failed on '" + p + "'";
    return 6;
  }
  return 0;
}

int numpmp_write_transit_metadata(const char* path, int32_t stations, int32_t time_bins, double bin_minutes,
                                  double seats, int64_t dropped, int64_t n_edges, const int32_t* edge_from,
                                  const int32_t* edge_to, int64_t n_ods, const int32_t* od_origin,
                                  const int32_t* od_dest, const int64_t* od_route_ptr, const int64_t* route_ptr,
                                  const int32_t* route_edges, int64_t n_streams, const int32_t* s_od,
                                  const int32_t* s_route, const int32_t* s_t0) {
  // io.hpp:444-467 ("NUMT 1" sidecar)
  const std::string p(path);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_host_err = "cannot write '" + p + "'";
    return 6;
  }
  std::string buf = "NUMT 1 " + std::to_string(stations) + ' ' + std::to_string(time_bins) + ' ' +
                    std::to_string(n_edges) + ' ' + std::to_string(n_ods) + ' ' + std::to_string(n_streams) + '\n';
  buf += fmt_double(bin_minutes) + ' ' + fmt_double(seats) + ' ' + std::to_string(dropped) + '\n';
  bool ok = true;
  auto flush = [&](bool force) {
    if (buf.size() >= (1u << 22) || force) {
      ok = ok && std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
      buf.clear();
    }
  };
  for (int64_t e = 0; e < n_edges; ++e) {
    buf += std::to_string(edge_from[e]) + ' ' + std::to_string(edge_to[e]) + '\n';
    flush(false);
  }
  for (int64_t q = 0; q < n_ods; ++q) {
    const int64_t r0 = od_route_ptr[q], r1 = od_route_ptr[q + 1];
    buf += std::to_string(od_origin[q]) + ' ' + std::to_string(od_dest[q]) + ' ' + std::to_string(r1 - r0) + '\n';
    for (int64_t r = r0; r < r1; ++r) {
      buf += std::to_string(route_ptr[r + 1] - route_ptr[r]);
      for (int64_t i = route_ptr[r]; i < route_ptr[r + 1]; ++i) buf += ' ' + std::to_string(route_edges[i]);
      buf += '\n';
    }
    flush(false);
  }
  for (int64_t j = 0; j < n_streams; ++j) {
    buf += std::to_string(s_od[j]) + ' ' + std::to_string(s_route[j]) + ' ' + std::to_string(s_t0[j]) + '\n';
    flush(false);
  }
  flush(true);
  if (std::fclose(f) != 0 || !ok) {
    g_host_err = "write failed on '" + p + "'";
    return 6;
  }
  return 0;
}

}  // extern "C"
