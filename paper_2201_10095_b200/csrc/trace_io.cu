// Trace files on the GPU: the reference's text trace
// format (core/src/trace_io.cpp:48-158; ".gz" paths through zlib as
// core/src/line_io.cpp) parsed and formatted by sm_100a kernels.
//
// Reader.  The host streams the file (pread on plain files, gzread on ".gz")
// into a pinned chunk that ends at a line boundary; the header line is parsed
// on the host.  Per chunk, on the GPU:
//   nl_count / nl_write   '\n' positions (SWAR byte compare, tile-local scan)
//   pass1                 warp per line: tag, the space/comma structure of the
//                         line (ballots over 32-byte windows), sample and
//                         table tokens; T lines are listed for the host
//   scans                 record index and id offset of every R line
//   pass2                 warp per R line: table lookup (declared before the
//                         line), sample range, the record, every id token
//                         parsed by the lane that owns its first byte
//   order                 (sample, table) strictly increasing across records
// Every check that fails records its file line number (atomicMin).  The host
// parses the (few) T lines between the passes, so a record may only name a
// table declared on an earlier line, as the reference's incremental map
// (:101-113).  On an error the first failing line is re-read on the host with
// the reference's per-line logic, which reproduces its exception type and
// message exactly; the device work only decides WHICH line fails first.
//
// Writer.  Header, comments and T lines on the host (they are tiny); record
// lines are formatted on the GPU (warp per record: digit counts, line-length
// scan, lane-parallel digit writes) in batches, copied out and written.
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <future>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <sys/stat.h>
#include <map>
#include <string>
#include <string_view>
#include <thread>
#include <unistd.h>
#include <vector>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"

#include "trace_file.cuh"

namespace rs {
namespace tio {

constexpr uint32_t kTile = 4096;  // bytes per newline tile (256 threads x 16)
constexpr unsigned long long kNoLine = ~0ull;
enum : uint8_t { kSkip = 0, kT = 1, kR = 2, kBad = 3 };

// std::from_chars<uint64_t> over the whole token: non-empty, digits only, no
// overflow (core/src/trace_io.cpp:25-32).
// x*10 + c overflows u64 iff x > 1844674407370955161 or (x == that and c > 5)
// — a compare with constants instead of a 64-bit division per digit.
__device__ __forceinline__ bool parse_u64(const char* p, const char* e, uint64_t* v) {
  if (p == e) return false;
  constexpr uint64_t kLim = 1844674407370955161ull;  // (2^64 - 1) / 10
  uint64_t x = 0;
  for (; p < e; ++p) {
    const unsigned c = unsigned((unsigned char)*p) - unsigned('0');
    if (c > 9u) return false;
    if (x >= kLim && (x > kLim || c > 5u)) return false;
    x = x * 10ull + c;
  }
  *v = x;
  return true;
}

// Number of '\n' bytes in a 32-bit word (exact: no borrow between bytes).
__device__ __forceinline__ int nl_in_word(uint32_t w) {
  const uint32_t x = w ^ 0x0A0A0A0Au;
  const uint32_t t = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
  return __popc(t);
}

__global__ void __launch_bounds__(256) nl_count_kernel(const char* __restrict__ buf, uint64_t n,
                                                       uint32_t* __restrict__ counts) {
  __shared__ uint32_t warp_sum[8];
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t p = t * kTile + threadIdx.x * 16ull;
    int c = 0;
    if (p + 16 <= n) {
      const uint4 v = *reinterpret_cast<const uint4*>(buf + p);
      c = nl_in_word(v.x) + nl_in_word(v.y) + nl_in_word(v.z) + nl_in_word(v.w);
    } else {
      for (uint64_t q = p; q < n && q < p + 16; ++q) c += buf[q] == '\n';
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = uint32_t(c);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int w = 0; w < 8; ++w) s += warp_sum[w];
      counts[t] = s;
    }
    __syncthreads();
  }
}

// lend[k] = position of the k-th '\n' (tile bases from the scan of counts).
__global__ void __launch_bounds__(256) nl_write_kernel(const char* __restrict__ buf, uint64_t n,
                                                       const uint32_t* __restrict__ tbase,
                                                       uint32_t* __restrict__ lend) {
  __shared__ uint32_t warp_sum[8];
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t p = t * kTile + threadIdx.x * 16ull;
    char b[16];
    int m = 0;
    if (p + 16 <= n) {
      *reinterpret_cast<uint4*>(b) = *reinterpret_cast<const uint4*>(buf + p);
      m = 16;
    } else {
      for (uint64_t q = p; q < n && q < p + 16; ++q) b[m++] = buf[q];
    }
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) c += (k < m && b[k] == '\n');
    uint32_t inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sum[wid] = inc;
    __syncthreads();
    uint32_t wb = 0;
    for (int w = 0; w < wid; ++w) wb += warp_sum[w];
    uint32_t o = tbase[t] + wb + inc - c;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < m && b[k] == '\n') lend[o++] = uint32_t(p - 0) + k;
    __syncthreads();
  }
}

struct Lines {
  const char* buf;
  const uint32_t* lend;
  uint32_t nlines;
  uint64_t lbase;  // file line number of line 0
};

__device__ __forceinline__ void bounds(const Lines& L, uint32_t i, uint32_t& s, uint32_t& e) {
  s = i ? L.lend[i - 1] + 1 : 0u;
  e = L.lend[i];
  if (e > s && L.buf[e - 1] == '\r') --e;
}

struct Pass1Out {
  uint8_t* kind;
  uint32_t* isr;    // 1 for R lines (record slots)
  uint32_t* nids;   // ids on the line (R lines)
  uint64_t* smp;
  uint32_t* tab;
  uint32_t* idpos;  // first byte of the id field
  uint32_t* tlist;  // T lines: line index
  uint32_t* n_t;
  uint32_t t_cap;
  unsigned long long* err;
};

__global__ void __launch_bounds__(256) pass1_kernel(Lines L, Pass1Out o) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < L.nlines; i += nwarps) {
    uint32_t s, e;
    bounds(L, uint32_t(i), s, e);
    uint8_t kind = kSkip;
    uint32_t nid = 0, idp = 0, tab = 0;
    uint64_t smp = 0;
    if (s < e && L.buf[s] != '#') {
      uint32_t sp[3] = {e, e, e};
      uint32_t nsp = 0, ncm = 0;
      for (uint32_t base = s; base < e; base += 32) {
        const uint32_t pos = base + lane;
        const char ch = pos < e ? L.buf[pos] : 0;
        unsigned sm = __ballot_sync(0xffffffffu, ch == ' ');
        const unsigned cm = __ballot_sync(0xffffffffu, ch == ',');
        while (sm && nsp < 3) {
          sp[nsp++] = base + uint32_t(__ffs(sm) - 1);
          sm &= sm - 1;
        }
        nsp += __popc(sm);
        if (nsp >= 3) {
          const uint32_t from = sp[2] >= base ? sp[2] - base + 1 : 0u;  // bits after the 3rd space
          ncm += from >= 32 ? 0u : __popc(cm >> from);
        }
      }
      const uint32_t t0 = sp[0];
      if (t0 - s == 1 && L.buf[s] == 'T') {
        kind = kT;
      } else if (t0 - s == 1 && L.buf[s] == 'R') {
        kind = kR;
        bool ok = nsp == 3;
        if (ok) {
          uint64_t tv = 0;
          ok = parse_u64(L.buf + sp[0] + 1, L.buf + sp[1], &smp) && parse_u64(L.buf + sp[1] + 1, L.buf + sp[2], &tv);
          tab = uint32_t(tv);
          idp = sp[2] + 1;
          ok = ok && idp < e;  // "empty id list"
          nid = ncm + 1;
        }
        if (!ok) {
          kind = kBad;
          nid = 0;
        }
      } else {
        kind = kBad;
      }
    }
    if (lane == 0) {
      o.kind[i] = kind;
      o.isr[i] = kind == kR || kind == kBad;
      o.nids[i] = nid;
      o.smp[i] = smp;
      o.tab[i] = tab;
      o.idpos[i] = idp;
      if (kind == kT) {
        const uint32_t k = atomicAdd(o.n_t, 1u);
        if (k < o.t_cap) o.tlist[k] = uint32_t(i);
      }
      if (kind == kBad) atomicMin(o.err, (unsigned long long)(L.lbase + i));
    }
  }
}

// Declared tables, sorted by id: hash_size and the declaring line.
struct TableMap {
  const uint32_t* id;
  const uint64_t* hs;
  const uint64_t* line;
  uint32_t n;
};

struct Pass2Args {
  const uint8_t* kind;
  const uint32_t* rscan;
  const uint32_t* iscan;
  const uint32_t* nids;
  const uint64_t* smp;
  const uint32_t* tab;
  const uint32_t* idpos;
  uint64_t rbase, ibase, num_samples;
  uint64_t* rec_sample;
  uint32_t* rec_table;
  uint64_t* rec_offset;
  uint32_t* rec_len;
  uint32_t* recline;  // chunk-local record -> line index
  uint32_t* ids;
  unsigned long long* err;
};

__global__ void __launch_bounds__(256) pass2_kernel(Lines L, TableMap tm, Pass2Args a) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < L.nlines; i += nwarps) {
    const uint8_t kind = a.kind[i];
    if (kind != kR) {
      // a failed line keeps its record slot: point the slot at the line, so an
      // order check against its (unwritten) record blames this line, never a
      // stale one
      if (kind == kBad && lane == 0) a.recline[a.rscan[i]] = uint32_t(i);
      continue;
    }
    const uint64_t ln = L.lbase + i;
    uint32_t s, e;
    bounds(L, uint32_t(i), s, e);
    const uint32_t r = a.rscan[i];
    const uint64_t off = a.ibase + a.iscan[i];
    const uint32_t n = a.nids[i], t = a.tab[i];
    const uint64_t smp = a.smp[i];
    // table lookup (uniform binary search over the sorted ids)
    uint32_t lo = 0, hi = tm.n;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (tm.id[mid] < t) lo = mid + 1;
      else hi = mid;
    }
    const bool known = lo < tm.n && tm.id[lo] == t && tm.line[lo] < ln;
    const uint64_t H = known ? tm.hs[lo] : 0ull;
    bool bad = !known || smp >= a.num_samples;
    if (lane == 0) {
      a.rec_sample[a.rbase + r] = smp;
      a.rec_table[a.rbase + r] = t;
      a.rec_offset[a.rbase + r] = off;
      a.rec_len[a.rbase + r] = n;
      a.recline[r] = uint32_t(i);
    }
    // id tokens: a token starts at the field start and after every ','
    const uint32_t q = a.idpos[i];
    uint32_t k0 = 0;
    bool carry = true;  // the next window's first byte starts a token
    for (uint32_t base = q; base < e; base += 32) {
      const uint32_t pos = base + lane;
      const char ch = pos < e ? L.buf[pos] : 0;
      const unsigned cm = __ballot_sync(0xffffffffu, pos < e && ch == ',');
      const unsigned valid = __ballot_sync(0xffffffffu, pos < e);
      const unsigned starts = ((cm << 1) | (carry ? 1u : 0u)) & valid;
      carry = (cm >> 31) & 1u;
      if ((starts >> lane) & 1u) {
        const char* p = L.buf + pos;
        const char* te = p;
        while (te < L.buf + e && *te != ',') ++te;
        uint64_t v = 0;
        const bool ok = parse_u64(p, te, &v) && v < H;
        const uint32_t k = k0 + __popc(starts & lanemask_lt());
        if (ok && k < n) a.ids[off + k] = uint32_t(v);
        bad |= !ok;
      }
      k0 += __popc(starts);
    }
    // a ',' as the last byte ends the line with an empty token
    if (L.buf[e - 1] == ',') bad = true;
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicMin(a.err, (unsigned long long)ln);
  }
}

// (sample, table) strictly increasing from record rbase - 1 on.
__global__ void order_kernel(const uint64_t* __restrict__ rs, const uint32_t* __restrict__ rt, uint64_t rbase,
                             uint64_t n, const uint32_t* __restrict__ recline, uint64_t lbase,
                             unsigned long long* err) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n; r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g = rbase + r;
    if (g == 0) continue;
    const uint64_t ps = rs[g - 1], cs = rs[g];
    const uint32_t pt = rt[g - 1], ct = rt[g];
    if (cs < ps || (cs == ps && ct <= pt)) atomicMin(err, (unsigned long long)(lbase + recline[r]));
  }
}

// ---------------------------------------------------------------- host side
std::string strfmt(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  char small[512];
  va_list ap2;
  va_copy(ap2, ap);
  const int n = std::vsnprintf(small, sizeof small, fmt, ap);
  va_end(ap);
  std::string out;
  if (n < int(sizeof small)) {
    out.assign(small, size_t(n));
  } else {
    out.resize(size_t(n) + 1);
    std::vsnprintf(out.data(), out.size(), fmt, ap2);
    out.resize(size_t(n));
  }
  va_end(ap2);
  return out;
}

// The reference's ParseError(what, line) message (inc/error.hpp:51-56).
[[noreturn]] void parse_error(const std::string& what, size_t line) {
  throw ParseError(line ? strfmt("line %zu: %s", line, what.c_str()) : what);
}

bool host_u64(std::string_view tok, uint64_t* v) {
  if (tok.empty()) return false;
  uint64_t x = 0;
  for (char ch : tok) {
    const unsigned c = unsigned((unsigned char)ch) - unsigned('0');
    if (c > 9u || x > (~0ull - c) / 10ull) return false;
    x = x * 10ull + c;
  }
  *v = x;
  return true;
}

uint64_t need_u64(std::string_view tok, size_t line, const char* what) {
  uint64_t v = 0;
  if (!host_u64(tok, &v)) parse_error(strfmt("bad %s: '%.*s'", what, (int)tok.size(), tok.data()), line);
  return v;
}

std::vector<std::string_view> split(std::string_view s, char sep) {
  std::vector<std::string_view> out;
  size_t start = 0;
  while (start <= s.size()) {
    size_t end = s.find(sep, start);
    if (end == std::string_view::npos) end = s.size();
    out.push_back(s.substr(start, end - start));
    start = end + 1;
  }
  return out;
}

constexpr uint64_t kMaxHash = 0x7FFFFFFFULL;

// inc/types.hpp:40-55
void validate_table(const rs_table_spec& t) {
  if (t.hash_size < 1) throw InvalidArgument(strfmt("table %u: hash_size must be >= 1", t.table_id));
  if (t.hash_size > kMaxHash)
    throw InvalidArgument(strfmt("table %u: hash_size %llu exceeds the 2^31-1 row limit imposed "
                                 "by the 4-byte remap encoding",
                                 t.table_id, (unsigned long long)t.hash_size));
  if (t.dim < 1) throw InvalidArgument(strfmt("table %u: dim must be >= 1", t.table_id));
  if (t.elem_bytes != 2 && t.elem_bytes != 4)
    throw InvalidArgument(strfmt("table %u: elem_bytes must be 2 or 4", t.table_id));
  if (t.cardinality < 1) throw InvalidArgument(strfmt("table %u: cardinality must be >= 1", t.table_id));
}

struct Declared {
  uint64_t hash_size, line;
};

// One T line, exactly as core/src/trace_io.cpp:97-111.
void table_line(std::string_view line, size_t ln, std::vector<rs_table_spec>& tables,
                std::map<uint32_t, Declared>& decl) {
  auto toks = split(line, ' ');
  if (toks.size() != 6) parse_error("malformed table line", ln);
  rs_table_spec t{};
  t.table_id = uint32_t(need_u64(toks[1], ln, "table_id"));
  t.cardinality = need_u64(toks[2], ln, "cardinality");
  t.hash_size = need_u64(toks[3], ln, "hash_size");
  t.dim = uint32_t(need_u64(toks[4], ln, "dim"));
  t.elem_bytes = uint32_t(need_u64(toks[5], ln, "elem_bytes"));
  validate_table(t);
  if (decl.count(t.table_id)) throw InvalidArgument(strfmt("line %zu: duplicate table %u", ln, t.table_id));
  decl[t.table_id] = Declared{t.hash_size, ln};
  tables.push_back(t);
}

// The first failing line found by the kernels, re-read with the reference's
// per-line logic (core/src/trace_io.cpp:93-151): throws its exception.
[[noreturn]] void explain_line(std::string_view line, size_t ln, const std::map<uint32_t, Declared>& decl,
                               uint64_t num_samples, bool have_prev, uint64_t prev_sample, uint32_t prev_table) {
  auto toks = split(line, ' ');
  if (toks[0] == "T") {
    std::vector<rs_table_spec> tabs;
    std::map<uint32_t, Declared> d = decl;
    table_line(line, ln, tabs, d);
  } else if (toks[0] == "R") {
    if (toks.size() != 4) parse_error("malformed record line", ln);
    const uint64_t sample = need_u64(toks[1], ln, "sample_id");
    const uint32_t table = uint32_t(need_u64(toks[2], ln, "table_id"));
    auto it = decl.find(table);
    if (it == decl.end() || it->second.line >= ln)
      throw InvalidArgument(strfmt("line %zu: record references table %u not in header", ln, table));
    if (sample >= num_samples)
      throw InvalidArgument(strfmt("line %zu: sample_id %llu out of range", ln, (unsigned long long)sample));
    if (have_prev && (sample < prev_sample || (sample == prev_sample && table <= prev_table)))
      throw InvalidArgument(strfmt("line %zu: records not sorted by (sample, table)", ln));
    auto id_toks = split(toks[3], ',');
    if (id_toks.size() == 1 && id_toks[0].empty()) parse_error("empty id list", ln);
    for (auto tok : id_toks) {
      const uint64_t id = need_u64(tok, ln, "hashed id");
      if (id >= it->second.hash_size)
        throw InvalidArgument(strfmt("line %zu: id %llu out of range for table %u", ln,
                                     (unsigned long long)id, table));
    }
  } else {
    parse_error("unknown line tag: " + std::string(toks[0]), ln);
  }
  throw Error(-9, strfmt("read_trace: line %zu flagged by the parser but accepted on re-read", ln));
}

// File source: plain files by parallel pread, ".gz" through zlib.
struct Source {
  std::string path;
  int fd = -1;
  gzFile gz = nullptr;
  uint64_t off = 0;
  uint64_t size = 0;  // plain files: bytes on disk (sizes the outputs)
  bool eof = false;
  explicit Source(const std::string& p) : path(p) {
    const bool is_gz = p.size() > 3 && p.compare(p.size() - 3, 3, ".gz") == 0;
    if (is_gz) {
      gz = gzopen(p.c_str(), "rb");
      if (!gz) throw IoError("cannot open: " + p);
      gzbuffer(gz, 1u << 20);
    } else {
      fd = ::open(p.c_str(), O_RDONLY);
      if (fd < 0) throw IoError("cannot open: " + p);
      struct stat sb {};
      if (::fstat(fd, &sb) == 0 && sb.st_size > 0) size = uint64_t(sb.st_size);
    }
  }
  ~Source() {
    if (gz) gzclose(gz);
    if (fd >= 0) ::close(fd);
  }
  // Fills up to n bytes; returns the count (short only at EOF).
  size_t read(char* dst, size_t n) {
    if (eof || n == 0) return 0;
    if (gz) {
      size_t got = 0;
      while (got < n) {
        const unsigned want = unsigned(std::min<size_t>(n - got, size_t(1) << 30));
        const int r = gzread(gz, dst + got, want);
        if (r < 0) throw IoError("gzip read failed: " + path);
        if (r == 0) {
          eof = true;
          break;
        }
        got += size_t(r);
      }
      return got;
    }
    // plain: split the span over a few threads (page-cache copies are
    // memory-bound; one thread reaches a fraction of the host bandwidth)
    constexpr size_t kPiece = size_t(16) << 20;
    const int nth = int(std::min<size_t>(8, std::max<size_t>(1, n / kPiece)));
    std::vector<ssize_t> got(size_t(nth), 0);
    std::vector<int> errs(size_t(nth), 0);
    auto work = [&](int k) {
      const size_t a = n * size_t(k) / size_t(nth), b = n * size_t(k + 1) / size_t(nth);
      size_t done = 0;
      while (a + done < b) {
        const ssize_t r = ::pread(fd, dst + a + done, b - a - done, off_t(off + a + done));
        if (r < 0) {
          errs[size_t(k)] = 1;
          break;
        }
        if (r == 0) break;
        done += size_t(r);
      }
      got[size_t(k)] = ssize_t(done);
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nth; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
    size_t total = 0;
    for (int k = 0; k < nth; ++k) {
      if (errs[size_t(k)]) throw IoError("read failed: " + path);
      const size_t a = n * size_t(k) / size_t(nth), b = n * size_t(k + 1) / size_t(nth);
      total += size_t(got[size_t(k)]);
      if (size_t(got[size_t(k)]) < b - a) {  // EOF inside piece k: later pieces read nothing
        eof = true;
        break;
      }
    }
    off += total;
    return total;
  }
};

template <class T>
void grow(T*& p, uint64_t& cap, uint64_t used, uint64_t need, cudaStream_t st) {
  if (need <= cap) return;
  uint64_t nc = std::max<uint64_t>(need, cap * 2);
  nc = std::max<uint64_t>(nc, 1024);
  T* q = nullptr;
  RS_CUDA(cudaMalloc(&q, nc * sizeof(T)));
  if (used) RS_CUDA(cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, st));
  RS_CUDA(cudaStreamSynchronize(st));
  if (p) RS_CUDA(cudaFree(p));
  p = q;
  cap = nc;
}

unsigned grid_for(uint64_t work, unsigned per_block) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((work + per_block - 1) / per_block,
                                                            uint64_t(sm_count()) * 16)));
}

}  // namespace tio

rs_trace_file* trace_read(rs_context* ctx, const char* path, uint64_t chunk_bytes) {
  using namespace tio;
  cudaStream_t st = ctx->stream;
  Source src(path);
  auto tf = std::make_unique<rs_trace_file>();
  if (chunk_bytes == 0) chunk_bytes = size_t(64) << 20;
  chunk_bytes = std::max<uint64_t>(chunk_bytes, 4096);
  static const bool dbg = getenv("RS_TRACE_DEBUG") != nullptr;
  double t_read = 0, t_nl = 0, t_p1 = 0, t_tl = 0, t_p2 = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  // two pinned chunks (+1 for a final '\n'): the next one is read while the
  // current one is parsed; both grow when one line outgrows a chunk
  size_t hcap = 0, ocap = 0;
  char* hbuf = static_cast<char*>(ctx->host_pool->take(chunk_bytes + 1, &hcap));
  char* obuf = static_cast<char*>(ctx->host_pool->take(chunk_bytes + 1, &ocap));
  struct Give {
    rs_context* c;
    char*& p;
    size_t& cap;
    ~Give() { c->host_pool->give(p, cap); }
  } give{ctx, hbuf, hcap}, give2{ctx, obuf, ocap};
  auto t00 = now();
  size_t have = src.read(hbuf, hcap - 1);
  t_read += secs(t00, now());

  // ---- header line (core/src/trace_io.cpp:75-89)
  if (have == 0) parse_error("empty trace file", 1);
  size_t hl = 0;
  while (true) {
    const char* nl = static_cast<const char*>(std::memchr(hbuf, '\n', have));
    if (nl) {
      hl = size_t(nl - hbuf);
      break;
    }
    if (src.eof) {
      hl = have;
      break;
    }
    // a header longer than the buffer: grow
    size_t ncap = 0;
    char* nb = static_cast<char*>(ctx->host_pool->take(hcap * 2, &ncap));
    std::memcpy(nb, hbuf, have);
    ctx->host_pool->give(hbuf, hcap);
    hbuf = nb;
    hcap = ncap;
    have += src.read(hbuf + have, hcap - 1 - have);
  }
  uint64_t expect_tables = 0;
  {
    std::string_view line(hbuf, hl);
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    auto toks = split(line, ' ');
    if (toks.size() != 4 || toks[0] != "#shardplan-trace" || toks[1] != "v1" || toks[2].substr(0, 7) != "tables=" ||
        toks[3].substr(0, 8) != "samples=")
      parse_error("bad trace header: " + std::string(line), 1);
    expect_tables = need_u64(toks[2].substr(7), 1, "table count");
    tf->num_samples = need_u64(toks[3].substr(8), 1, "sample count");
  }
  size_t start = std::min(have, hl + 1);  // first byte after the header line
  uint64_t lbase = 2;

  std::map<uint32_t, Declared> decl;
  std::vector<uint32_t> map_id;
  std::vector<uint64_t> map_hs, map_line;
  // per-call device buffers (freed on every exit, errors included)
  struct Work {
    uint32_t* mid = nullptr;
    uint64_t* mhs = nullptr;
    uint64_t* mline = nullptr;
    uint64_t map_cap = 0;
    char* buf = nullptr;
    uint64_t buf_cap = 0;
    uint32_t* lend = nullptr;
    size_t lend_cap = 0;
    char* blk = nullptr;
    size_t blk_cap = 0;
    uint32_t* recline = nullptr;
    uint64_t recline_cap = 0;
    unsigned long long* err = nullptr;
    uint32_t* nt = nullptr;
    ~Work() {
      for (void* p : {(void*)mid, (void*)mhs, (void*)mline, (void*)buf, (void*)recline, (void*)err, (void*)nt,
                      (void*)lend, (void*)blk})
        if (p) cudaFree(p);
    }
  } w;
  RS_CUDA(cudaMalloc(&w.err, 8));
  RS_CUDA(cudaMalloc(&w.nt, 4));
  unsigned long long* d_err = w.err;
  uint32_t* d_nt = w.nt;
  uint64_t* h_small = ctx->pinned_buf<uint64_t>(8);

  while (true) {
    // complete lines in [start, cut); the rest carries over
    size_t cut = have;
    const bool last = src.eof || have < hcap - 1;
    if (!last) {
      const char* p = static_cast<const char*>(memrchr(hbuf + start, '\n', have - start));
      if (!p) {  // one line longer than the chunk: grow both and read more
        size_t ncap = 0;
        char* nb = static_cast<char*>(ctx->host_pool->take(hcap * 2, &ncap));
        std::memcpy(nb, hbuf + start, have - start);
        ctx->host_pool->give(hbuf, hcap);
        hbuf = nb;
        hcap = ncap;
        ctx->host_pool->give(obuf, ocap);
        obuf = nullptr;
        ocap = 0;
        obuf = static_cast<char*>(ctx->host_pool->take(hcap, &ocap));
        have -= start;
        start = 0;
        have += src.read(hbuf + have, hcap - 1 - have);
        continue;
      }
      cut = size_t(p - hbuf) + 1;
    } else if (have > start && hbuf[have - 1] != '\n') {
      hbuf[have++] = '\n';  // the final line without a terminator is a line
      cut = have;
    }
    const uint64_t n = cut - start;
    // the next chunk (this one's partial last line + fresh bytes) is read
    // into the other buffer while this one is parsed
    std::future<size_t> next;
    if (!last) {
      char* ob = obuf;
      const size_t oc = ocap;
      const char* tail = hbuf + cut;
      const size_t rest = have - cut;
      next = std::async(std::launch::async, [&src, ob, oc, tail, rest] {
        std::memmove(ob, tail, rest);
        return rest + src.read(ob + rest, oc - 1 - rest);
      });
    }
    if (n > 0) {
      auto tc0 = now();
      if (n > w.buf_cap) {
        if (w.buf) RS_CUDA(cudaFree(w.buf));
        w.buf = nullptr;
        w.buf_cap = std::max<uint64_t>(n, chunk_bytes) + 16;
        RS_CUDA(cudaMalloc(&w.buf, w.buf_cap));
      }
      char* d_buf = w.buf;
      RS_CUDA(cudaMemcpyAsync(d_buf, hbuf + start, n, cudaMemcpyHostToDevice, st));
      // newline positions
      const uint64_t ntiles = (n + kTile - 1) / kTile;
      Scratch scr = ctx->scratch(scan_scratch_bytes(ntiles + 1, 4) + (ntiles + 2) * 8 + (1 << 16));
      uint32_t* tcnt = scr.take<uint32_t>(ntiles + 1);
      uint32_t* tbase = scr.take<uint32_t>(ntiles + 1);
      nl_count_kernel<<<grid_for(ntiles, 1), 256, 0, st>>>(d_buf, n, tcnt);
      exclusive_scan<uint32_t>(ArrayIn<uint32_t>{tcnt}, ntiles, tbase, tbase + ntiles, scr, st);
      RS_CUDA(cudaMemcpyAsync(h_small, tbase + ntiles, 4, cudaMemcpyDeviceToHost, st));
      ctx->sync();
      const uint32_t nlines = *reinterpret_cast<uint32_t*>(h_small);
      auto tc1 = now();
      t_nl += secs(tc0, tc1);
      if (size_t(nlines) + 1 > w.lend_cap) {
        if (w.lend) RS_CUDA(cudaFree(w.lend));
        w.lend = nullptr;
        w.lend_cap = size_t(nlines) + 1 + (size_t(nlines) >> 2);
        RS_CUDA(cudaMalloc(&w.lend, w.lend_cap * 4));
      }
      uint32_t* lend = w.lend;
      nl_write_kernel<<<grid_for(ntiles, 1), 256, 0, st>>>(d_buf, n, tbase, lend);
      RS_COUNT(2);
      // pass 1
      Pass1Out o{};
      const size_t nl1 = size_t(nlines) + 1;
      const uint32_t t_cap = 1u << 20;
      const size_t bytes = nl1 * (1 + 4 * 6 + 8) + size_t(t_cap) * 4 + 8 * 256;
      if (bytes > w.blk_cap) {
        if (w.blk) RS_CUDA(cudaFree(w.blk));
        w.blk = nullptr;
        w.blk_cap = bytes + bytes / 4;
        RS_CUDA(cudaMalloc(&w.blk, w.blk_cap));
      }
      char* blk = w.blk;
      size_t at = 0;
      auto carve = [&](size_t b) {
        char* p = blk + at;
        at += (b + 255) & ~size_t(255);
        return p;
      };
      o.kind = reinterpret_cast<uint8_t*>(carve(nl1));
      o.isr = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      o.nids = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      o.smp = reinterpret_cast<uint64_t*>(carve(nl1 * 8));
      o.tab = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      o.idpos = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      o.tlist = reinterpret_cast<uint32_t*>(carve(size_t(t_cap) * 4));
      uint32_t* rscan = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      uint32_t* iscan = reinterpret_cast<uint32_t*>(carve(nl1 * 4));
      o.n_t = d_nt;
      o.t_cap = t_cap;
      o.err = d_err;
      RS_CUDA(cudaMemsetAsync(d_nt, 0, 4, st));
      RS_CUDA(cudaMemsetAsync(d_err, 0xFF, 8, st));
      Lines L{d_buf, lend, nlines, lbase};
      if (nlines) {
        pass1_kernel<<<grid_for(uint64_t(nlines) * 32, 256), 256, 0, st>>>(L, o);
        RS_COUNT(1);
      }
      Scratch scr2 = ctx->scratch(scan_scratch_bytes(nl1, 4) * 2 + (1 << 16));
      exclusive_scan<uint32_t>(ArrayIn<uint32_t>{o.isr}, nlines, rscan, rscan + nlines, scr2, st);
      exclusive_scan<uint32_t>(ArrayIn<uint32_t>{o.nids}, nlines, iscan, iscan + nlines, scr2, st);
      RS_CUDA(cudaMemcpyAsync(h_small, rscan + nlines, 4, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(h_small) + 1, iscan + nlines, 4, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(h_small + 1, d_err, 8, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(h_small + 2, d_nt, 4, cudaMemcpyDeviceToHost, st));
      ctx->sync();
      const uint32_t nR = reinterpret_cast<uint32_t*>(h_small)[0];
      const uint32_t nI = reinterpret_cast<uint32_t*>(h_small)[1];
      unsigned long long err_line = h_small[1];
      const uint32_t nT = reinterpret_cast<uint32_t*>(h_small + 2)[0];
      if (nT > t_cap) throw Error(-9, "read_trace: too many table lines in one chunk");
      auto tc2 = now();
      t_p1 += secs(tc1, tc2);
      // T lines on the host, in line order (only those before the first error)
      std::vector<uint32_t> tl(nT);
      std::vector<uint32_t> tb(nT * 2);
      if (nT) {
        RS_CUDA(cudaMemcpyAsync(tl.data(), o.tlist, size_t(nT) * 4, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        std::sort(tl.begin(), tl.end());
        std::vector<uint32_t> hl_end(nlines);
        RS_CUDA(cudaMemcpyAsync(hl_end.data(), lend, size_t(nlines) * 4, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        bool changed = false;
        for (uint32_t i : tl) {
          const uint64_t ln = lbase + i;
          if (ln >= err_line) break;
          uint32_t s = i ? hl_end[i - 1] + 1 : 0, e = hl_end[i];
          if (e > s && hbuf[start + e - 1] == '\r') --e;
          std::string_view line(hbuf + start + s, e - s);
          try {
            table_line(line, ln, tf->tables, decl);
            changed = true;
          } catch (...) {
            err_line = ln;  // the R lines before it may still fail first
            break;
          }
        }
        if (changed) {
          map_id.clear();
          map_hs.clear();
          map_line.clear();
          for (auto& kv : decl) {
            map_id.push_back(kv.first);
            map_hs.push_back(kv.second.hash_size);
            map_line.push_back(kv.second.line);
          }
          if (map_id.size() > w.map_cap) {
            for (void* p : {(void*)w.mid, (void*)w.mhs, (void*)w.mline})
              if (p) RS_CUDA(cudaFree(p));
            w.mid = nullptr;
            w.mhs = w.mline = nullptr;
            w.map_cap = map_id.size() * 2;
            RS_CUDA(cudaMalloc(&w.mid, w.map_cap * 4));
            RS_CUDA(cudaMalloc(&w.mhs, w.map_cap * 8));
            RS_CUDA(cudaMalloc(&w.mline, w.map_cap * 8));
          }
          RS_CUDA(cudaMemcpyAsync(w.mid, map_id.data(), map_id.size() * 4, cudaMemcpyHostToDevice, st));
          RS_CUDA(cudaMemcpyAsync(w.mhs, map_hs.data(), map_hs.size() * 8, cudaMemcpyHostToDevice, st));
          RS_CUDA(cudaMemcpyAsync(w.mline, map_line.data(), map_line.size() * 8, cudaMemcpyHostToDevice, st));
          ctx->sync();  // the host vectors are reused by the next chunk
        }
      }
      auto tc3 = now();
      t_tl += secs(tc2, tc3);
      // pass 2 + record order; the first chunk sizes the outputs for the file
      uint64_t want_rec = tf->nrec + nR, want_ids = tf->nids + nI;
      if (tf->nrec == 0 && src.size && n) {
        const double scale = double(src.size) / double(n) * 1.02;
        want_rec = std::max<uint64_t>(want_rec, uint64_t(double(nR) * scale) + 1024);
        want_ids = std::max<uint64_t>(want_ids, uint64_t(double(nI) * scale) + 4096);
      }
      if (want_rec > tf->rec_cap) {
        uint64_t c = tf->rec_cap;
        grow(tf->rec_sample, c, tf->nrec, want_rec, st);
        c = tf->rec_cap;
        grow(tf->rec_table, c, tf->nrec, want_rec, st);
        c = tf->rec_cap;
        grow(tf->rec_offset, c, tf->nrec, want_rec, st);
        c = tf->rec_cap;
        grow(tf->rec_len, c, tf->nrec, want_rec, st);
        tf->rec_cap = c;
      }
      if (nR > w.recline_cap) {
        if (w.recline) RS_CUDA(cudaFree(w.recline));
        w.recline = nullptr;
        w.recline_cap = std::max<uint64_t>(nR, 1024);
        RS_CUDA(cudaMalloc(&w.recline, w.recline_cap * 4));
      }
      grow(tf->ids, tf->ids_cap, tf->nids, want_ids, st);
      if (nlines && nR) {
        Pass2Args a{o.kind, rscan, iscan, o.nids, o.smp, o.tab, o.idpos, tf->nrec, tf->nids, tf->num_samples,
                    tf->rec_sample, tf->rec_table, tf->rec_offset, tf->rec_len, w.recline, tf->ids, d_err};
        TableMap tm{w.mid, w.mhs, w.mline, uint32_t(map_id.size())};
        pass2_kernel<<<grid_for(uint64_t(nlines) * 32, 256), 256, 0, st>>>(L, tm, a);
        order_kernel<<<grid_for(nR, 256), 256, 0, st>>>(tf->rec_sample, tf->rec_table, tf->nrec, nR, w.recline,
                                                         lbase, d_err);
        RS_COUNT(2);
        RS_LAUNCH_CHECK();
        RS_CUDA(cudaMemcpyAsync(h_small + 1, d_err, 8, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        err_line = std::min<unsigned long long>(err_line, h_small[1]);
      }
      if (err_line != kNoLine) {
        // the first failing line: re-read it with the reference's logic
        const uint32_t i = uint32_t(err_line - lbase);
        uint32_t se[2] = {0, 0};
        if (i) RS_CUDA(cudaMemcpyAsync(&se[0], lend + i - 1, 4, cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaMemcpyAsync(&se[1], lend + i, 4, cudaMemcpyDeviceToHost, st));
        uint32_t r = 0;
        RS_CUDA(cudaMemcpyAsync(&r, rscan + i, 4, cudaMemcpyDeviceToHost, st));
        ctx->sync();
        const uint64_t g = tf->nrec + r;  // the line's record slot (if R)
        uint64_t ps = 0;
        uint32_t pt = 0;
        const bool hp = g > 0;
        if (hp) {
          RS_CUDA(cudaMemcpyAsync(&ps, tf->rec_sample + g - 1, 8, cudaMemcpyDeviceToHost, st));
          RS_CUDA(cudaMemcpyAsync(&pt, tf->rec_table + g - 1, 4, cudaMemcpyDeviceToHost, st));
          ctx->sync();
        }
        uint32_t s = i ? se[0] + 1 : 0, e = se[1];
        if (e > s && hbuf[start + e - 1] == '\r') --e;
        explain_line(std::string_view(hbuf + start + s, e - s), size_t(err_line), decl, tf->num_samples, hp, ps,
                     pt);
      }
      tf->nrec += nR;
      tf->nids += nI;
      t_p2 += secs(tc3, now());
      lbase += nlines;
    }
    if (last) break;
    auto tw = now();
    have = next.get();
    t_read += secs(tw, now());
    std::swap(hbuf, obuf);
    std::swap(hcap, ocap);
    start = 0;
  }
  if (dbg)
    std::fprintf(stderr, "read_trace: read-wait %.3f s, newlines %.3f, pass1 %.3f, T lines %.3f, pass2 %.3f\n",
                 t_read, t_nl, t_p1, t_tl, t_p2);
  if (tf->tables.size() != expect_tables)
    parse_error(strfmt("header announced %zu tables, found %zu", size_t(expect_tables), tf->tables.size()), 0);
  return tf.release();
}

// ---------------------------------------------------------------- writer
namespace tio {

__device__ __forceinline__ int ndig(uint64_t v) {
  int d = 1;
  while (v >= 10ull) {
    v /= 10ull;
    ++d;
  }
  return d;
}

__device__ __forceinline__ void put_dec(char* p, uint64_t v, int d) {
  for (int k = d - 1; k >= 0; --k) {
    p[k] = char('0' + int(v % 10ull));
    v /= 10ull;
  }
}

struct RecArrays {
  const uint64_t* sample;
  const uint32_t* table;
  const uint64_t* offset;
  const uint32_t* len;
  const uint32_t* ids;
  uint64_t nids;
};

// Warp per record: the byte length of "R <sample> <table> <id,id,...>\n".
__global__ void __launch_bounds__(256) fmt_len_kernel(RecArrays a, uint64_t r0, uint64_t n,
                                                      uint64_t* __restrict__ lens, unsigned* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const uint64_t r = r0 + i;
    const uint64_t off = a.offset[r];
    const uint32_t m = a.len[r];
    if (off > a.nids || m > a.nids - off) {
      if (lane == 0) {
        atomicOr(err, 1u);
        lens[i] = 0;
      }
      continue;
    }
    uint64_t sum = 0;
    for (uint32_t k = lane; k < m; k += 32) sum += uint64_t(ndig(a.ids[off + k]));
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0)
      lens[i] = 2ull + ndig(a.sample[r]) + 1ull + ndig(a.table[r]) + 1ull + sum + (m ? m - 1ull : 0ull) + 1ull;
  }
}

__global__ void __launch_bounds__(256) fmt_write_kernel(RecArrays a, uint64_t r0, uint64_t n,
                                                        const uint64_t* __restrict__ pos, char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const uint64_t r = r0 + i;
    char* p = out + pos[i];
    const uint64_t smp = a.sample[r];
    const uint32_t t = a.table[r];
    const int ds = ndig(smp), dt = ndig(t);
    if (lane == 0) {
      p[0] = 'R';
      p[1] = ' ';
      put_dec(p + 2, smp, ds);
      p[2 + ds] = ' ';
      put_dec(p + 3 + ds, t, dt);
      p[3 + ds + dt] = ' ';
    }
    uint64_t q = 4ull + ds + dt;  // first byte of the id list
    const uint64_t off = a.offset[r];
    const uint32_t m = a.len[r];
    for (uint32_t k0 = 0; k0 < m; k0 += 32) {
      const uint32_t k = k0 + lane;
      const uint32_t v = k < m ? a.ids[off + k] : 0u;
      const int d = k < m ? ndig(v) : 0;
      const uint32_t w = k < m ? uint32_t(d) + (k > 0 ? 1u : 0u) : 0u;  // ',' before all but the first
      uint32_t inc = w;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (k < m) {
        char* c = p + q + (inc - w);
        if (k > 0) *c++ = ',';
        put_dec(c, v, d);
      }
      q += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) p[q] = '\n';
  }
}

// The reference's LineWriter (core/src/line_io.cpp:31-86): plain or gzip.
// Plain files are written with positioned writes, large spans split over a
// few threads (page-cache copies are memory-bound, one thread reaches a
// fraction of the host's bandwidth).  ".gz" files are one gzip member whose
// deflate stream is compressed in 1 MiB blocks on all threads (each block
// primed with the 32 KiB before it, joined with sync flushes; the CRC-32 by
// crc32_combine) — what any zlib reader, the reference's gzread included,
// reads back as one stream.  zlib's default level, as the reference's
// gzopen(path, "wb"); the compressed bytes differ from a one-thread stream,
// the text they hold does not.
struct Sink {
  std::string path;
  int fd = -1;
  uint64_t off = 0;
  bool gz = false;
  uint32_t crc = 0;
  uint64_t isize = 0;
  std::string tail;  // the last 32 KiB written (the next block's dictionary)
  explicit Sink(const std::string& p) : path(p) {
    gz = p.size() > 3 && p.compare(p.size() - 3, 3, ".gz") == 0;
    fd = ::open(p.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) throw IoError("cannot open for writing: " + p);
    if (gz) {
      const unsigned char hdr[10] = {0x1f, 0x8b, 8, 0, 0, 0, 0, 0, 0, 3};  // deflate, no name/mtime, unix
      raw(reinterpret_cast<const char*>(hdr), sizeof hdr);
      crc = uint32_t(crc32(0L, Z_NULL, 0));
    }
  }
  void raw(const char* b, size_t n) {
    if (!n) return;
    constexpr size_t kPiece = size_t(16) << 20;
    const int nth = int(std::min<size_t>(8, std::max<size_t>(1, n / kPiece)));
    std::vector<int> bad(size_t(nth), 0);
    auto work = [&](int k) {
      const size_t a = n * size_t(k) / size_t(nth), e = n * size_t(k + 1) / size_t(nth);
      size_t done = 0;
      while (a + done < e) {
        const ssize_t r = ::pwrite(fd, b + a + done, e - a - done, off_t(off + a + done));
        if (r <= 0) {
          bad[size_t(k)] = 1;
          return;
        }
        done += size_t(r);
      }
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nth; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
    for (int x : bad)
      if (x) throw IoError(std::string(gz ? "gzip write failed: " : "write failed: ") + path);
    off += n;
  }
  // One raw-deflate block: `dict` primes the window, Z_SYNC_FLUSH (or
  // Z_FINISH for the stream's end) closes it on a byte boundary.
  static std::string deflate_block(const char* b, size_t n, const char* dict, size_t nd, int flush) {
    z_stream z{};
    if (deflateInit2(&z, Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK)
      throw IoError("gzip write failed: deflateInit2");
    if (nd) deflateSetDictionary(&z, reinterpret_cast<const Bytef*>(dict), uInt(nd));
    std::string out(deflateBound(&z, uLong(n)) + 64, '\0');
    z.next_in = reinterpret_cast<Bytef*>(const_cast<char*>(b));
    z.avail_in = uInt(n);
    z.next_out = reinterpret_cast<Bytef*>(out.data());
    z.avail_out = uInt(out.size());
    const int rc = deflate(&z, flush);
    const size_t used = out.size() - z.avail_out;
    deflateEnd(&z);
    if (rc == Z_STREAM_ERROR || z.avail_in != 0) throw IoError("gzip write failed: deflate");
    out.resize(used);
    return out;
  }
  void write(const char* b, size_t n) {
    if (!gz) return raw(b, n);
    if (!n) return;
    constexpr size_t kBlock = size_t(1) << 20, kDict = size_t(32) << 10;
    const size_t nb = (n + kBlock - 1) / kBlock;
    std::vector<std::string> outs(nb);
    std::vector<uint32_t> crcs(nb);
    std::atomic<size_t> next{0};
    std::atomic<int> failed{0};
    auto work = [&] {
      for (size_t i; (i = next.fetch_add(1)) < nb;) {
        try {
          const size_t a = i * kBlock, e = std::min(n, a + kBlock);
          const char* dict = nullptr;
          size_t nd = 0;
          if (a >= kDict) {
            dict = b + a - kDict;
            nd = kDict;
          } else if (a > 0 || !tail.empty()) {  // the window spans the previous call
            std::string& d = outs[i];  // scratch: replaced by the block below
            d = tail.substr(tail.size() - std::min(tail.size(), kDict - a)) + std::string(b, a);
            std::string block = deflate_block(b + a, e - a, d.data(), d.size(), Z_SYNC_FLUSH);
            crcs[i] = uint32_t(crc32(0L, reinterpret_cast<const Bytef*>(b + a), uInt(e - a)));
            outs[i] = std::move(block);
            continue;
          }
          outs[i] = deflate_block(b + a, e - a, dict, nd, Z_SYNC_FLUSH);
          crcs[i] = uint32_t(crc32(0L, reinterpret_cast<const Bytef*>(b + a), uInt(e - a)));
        } catch (...) {
          failed = 1;
        }
      }
    };
    const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), unsigned(nb)));
    std::vector<std::thread> th;
    for (unsigned k = 1; k < nth; ++k) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    if (failed) throw IoError("gzip write failed: " + path);
    std::string all;
    for (size_t i = 0; i < nb; ++i) {
      const size_t len = std::min(n, (i + 1) * kBlock) - i * kBlock;
      crc = uint32_t(crc32_combine(crc, crcs[i], z_off_t(len)));
      all += outs[i];
    }
    isize += n;
    raw(all.data(), all.size());
    if (n >= kDict) {
      tail.assign(b + n - kDict, kDict);
    } else {
      tail += std::string(b, n);
      if (tail.size() > kDict) tail.erase(0, tail.size() - kDict);
    }
  }
  void close() {
    if (fd < 0) return;
    if (gz) {
      // the stream's final (empty) block, then CRC-32 and ISIZE, little-endian
      std::string fin = deflate_block("", 0, nullptr, 0, Z_FINISH);
      unsigned char tr[8];
      for (int k = 0; k < 4; ++k) tr[k] = (crc >> (8 * k)) & 0xFF;
      for (int k = 0; k < 4; ++k) tr[4 + k] = (uint32_t(isize) >> (8 * k)) & 0xFF;
      fin.append(reinterpret_cast<const char*>(tr), 8);
      raw(fin.data(), fin.size());
    }
    const int f = fd;
    fd = -1;
    if (::close(f) != 0) throw IoError(std::string(gz ? "gzip close failed: " : "close failed: ") + path);
  }
  ~Sink() {
    if (fd >= 0) ::close(fd);
  }
};

}  // namespace tio

void trace_write(rs_context* ctx, const rs_trace* tr, const char* path, const char* const* comments,
                 uint32_t n_comments, uint64_t batch_records) {
  using namespace tio;
  if (!tr->ids && tr->num_ids) throw InvalidArgument("write_trace: the trace carries raw ids; hash them first");
  cudaStream_t st = ctx->stream;
  Sink out(path);
  std::string head = strfmt("#shardplan-trace v1 tables=%zu samples=%llu\n", size_t(tr->num_tables),
                            (unsigned long long)tr->num_samples);
  for (uint32_t c = 0; c < n_comments; ++c) head += std::string("# ") + comments[c] + "\n";
  for (uint32_t t = 0; t < tr->num_tables; ++t) {
    const rs_table_spec& s = tr->tables[t];
    head += strfmt("T %u %llu %llu %u %u\n", s.table_id, (unsigned long long)s.cardinality,
                   (unsigned long long)s.hash_size, s.dim, s.elem_bytes);
  }
  out.write(head.data(), head.size());
  const uint64_t R = tr->num_records;
  if (R) {
    const bool dev = tr->location == RS_MEM_DEVICE;
    struct Owned {
      std::vector<void*> v;
      ~Owned() {
        for (void* p : v) cudaFree(p);
      }
    } own;
    auto to_dev = [&](const void* src, size_t bytes) -> const void* {
      if (dev) return src;
      void* d = nullptr;
      RS_CUDA(cudaMalloc(&d, std::max<size_t>(bytes, 4)));
      own.v.push_back(d);
      if (bytes) RS_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st));
      return d;
    };
    RecArrays a{static_cast<const uint64_t*>(to_dev(tr->rec_sample, R * 8)),
                static_cast<const uint32_t*>(to_dev(tr->rec_table, R * 4)),
                static_cast<const uint64_t*>(to_dev(tr->rec_offset, R * 8)),
                static_cast<const uint32_t*>(to_dev(tr->rec_len, R * 4)),
                static_cast<const uint32_t*>(to_dev(tr->ids, tr->num_ids * 4)), tr->num_ids};
    if (batch_records == 0) batch_records = uint64_t(1) << 20;
    const uint64_t nb = std::min<uint64_t>(batch_records, R);
    uint64_t* lens = nullptr;
    uint64_t* pos = nullptr;
    unsigned* err = nullptr;
    RS_CUDA(cudaMalloc(&lens, (nb + 1) * 8));
    own.v.push_back(lens);
    RS_CUDA(cudaMalloc(&pos, (nb + 1) * 8));
    own.v.push_back(pos);
    RS_CUDA(cudaMalloc(&err, 4));
    own.v.push_back(err);
    RS_CUDA(cudaMemsetAsync(err, 0, 4, st));
    char* text = nullptr;
    uint64_t text_cap = 0;
    // two pinned text buffers: batch k+1 is formatted and copied out while
    // batch k is written
    size_t hcap[2] = {0, 0};
    char* hb[2] = {nullptr, nullptr};
    std::future<void> writing;
    struct Bufs {
      rs_context* c;
      char*& t;
      char** h;
      size_t* hc;
      std::future<void>& w;
      ~Bufs() {
        if (w.valid()) w.wait();
        if (t) cudaFree(t);
        for (int k = 0; k < 2; ++k) c->host_pool->give(h[k], hc[k]);
      }
    } bufs{ctx, text, hb, hcap, writing};
    uint64_t* h_small = ctx->pinned_buf<uint64_t>(2);
    int cur = 0;
    for (uint64_t r0 = 0; r0 < R; r0 += nb, cur ^= 1) {
      const uint64_t n = std::min<uint64_t>(nb, R - r0);
      const unsigned g = grid_for(n * 32, 256);
      fmt_len_kernel<<<g, 256, 0, st>>>(a, r0, n, lens, err);
      Scratch scr = ctx->scratch(scan_scratch_bytes(n + 1, 8) + (1 << 16));
      exclusive_scan<uint64_t>(ArrayIn<uint64_t>{lens}, n, pos, pos + n, scr, st);
      RS_CUDA(cudaMemcpyAsync(h_small, pos + n, 8, cudaMemcpyDeviceToHost, st));
      RS_CUDA(cudaMemcpyAsync(h_small + 1, err, 4, cudaMemcpyDeviceToHost, st));
      ctx->sync();
      if (reinterpret_cast<uint32_t*>(h_small + 1)[0])
        throw InvalidArgument("write_trace: a record's id range lies outside the id array");
      const uint64_t bytes = h_small[0];
      if (bytes > text_cap) {
        if (text) RS_CUDA(cudaFree(text));
        text = nullptr;
        text_cap = bytes + bytes / 4;
        RS_CUDA(cudaMalloc(&text, text_cap));
      }
      if (bytes > hcap[cur]) {
        ctx->host_pool->give(hb[cur], hcap[cur]);
        hb[cur] = nullptr;
        hcap[cur] = 0;
        hb[cur] = static_cast<char*>(ctx->host_pool->take(bytes + bytes / 4, &hcap[cur]));
      }
      fmt_write_kernel<<<g, 256, 0, st>>>(a, r0, n, pos, text);
      RS_COUNT(2);
      RS_LAUNCH_CHECK();
      RS_CUDA(cudaMemcpyAsync(hb[cur], text, bytes, cudaMemcpyDeviceToHost, st));
      ctx->sync();
      if (writing.valid()) writing.get();  // the previous batch is on disk (errors surface here)
      char* buf = hb[cur];
      writing = std::async(std::launch::async, [&out, buf, bytes] { out.write(buf, bytes); });
    }
    if (writing.valid()) writing.get();
  }
  out.close();
}

}  // namespace rs
