// libpdcs_io: fast reader of the problem-file JSON documents (the wire format
// of conic_pdhg.fileio, /root/reference/pkg/src/conic_pdhg/fileio.py:114-192)
// for large instances: the file is memory-mapped, the document's structure is
// walked once, and every numeric array is parsed with std::from_chars on all
// host threads (chunks cut at commas).  Host code only -- no CUDA.
//
// Anything outside the plain shape of a problem document (a NaN / Infinity
// token, an out-of-range or non-integral number where an integer is expected,
// a string other than "inf" / "-inf" inside bl / bu, a nested array, duplicate
// keys) returns PDCS_IO_UNSUPPORTED; the Python caller then parses with the
// json module so the reference's exact error messages are kept.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

extern "C" {
#define PDCS_IO_OK 0
#define PDCS_IO_ERROR 1        // I/O error or invalid JSON
#define PDCS_IO_UNSUPPORTED 2  // valid JSON outside the fast grammar
}

namespace {

thread_local std::string g_io_err;

struct Arr {
  bool is_int = false;    // every element integral (rows, cols, socG, rsocG)
  std::vector<double> f;  // numbers (and +-inf for "inf" / "-inf" strings when allowed)
  std::vector<int64_t> i;
};

struct Doc {
  std::map<std::string, double> scalars;  // numeric scalars (top level)
  std::map<std::string, Arr> arrays;      // "c", "h", "bl", "bu", "G.rows", ...
  std::vector<std::string> keys;          // top-level keys in order
};

struct Unsupported {};
struct Invalid {
  std::string what;
};

struct Parser {
  const char* p;
  const char* e;
  int nthreads;

  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  [[noreturn]] void bad(const char* what) { throw Invalid{what}; }
  void expect(char c) {
    ws();
    if (p >= e || *p != c) bad("unexpected character");
    ++p;
  }
  std::string str() {
    ws();
    if (p >= e || *p != '"') bad("expected a string");
    ++p;
    std::string out;
    while (p < e && *p != '"') {
      if (*p == '\\') throw Unsupported{};  // escapes: leave to the json module
      out.push_back(*p++);
    }
    if (p >= e) bad("unterminated string");
    ++p;
    return out;
  }
  double number() {
    ws();
    const char* q = p;
    if (q < e && (*q == 'N' || *q == 'I' || (*q == '-' && q + 1 < e && q[1] == 'I'))) throw Unsupported{};
    double v = 0.0;
    auto r = std::from_chars(q, e, v);
    if (r.ec == std::errc::result_out_of_range) throw Unsupported{};
    if (r.ec != std::errc() || r.ptr == q) bad("expected a number");
    p = r.ptr;
    return v;
  }
  void skip_value() {
    ws();
    if (p >= e) bad("unexpected end");
    if (*p == '{') {
      ++p;
      ws();
      if (p < e && *p == '}') { ++p; return; }
      for (;;) {
        str();
        expect(':');
        skip_value();
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        expect('}');
        return;
      }
    } else if (*p == '[') {
      ++p;
      ws();
      if (p < e && *p == ']') { ++p; return; }
      for (;;) {
        skip_value();
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        expect(']');
        return;
      }
    } else if (*p == '"') {
      str();
    } else if (!strncmp(p, "true", std::min<size_t>(4, e - p)) && e - p >= 4) {
      p += 4;
    } else if (!strncmp(p, "false", std::min<size_t>(5, e - p)) && e - p >= 5) {
      p += 5;
    } else if (!strncmp(p, "null", std::min<size_t>(4, e - p)) && e - p >= 4) {
      p += 4;
    } else {
      number();
    }
  }

  // A flat array of numbers (bounds: also "inf" / "-inf"), parsed in parallel
  // chunks cut at commas.
  Arr array(bool bounds) {
    const auto t_start = std::chrono::steady_clock::now();
    struct Rep {
      std::chrono::steady_clock::time_point t0;
      ~Rep() {
        if (getenv("PDCS_IO_TIMING"))
          fprintf(stderr, "[pdcs_io] array %.3f ms\n",
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      }
    } rep{t_start};
    ws();
    if (p >= e || *p != '[') throw Unsupported{};
    ++p;
    const char* b = p;
    const char* close = static_cast<const char*>(memchr(p, ']', e - p));
    if (!close) bad("unterminated array");
    if (memchr(b, '[', close - b) || memchr(b, '{', close - b)) throw Unsupported{};
    p = close + 1;
    const size_t len = close - b;
    int T = (int)std::max<size_t>(1, std::min<size_t>(nthreads, len / (1 << 20)));
    std::vector<const char*> cut(T + 1);
    cut[0] = b;
    cut[T] = close;
    for (int t = 1; t < T; ++t) {
      const char* q = b + len * t / T;
      const char* c = static_cast<const char*>(memchr(q, ',', close - q));
      cut[t] = c ? c + 1 : close;
      if (cut[t] < cut[t - 1]) cut[t] = cut[t - 1];
    }
    std::vector<std::vector<double>> part(T);
    std::vector<int> status(T, 0);  // 0 ok, 1 invalid, 2 unsupported
    std::vector<int> integral(T, 1);
    auto work = [&](int t) {
      const char* q = cut[t];
      const char* end = cut[t + 1];
      std::vector<double>& out = part[t];
      out.reserve((end - q) / 8 + 1);
      auto sp = [&]() {
        while (q < end && (*q == ' ' || *q == '\n' || *q == '\r' || *q == '\t')) ++q;
      };
      sp();
      while (q < end) {
        double v;
        if (*q == '"') {
          if (!bounds) { status[t] = 2; return; }
          if (end - q >= 5 && !memcmp(q, "\"inf\"", 5)) { v = INFINITY; q += 5; }
          else if (end - q >= 6 && !memcmp(q, "\"-inf\"", 6)) { v = -INFINITY; q += 6; }
          else { status[t] = 2; return; }
          integral[t] = 0;
        } else {
          if (*q == 'N' || *q == 'I' || (*q == '-' && q + 1 < end && q[1] == 'I')) { status[t] = 2; return; }
          auto r = std::from_chars(q, end, v);
          if (r.ec == std::errc::result_out_of_range) { status[t] = 2; return; }
          if (r.ec != std::errc() || r.ptr == q) { status[t] = 1; return; }
          if (integral[t] && !(v == std::floor(v) && std::fabs(v) < 9.0e15)) integral[t] = 0;
          q = r.ptr;
        }
        out.push_back(v);
        sp();
        if (q < end) {
          if (*q != ',') { status[t] = 1; return; }
          ++q;
          sp();
          if (q >= end && t + 1 == (int)part.size()) { status[t] = 1; return; }  // trailing comma
        }
      }
    };
    if (T == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back(work, t);
      for (auto& x : th) x.join();
    }
    Arr a;
    size_t total = 0;
    for (int t = 0; t < T; ++t) {
      if (status[t] == 1) bad("malformed number array");
      if (status[t] == 2) throw Unsupported{};
      total += part[t].size();
    }
    a.is_int = std::all_of(integral.begin(), integral.end(), [](int v) { return v; });
    a.f.reserve(total);
    for (auto& v : part) a.f.insert(a.f.end(), v.begin(), v.end());
    return a;
  }
};

const std::map<std::string, int> kTop = {  // 0 scalar, 1 number array, 2 bounds, 3 int array, 4 G
    {"format_version", 0}, {"n", 0}, {"m", 0}, {"nb", 0}, {"mGzero", 0}, {"mGnonnegative", 0},
    {"expG", 0}, {"dual_expG", 0}, {"c", 1}, {"h", 1}, {"bl", 2}, {"bu", 2}, {"socG", 3}, {"rsocG", 3},
    {"G", 4}};

int parse(const char* buf, size_t len, Doc& D, int nthreads) {
  Parser P{buf, buf + len, nthreads};
  try {
    P.expect('{');
    P.ws();
    if (P.p < P.e && *P.p == '}') {
      ++P.p;
    } else {
      for (;;) {
        const std::string k = P.str();
        P.expect(':');
        if (std::find(D.keys.begin(), D.keys.end(), k) != D.keys.end()) throw Unsupported{};
        D.keys.push_back(k);
        auto it = kTop.find(k);
        if (it == kTop.end()) {
          P.skip_value();  // unknown key: Python warns about it
        } else if (it->second == 0) {
          P.ws();
          if (P.p >= P.e || !(*P.p == '-' || (*P.p >= '0' && *P.p <= '9'))) throw Unsupported{};
          D.scalars[k] = P.number();
        } else if (it->second == 4) {
          P.expect('{');
          P.ws();
          std::vector<std::string> seen;
          if (P.p < P.e && *P.p == '}') {
            ++P.p;
          } else {
            for (;;) {
              const std::string g = P.str();
              P.expect(':');
              if (std::find(seen.begin(), seen.end(), g) != seen.end()) throw Unsupported{};
              seen.push_back(g);
              if (g == "rows" || g == "cols" || g == "vals") D.arrays["G." + g] = P.array(false);
              else throw Unsupported{};
              P.ws();
              if (P.p < P.e && *P.p == ',') { ++P.p; continue; }
              P.expect('}');
              break;
            }
          }
        } else {
          D.arrays[k] = P.array(it->second == 2);
        }
        P.ws();
        if (P.p < P.e && *P.p == ',') { ++P.p; continue; }
        P.expect('}');
        break;
      }
    }
    P.ws();
    if (P.p != P.e) throw Invalid{"trailing data after the document"};
  } catch (const Unsupported&) {
    g_io_err = "document outside the fast reader's grammar";
    return PDCS_IO_UNSUPPORTED;
  } catch (const Invalid& x) {
    g_io_err = std::string("invalid JSON: ") + x.what + " at byte " + std::to_string(P.p - buf);
    return PDCS_IO_ERROR;
  }
  // integer arrays must be integral (numpy would truncate; let Python decide)
  for (const char* k : {"G.rows", "G.cols", "socG", "rsocG"}) {
    auto it = D.arrays.find(k);
    if (it == D.arrays.end()) continue;
    Arr& a = it->second;
    if (!a.is_int) {
      g_io_err = "non-integral index array";
      return PDCS_IO_UNSUPPORTED;
    }
    a.i.resize(a.f.size());
    for (size_t j = 0; j < a.f.size(); ++j) a.i[j] = (int64_t)a.f[j];
    std::vector<double>().swap(a.f);
  }
  return PDCS_IO_OK;
}

}  // namespace

struct PdcsDoc : public Doc {};

extern "C" {

const char* pdcs_io_error(void) { return g_io_err.c_str(); }

int pdcs_io_parse_file(const char* path, int32_t nthreads, PdcsDoc** out) {
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    g_io_err = std::string("cannot open ") + path;
    return PDCS_IO_ERROR;
  }
  struct stat st;
  if (fstat(fd, &st) != 0) {
    close(fd);
    g_io_err = "fstat failed";
    return PDCS_IO_ERROR;
  }
  const size_t len = (size_t)st.st_size;
  void* map = len ? mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0) : nullptr;
  close(fd);
  if (len && map == MAP_FAILED) {
    g_io_err = "mmap failed";
    return PDCS_IO_ERROR;
  }
  if (len) madvise(map, len, MADV_SEQUENTIAL);
  if (nthreads < 1) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  PdcsDoc* D = new PdcsDoc();
  const int rc = parse(static_cast<const char*>(map), len, *D, nthreads);
  if (len) munmap(map, len);
  if (rc != PDCS_IO_OK) {
    delete D;
    return rc;
  }
  *out = D;
  return PDCS_IO_OK;
}

// Number of top-level keys; key(i) is the i-th key in document order.
int32_t pdcs_io_nkeys(const PdcsDoc* D) { return (int32_t)D->keys.size(); }
const char* pdcs_io_key(const PdcsDoc* D, int32_t i) { return D->keys[i].c_str(); }

// Numeric scalar: 1 and *out set when present.
int32_t pdcs_io_scalar(const PdcsDoc* D, const char* key, double* out) {
  auto it = D->scalars.find(key);
  if (it == D->scalars.end()) return 0;
  *out = it->second;
  return 1;
}

// Array length (-1 when absent); kind 0 = float64, 1 = int64.
int64_t pdcs_io_len(const PdcsDoc* D, const char* key, int32_t* kind) {
  auto it = D->arrays.find(key);
  if (it == D->arrays.end()) return -1;
  const Arr& a = it->second;
  const bool isint = !a.i.empty() || (a.f.empty() && a.is_int);
  if (kind) *kind = isint ? 1 : 0;
  return isint ? (int64_t)a.i.size() : (int64_t)a.f.size();
}

int32_t pdcs_io_copy(const PdcsDoc* D, const char* key, void* dst) {
  auto it = D->arrays.find(key);
  if (it == D->arrays.end()) return 1;
  const Arr& a = it->second;
  if (!a.i.empty()) std::memcpy(dst, a.i.data(), a.i.size() * sizeof(int64_t));
  else if (!a.f.empty()) std::memcpy(dst, a.f.data(), a.f.size() * sizeof(double));
  return 0;
}

void pdcs_io_free(PdcsDoc* D) { delete D; }

}  // extern "C"
