// Row f2: the reference's on-disk image format (include/voxellate/image_io.hpp:
// 17-29, src/image_io.cpp:20-50,164-202): a raw little-endian payload -- labels
// as u32, distances as IEEE-754 f64, voxel order axis 0 fastest -- plus a JSON
// sidecar at `<path>.json` with format_version, type, d, dims, lengths,
// boundary, kind, n_sites, seed and payload_bytes.
//
// Host code only.  The sidecar text reproduces, byte for byte, what the
// reference library writes when built here (nlohmann::json::dump(2) with its
// keys in sorted order; that json.hpp prints integer arrays on one line and
// other arrays one element per line; numbers in shortest round-trip form with
// nlohmann's fixed/exponent rule).  Reading applies the reference's checks in
// its order and with its messages (image_io.cpp:52-102,177-202).
// vx_tessellate_to_files (capi.cu) streams the payload out of device memory
// chunk by chunk with the helpers at the bottom.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <thread>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "voxellate_b200.h"
#include "vx_internal.cuh"

namespace vxb {
namespace io {

// ---- number formatting (nlohmann::detail::dtoa_impl::format_buffer rules) ----
std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  // shortest round-trip digits in scientific form: d[.ddd]e[+-]X
  auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const size_t epos = sci.find('e');
  std::string mant = sci.substr(0, epos);
  const int e10 = std::atoi(sci.c_str() + epos + 1);
  std::string digits;
  for (char c : mant)
    if (c != '.') digits.push_back(c);
  const int k = (int)digits.size();
  const int n = e10 + 1;  // value = 0.d1..dk * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  std::string out;
  if (k <= n && n <= kMaxExp) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= kMaxExp) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (kMinExp < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return sign + out;
}

const char* kind_name(int kind) {  // geometry.cpp:23-29
  return kind == VX_VORONOI ? "voronoi" : (kind == VX_JOHNSON_MEHL ? "johnson-mehl" : "laguerre");
}

std::string sidecar_text(const char* type, int dim, const int64_t* counts, const double* lengths,
                         int periodic, int kind, int64_t n_sites, int64_t seed, uint64_t payload_bytes) {
  std::string s = "{\n";
  s += "  \"boundary\": \"" + std::string(periodic ? "periodic" : "non-periodic") + "\",\n";
  s += "  \"d\": " + std::to_string(dim) + ",\n";
  s += "  \"dims\": [";
  for (int i = 0; i < dim; ++i) s += (i ? "," : "") + std::to_string(counts[i]);
  s += "],\n";
  s += "  \"format_version\": 1,\n";
  s += "  \"kind\": \"" + std::string(kind_name(kind)) + "\",\n";
  s += "  \"lengths\": [\n";
  for (int i = 0; i < dim; ++i) s += "    " + format_double(lengths[i]) + (i + 1 < dim ? ",\n" : "\n");
  s += "  ],\n";
  s += "  \"n_sites\": " + std::to_string(n_sites) + ",\n";
  s += "  \"payload_bytes\": " + std::to_string(payload_bytes) + ",\n";
  s += "  \"seed\": " + std::to_string(seed) + ",\n";
  s += "  \"type\": \"" + std::string(type) + "\"\n";
  s += "}\n";
  return s;
}

// ---- a minimal JSON reader for the sidecar schema ----
struct JVal {
  enum T { Null, Bool, Num, Str, Arr, Obj } t = Null;
  double num = 0;
  bool is_int = false;
  long long inum = 0;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct JParser {
  const char* p;
  const char* e;
  std::string err;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool fail(const std::string& m) {
    if (err.empty()) err = m;
    return false;
  }
  bool str(std::string& out) {
    if (p >= e || *p != '"') return fail("expected string");
    ++p;
    while (p < e && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= e) return fail("bad escape");
        const char c = *p;
        out.push_back(c == 'n' ? '\n' : c == 't' ? '\t' : c == 'r' ? '\r' : c == 'b' ? '\b' : c == 'f' ? '\f' : c);
      } else {
        out.push_back(*p);
      }
      ++p;
    }
    if (p >= e) return fail("unterminated string");
    ++p;
    return true;
  }
  bool val(JVal& v) {
    ws();
    if (p >= e) return fail("unexpected end of input");
    if (*p == '{') {
      v.t = JVal::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        std::string k;
        if (!str(k)) return false;
        ws();
        if (p >= e || *p != ':') return fail("expected ':'");
        ++p;
        JVal x;
        if (!val(x)) return false;
        v.obj[k] = std::move(x);
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return true;
        }
        return fail("expected ',' or '}'");
      }
    }
    if (*p == '[') {
      v.t = JVal::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return true;
      }
      for (;;) {
        JVal x;
        if (!val(x)) return false;
        v.arr.push_back(std::move(x));
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return true;
        }
        return fail("expected ',' or ']'");
      }
    }
    if (*p == '"') {
      v.t = JVal::Str;
      return str(v.str);
    }
    if (e - p >= 4 && !std::strncmp(p, "null", 4)) {
      p += 4;
      v.t = JVal::Null;
      return true;
    }
    if (e - p >= 4 && !std::strncmp(p, "true", 4)) {
      p += 4;
      v.t = JVal::Bool;
      v.num = 1;
      return true;
    }
    if (e - p >= 5 && !std::strncmp(p, "false", 5)) {
      p += 5;
      v.t = JVal::Bool;
      return true;
    }
    const char* s0 = p;
    bool frac = false;
    if (p < e && (*p == '-' || *p == '+')) ++p;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+')) {
      if (*p == '.' || *p == 'e' || *p == 'E') frac = true;
      ++p;
    }
    if (p == s0) return fail("syntax error");
    const std::string tok(s0, p);
    v.t = JVal::Num;
    v.num = std::strtod(tok.c_str(), nullptr);
    v.is_int = !frac;
    if (!frac) v.inum = std::strtoll(tok.c_str(), nullptr, 10);
    return true;
  }
};

struct Header {
  int dim = 0;
  int64_t counts[VX_MAX_DIM] = {};
  double lengths[VX_MAX_DIM] = {};
  int periodic = 0;
  int kind = 0;
  int64_t n_sites = 0;
  int64_t seed = -1;
  int format_version = 0;
  uint64_t payload_bytes = 0;
};

int io_fail(int code, const std::string& m) {
  set_last_error(m);  // capi.cu: vx_last_error()
  return code;
}

// read_sidecar, image_io.cpp:52-86
int read_sidecar(const std::string& path, const char* expected_type, Header& h) {
  FILE* f = std::fopen((path + ".json").c_str(), "rb");
  if (!f) return io_fail(VX_EIO, "cannot open image sidecar: " + path + ".json");
  std::string text;
  char buf[4096];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, got);
  std::fclose(f);
  JParser P{text.data(), text.data() + text.size(), {}};
  JVal root;
  bool ok = P.val(root);
  if (ok) {
    P.ws();
    if (P.p != P.e) ok = P.fail("unexpected trailing input");
  }
  if (!ok) return io_fail(VX_EIO, "malformed image sidecar " + path + ".json: " + P.err);
  if (root.t != JVal::Obj) return io_fail(VX_EIO, "image sidecar " + path + ".json missing fields: not an object");
  auto need = [&](const char* k) -> const JVal* {
    auto it = root.obj.find(k);
    return it == root.obj.end() ? nullptr : &it->second;
  };
  const char* keys[] = {"format_version", "type", "kind", "n_sites", "dims", "lengths", "boundary", "payload_bytes"};
  for (const char* k : keys)
    if (!need(k))
      return io_fail(VX_EIO, "image sidecar " + path + ".json missing fields: [json.exception.out_of_range.403] key '" +
                                 k + "' not found");
  const JVal* fv = need("format_version");
  const JVal* ty = need("type");
  const JVal* kd = need("kind");
  const JVal* ns = need("n_sites");
  const JVal* dm = need("dims");
  const JVal* ln = need("lengths");
  const JVal* bd = need("boundary");
  const JVal* pb = need("payload_bytes");
  if (fv->t != JVal::Num || ty->t != JVal::Str || kd->t != JVal::Str || ns->t != JVal::Num || dm->t != JVal::Arr ||
      ln->t != JVal::Arr || bd->t != JVal::Str || pb->t != JVal::Num)
    return io_fail(VX_EIO, "image sidecar " + path + ".json missing fields: type mismatch");
  const std::string kname = kd->str;
  if (kname == "voronoi") h.kind = VX_VORONOI;
  else if (kname == "johnson-mehl" || kname == "johnsonmehl" || kname == "jm") h.kind = VX_JOHNSON_MEHL;
  else if (kname == "laguerre") h.kind = VX_LAGUERRE;
  else return io_fail(VX_EINVAL, "unknown tessellation kind: " + kname);  // kind_from_string
  h.format_version = (int)fv->num;
  h.n_sites = ns->is_int ? ns->inum : (int64_t)ns->num;
  auto sd = root.obj.find("seed");
  h.seed = sd != root.obj.end() && sd->second.t == JVal::Num ? (sd->second.is_int ? sd->second.inum : (int64_t)sd->second.num) : -1;
  if (dm->arr.size() != ln->arr.size() || dm->arr.empty() || dm->arr.size() > VX_MAX_DIM)
    return io_fail(VX_EINVAL, "domain and voxel counts must have the same dimension");
  h.dim = (int)dm->arr.size();
  for (int i = 0; i < h.dim; ++i) {
    h.counts[i] = dm->arr[i].is_int ? dm->arr[i].inum : (int64_t)dm->arr[i].num;
    h.lengths[i] = ln->arr[i].num;
  }
  if (bd->str == "periodic") h.periodic = 1;
  else if (bd->str == "non-periodic" || bd->str == "nonperiodic") h.periodic = 0;
  else return io_fail(VX_EINVAL, "unknown boundary: " + bd->str);
  h.payload_bytes = pb->is_int ? (uint64_t)pb->inum : (uint64_t)pb->num;
  if (h.format_version != 1) return io_fail(VX_EIO, "unsupported image format version in " + path + ".json");
  if (ty->str != expected_type)
    return io_fail(VX_EIO, "image " + path + " has type '" + ty->str + "', expected '" + expected_type + "'");
  return VX_OK;
}

}  // namespace io

// ---- payload streaming helpers used by vx_tessellate_to_files (capi.cu) ----
// The payload file is written with pwrite at explicit offsets (several host
// threads per large piece).  The host page-cache write, ~3.3 GB/s on the test
// box whether written by one thread, several, or through a shared mapping, is
// the bound of a streamed image; the D2H (~50 GB/s) hides behind it.
int io_open_payload(const char* path, int* fd) {
  *fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (*fd < 0) return io::io_fail(VX_EIO, std::string("cannot open image file for writing: ") + path);
  return VX_OK;
}
int io_write_payload_at(int fd, const char* path, const void* data, size_t bytes, int64_t offset) {
  const size_t kMinSlice = 8u << 20;
  const int nt = (int)std::max<size_t>(1, std::min<size_t>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())),
                                                         bytes / kMinSlice));
  std::vector<int> ok(nt, 1);
  auto work = [&](int t) {
    const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
    const char* src = static_cast<const char*>(data);
    size_t done = a;
    while (done < b) {
      const ssize_t w = ::pwrite(fd, src + done, b - done, (off_t)(offset + (int64_t)done));
      if (w <= 0) {
        ok[t] = 0;
        return;
      }
      done += (size_t)w;
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  for (int v : ok)
    if (!v) return io::io_fail(VX_EIO, std::string("failed writing image payload: ") + path);
  return VX_OK;
}
// pinned staging buffer -> caller's pageable memory, several threads (the
// destination's first-touch page faults parallelise across threads)
void io_copy_parallel(void* dst, const void* src, size_t bytes) {
  const size_t kMinSlice = 4u << 20;
  const int nt = (int)std::max<size_t>(1, std::min<size_t>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                         bytes / kMinSlice));
  auto work = [&](int t) {
    const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  };
  if (nt == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

int io_close_payload(int fd, const char* path) {
  if (::close(fd) != 0) return io::io_fail(VX_EIO, std::string("failed writing image payload: ") + path);
  return VX_OK;
}

}  // namespace vxb

using namespace vxb;

extern "C" {

int vx_image_sidecar_text(const char* type, int dim, const int64_t* counts, const double* lengths,
                          int periodic, int kind, int64_t n_sites, int64_t seed, uint64_t payload_bytes,
                          char* buf, int64_t cap) {
  if (!type || !counts || !lengths || dim < 1 || dim > VX_MAX_DIM) return VX_EINVAL;
  const std::string s = io::sidecar_text(type, dim, counts, lengths, periodic, kind, n_sites, seed, payload_bytes);
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>((size_t)cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return (int)s.size();
}

int vx_write_image_sidecar(const char* path, const char* type, int dim, const int64_t* counts,
                           const double* lengths, int periodic, int kind, int64_t n_sites, int64_t seed,
                           uint64_t payload_bytes) {
  if (!path || !type || !counts || !lengths || dim < 1 || dim > VX_MAX_DIM)
    return io::io_fail(VX_EINVAL, "invalid sidecar arguments");
  const std::string side = std::string(path) + ".json";
  FILE* f = std::fopen(side.c_str(), "wb");
  if (!f) return io::io_fail(VX_EIO, "cannot open sidecar for writing: " + side);
  const std::string s = io::sidecar_text(type, dim, counts, lengths, periodic, kind, n_sites, seed, payload_bytes);
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  if (std::fclose(f) != 0 || !ok) return io::io_fail(VX_EIO, "failed writing sidecar: " + side);
  return VX_OK;
}

// write_label_image / write_distance_image (image_io.cpp:164-175): payload, then sidecar
int vx_write_image(const char* path, int type, int dim, const int64_t* counts, const double* lengths,
                   int periodic, int kind, int64_t n_sites, int64_t seed, const void* data) {
  if (!path || !counts || !lengths || dim < 1 || dim > VX_MAX_DIM || (type != 0 && type != 1))
    return io::io_fail(VX_EINVAL, "invalid image arguments");
  uint64_t nv = 1;
  for (int i = 0; i < dim; ++i) nv *= (uint64_t)counts[i];
  const uint64_t bytes = nv * (type == 0 ? 4u : 8u);
  if (bytes && !data) return io::io_fail(VX_EINVAL, "image data must not be NULL");
  int fd = -1;
  int rc = io_open_payload(path, &fd);
  if (rc) return rc;
  rc = io_write_payload_at(fd, path, data, bytes, 0);
  const int rc2 = io_close_payload(fd, path);
  if (rc) return rc;
  if (rc2) return rc2;
  return vx_write_image_sidecar(path, type == 0 ? "labels" : "distances", dim, counts, lengths, periodic, kind,
                                n_sites, seed, bytes);
}

// read_label_image / read_distance_image (image_io.cpp:177-202).  header_out:
// [dim, periodic, kind, n_sites, seed, format_version]; counts/lengths: VX_MAX_DIM
// entries; data (may be NULL: header only) receives voxel_count elements when
// cap_voxels is large enough.
int vx_read_image(const char* path, int type, int64_t* header_out, int64_t* counts_out, double* lengths_out,
                  void* data, int64_t cap_voxels) {
  if (!path || (type != 0 && type != 1)) return io::io_fail(VX_EINVAL, "invalid image arguments");
  io::Header h;
  const std::string p(path);
  int rc = io::read_sidecar(p, type == 0 ? "labels" : "distances", h);
  if (rc) return rc;
  uint64_t nv = 1;
  for (int i = 0; i < h.dim; ++i) nv *= (uint64_t)h.counts[i];
  const uint64_t expected = nv * (type == 0 ? 4u : 8u);
  if (h.payload_bytes != expected)
    return io::io_fail(VX_EIO, "image sidecar " + p + ".json payload size disagrees with dims");
  if (header_out) {
    header_out[0] = h.dim;
    header_out[1] = h.periodic;
    header_out[2] = h.kind;
    header_out[3] = h.n_sites;
    header_out[4] = h.seed;
    header_out[5] = h.format_version;
  }
  for (int i = 0; i < h.dim; ++i) {
    if (counts_out) counts_out[i] = h.counts[i];
    if (lengths_out) lengths_out[i] = h.lengths[i];
  }
  FILE* f = std::fopen(path, "rb");
  if (!f) return io::io_fail(VX_EIO, "cannot open image file: " + p);
  std::fseek(f, 0, SEEK_END);
  const long long actual = std::ftell(f);
  if (actual < 0 || (uint64_t)actual != expected) {
    std::fclose(f);
    return io::io_fail(VX_EIO, "image " + p + " payload is " + std::to_string(actual) + " bytes, header expects " +
                                   std::to_string(expected));
  }
  if (data && (int64_t)nv <= cap_voxels) {
    std::fseek(f, 0, SEEK_SET);
    const bool ok = std::fread(data, 1, expected, f) == expected;
    std::fclose(f);
    if (!ok) return io::io_fail(VX_EIO, "failed reading image payload: " + p);
  } else {
    std::fclose(f);
  }
  return VX_OK;
}

}  // extern "C"
