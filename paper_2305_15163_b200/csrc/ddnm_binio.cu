// binio (the reference's language-neutral matrix format, binio.py:1-87) and
// the instance file that feeds a GPU context without Python.
//
// File layout (binio.py:1-8): 8-byte magic "DDNMROM1", then per record a
// little-endian u32 name length, the UTF-8 name, u64 rows, u64 cols and
// rows*cols little-endian float64 values in column-major order.  Readers
// raise FormatError (here DDNM_EFORMAT) on a bad magic, a truncated record or
// a record that overruns the file (binio.py:43-70).  Meta files are flat
// "key = value" text (binio.py:73-87).
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/ddnm.h"

namespace ddnm {
void set_error(const std::string& msg);   // ddnm_abi.cu
}

namespace {

int bfail(int code, const std::string& msg) {
  ddnm::set_error(msg);      // the ABI's error channel (ddnm_last_error)
  return code;
}

struct Record {
  std::string name;
  int64_t rows = 0, cols = 0;
  std::vector<double> data;       // column-major, as stored
};

}  // namespace

struct ddnm_binio {
  std::vector<Record> recs;
  std::map<std::string, size_t> index;
};

namespace {

int read_file(const char* path, std::vector<unsigned char>& raw) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return bfail(DDNM_EINVAL, std::string(path) + ": cannot open");
  f.seekg(0, std::ios::end);
  const std::streamoff n = f.tellg();
  f.seekg(0, std::ios::beg);
  raw.resize((size_t)n);
  if (n > 0 && !f.read(reinterpret_cast<char*>(raw.data()), n))
    return bfail(DDNM_EINVAL, std::string(path) + ": read failed");
  return 0;
}

template <typename T>
T le(const unsigned char* p) {          // little-endian decode (host-order independent)
  T v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= (T)p[i] << (8 * i);
  return v;
}

int parse(const char* path, const std::vector<unsigned char>& raw, ddnm_binio& out) {
  const char magic[8] = {'D', 'D', 'N', 'M', 'R', 'O', 'M', '1'};
  if (raw.size() < 8 || std::memcmp(raw.data(), magic, 8) != 0)
    return bfail(DDNM_EFORMAT, std::string(path) + ": bad magic");
  size_t pos = 8;
  auto need = [&](size_t n) { return pos + n <= raw.size(); };
  while (pos < raw.size()) {
    if (!need(4)) return bfail(DDNM_EFORMAT, std::string(path) + ": truncated at byte " + std::to_string(pos));
    const uint32_t nlen = le<uint32_t>(raw.data() + pos);
    pos += 4;
    if (!need(nlen)) return bfail(DDNM_EFORMAT, std::string(path) + ": truncated at byte " + std::to_string(pos));
    Record r;
    r.name.assign(reinterpret_cast<const char*>(raw.data() + pos), nlen);
    pos += nlen;
    if (!need(16)) return bfail(DDNM_EFORMAT, std::string(path) + ": truncated at byte " + std::to_string(pos));
    const uint64_t rows = le<uint64_t>(raw.data() + pos), cols = le<uint64_t>(raw.data() + pos + 8);
    pos += 16;
    const uint64_t avail = (raw.size() - pos) / 8;
    // rows * cols > avail without overflowing (binio.py:63-64)
    if (rows != 0 && cols > avail / rows)
      return bfail(DDNM_EFORMAT, std::string(path) + ": record '" + r.name + "' overruns file");
    r.rows = (int64_t)rows;
    r.cols = (int64_t)cols;
    const size_t n = (size_t)(rows * cols);
    r.data.resize(n);
    for (size_t i = 0; i < n; ++i) {
      const uint64_t bits = le<uint64_t>(raw.data() + pos + 8 * i);
      std::memcpy(&r.data[i], &bits, 8);
    }
    pos += 8 * n;
    out.index[r.name] = out.recs.size();   // a repeated name keeps the last (dict semantics)
    out.recs.push_back(std::move(r));
  }
  return 0;
}

void put_u32(std::string& s, uint32_t v) {
  for (int i = 0; i < 4; ++i) s.push_back((char)((v >> (8 * i)) & 0xff));
}
void put_u64(std::string& s, uint64_t v) {
  for (int i = 0; i < 8; ++i) s.push_back((char)((v >> (8 * i)) & 0xff));
}

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && std::isspace((unsigned char)s[a])) ++a;
  while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

int read_meta(const std::string& path, std::map<std::string, std::string>& out) {
  std::ifstream f(path);
  if (!f) return bfail(DDNM_EINVAL, path + ": cannot open");
  std::string line;
  int lineno = 0;
  while (std::getline(f, line)) {
    ++lineno;
    line = trim(line);
    if (line.empty() || line[0] == '#') continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos)
      return bfail(DDNM_EFORMAT, path + ":" + std::to_string(lineno) + ": expected 'key = value'");
    out[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
  }
  return 0;
}

}  // namespace

extern "C" {

int ddnm_binio_read(const char* path, ddnm_binio** out) {
  if (!path || !out) return bfail(DDNM_EINVAL, "null argument");
  *out = nullptr;
  std::vector<unsigned char> raw;
  int rc = read_file(path, raw);
  if (rc) return rc;
  auto* b = new ddnm_binio();
  if ((rc = parse(path, raw, *b))) {
    delete b;
    return rc;
  }
  *out = b;
  return 0;
}

int ddnm_binio_count(const ddnm_binio* b, int64_t* n) {
  if (!b || !n) return bfail(DDNM_EINVAL, "null argument");
  *n = (int64_t)b->recs.size();
  return 0;
}

int ddnm_binio_entry(const ddnm_binio* b, int64_t i, const char** name, int64_t* name_len,
                     int64_t* rows, int64_t* cols, const double** data) {
  if (!b || i < 0 || i >= (int64_t)b->recs.size()) return bfail(DDNM_EINVAL, "record index out of range");
  const Record& r = b->recs[(size_t)i];
  if (name) *name = r.name.data();
  if (name_len) *name_len = (int64_t)r.name.size();   // names may hold NUL bytes
  if (rows) *rows = r.rows;
  if (cols) *cols = r.cols;
  if (data) *data = r.data.data();
  return 0;
}

int ddnm_binio_find(const ddnm_binio* b, const char* name, int64_t* rows, int64_t* cols,
                    const double** data) {
  if (!b || !name) return bfail(DDNM_EINVAL, "null argument");
  auto it = b->index.find(name);
  if (it == b->index.end()) return bfail(DDNM_EINVAL, std::string("no record '") + name + "'");
  return ddnm_binio_entry(b, (int64_t)it->second, nullptr, nullptr, rows, cols, data);
}

int ddnm_binio_free(ddnm_binio* b) {
  delete b;
  return 0;
}

int ddnm_binio_write(const char* path, int64_t n, const char* const* names,
                     const int64_t* name_lens, const int64_t* rows, const int64_t* cols,
                     const double* const* data) {
  if (!path || (n > 0 && (!names || !rows || !cols || !data))) return bfail(DDNM_EINVAL, "null argument");
  std::string s("DDNMROM1", 8);
  for (int64_t k = 0; k < n; ++k) {
    if (rows[k] < 0 || cols[k] < 0) return bfail(DDNM_EINVAL, "negative matrix dimension");
    const size_t nl = name_lens ? (size_t)name_lens[k] : std::strlen(names[k]);
    put_u32(s, (uint32_t)nl);
    s.append(names[k], nl);
    put_u64(s, (uint64_t)rows[k]);
    put_u64(s, (uint64_t)cols[k]);
    const size_t cnt = (size_t)(rows[k] * cols[k]);
    for (size_t i = 0; i < cnt; ++i) {
      uint64_t bits;
      std::memcpy(&bits, data[k] + i, 8);
      put_u64(s, bits);
    }
  }
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f || !f.write(s.data(), (std::streamsize)s.size())) return bfail(DDNM_EINVAL, std::string(path) + ": write failed");
  return 0;
}

// ---- instance files ----------------------------------------------------------

namespace {

struct Inst {
  const ddnm_binio* b;
  std::vector<std::vector<double>> dkeep;     // row-major copies
  std::vector<std::vector<int64_t>> ikeep;
  std::string err;

  const Record* rec(const std::string& name) const {
    auto it = b->index.find(name);
    return it == b->index.end() ? nullptr : &b->recs[it->second];
  }
  // row-major double array of a record (binio stores column-major)
  const double* f(const std::string& name, int64_t* n = nullptr, int64_t* rows = nullptr) {
    const Record* r = rec(name);
    if (!r) { err = "instance file has no record '" + name + "'"; return nullptr; }
    std::vector<double> v((size_t)(r->rows * r->cols));
    for (int64_t i = 0; i < r->rows; ++i)
      for (int64_t j = 0; j < r->cols; ++j) v[(size_t)(i * r->cols + j)] = r->data[(size_t)(j * r->rows + i)];
    if (n) *n = r->rows * r->cols;
    if (rows) *rows = r->rows;
    dkeep.push_back(std::move(v));
    return dkeep.back().data();
  }
  const int64_t* i64(const std::string& name, int64_t* n = nullptr) {
    const Record* r = rec(name);
    if (!r) { err = "instance file has no record '" + name + "'"; return nullptr; }
    std::vector<int64_t> v((size_t)(r->rows * r->cols));
    for (int64_t i = 0; i < r->rows; ++i)
      for (int64_t j = 0; j < r->cols; ++j) v[(size_t)(i * r->cols + j)] = (int64_t)r->data[(size_t)(j * r->rows + i)];
    if (n) *n = r->rows * r->cols;
    ikeep.push_back(std::move(v));
    return ikeep.back().data();
  }
  bool fill_decoder(ddnm_decoder& d, const std::string& pre, bool nm) {
    std::memset(&d, 0, sizeof d);
    int64_t n = 0, rows = 0;
    if (nm) {
      if (!(d.scale = f(pre + "scale", &n))) return false;
      d.n_out = (int32_t)n;
      if (!(d.b1 = f(pre + "b1", &n))) return false;
      d.n_hidden = (int32_t)n;
      if (!(d.W1 = f(pre + "W1")) || !(d.indptr = i64(pre + "W2_indptr")) ||
          !(d.indices = i64(pre + "W2_indices")) || !(d.data = f(pre + "W2_data")) ||
          !(d.shift = f(pre + "shift")))
        return false;
    } else {
      if (!(d.W1 = f(pre + "Phi", &n, &rows))) return false;
      d.n_out = (int32_t)rows;
    }
    return true;
  }
};

std::vector<int> int_list(const std::string& v) {
  std::vector<int> out;
  std::stringstream ss(v);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    tok = trim(tok);
    if (!tok.empty()) out.push_back(std::atoi(tok.c_str()));
  }
  return out;
}

}  // namespace

int ddnm_ctx_create_binio(int32_t device, const char* path, int32_t slots, ddnm_ctx** out) {
  if (!path || !out) return bfail(DDNM_EINVAL, "null argument");
  *out = nullptr;
  std::string mp(path);
  const size_t dot = mp.rfind('.');
  mp = (dot == std::string::npos ? mp : mp.substr(0, dot)) + ".txt";
  std::map<std::string, std::string> meta;
  int rc = read_meta(mp, meta);
  if (rc) return rc;
  if (meta["format"] != "ddnm-instance-1") return bfail(DDNM_EFORMAT, mp + ": not a ddnm-instance-1 meta file");
  ddnm_binio* b = nullptr;
  if ((rc = ddnm_binio_read(path, &b))) return rc;
  Inst I;
  I.b = b;
  const bool nm = meta["kind"] == "nm";
  const bool srpc = meta["constraint"] == "srpc";
  const int nb = std::atoi(meta["nblocks"].c_str());
  const std::vector<int> ni = int_list(meta["n_int"]), ng = int_list(meta["n_gam"]);
  if (nb < 1 || (int)ni.size() != nb || (int)ng.size() != nb) {
    ddnm_binio_free(b);
    return bfail(DDNM_EFORMAT, mp + ": inconsistent block counts");
  }
  std::vector<ddnm_block> blocks(nb);
  std::vector<ddnm_decoder> full(nb), gfull(nb);
  bool ok = true, has_full = I.rec("b0_int_cols") != nullptr;
  for (int k = 0; k < nb && ok; ++k) {
    const std::string p = "b" + std::to_string(k) + "_";
    ddnm_block& B = blocks[k];
    std::memset(&B, 0, sizeof B);
    B.n_int = ni[k];
    B.n_gam = ng[k];
    ok = I.fill_decoder(B.interior, p + "int_", nm) && I.fill_decoder(B.interface, p + "gam_", nm);
    int64_t n = 0;
    if (ok && (B.res_rows = I.i64(p + "res_rows", &n))) B.n_rows = (int32_t)n; else ok = false;
    if (ok && (B.cols = I.i64(p + "cols", &n))) B.n_cols = (int32_t)n; else ok = false;
    const int64_t* io = ok ? I.i64(p + "io", &n) : nullptr;
    if (io) B.n_io = (int32_t)n; else ok = false;
    if (ok && (B.gio = I.i64(p + "gio", &n))) B.n_gio = (int32_t)n; else ok = false;
    if (ok && srpc) {
      // the interface decoder is the restriction to gio (driver.py:400-402)
      std::vector<int64_t> g(B.n_gio);
      for (int i = 0; i < B.n_gio; ++i) g[i] = i;
      I.ikeep.push_back(std::move(g));
      B.gio = I.ikeep.back().data();
    }
    if (ok && !(B.CA = I.f(p + (srpc ? "Ahat" : "CA")))) ok = false;
    int64_t wr = 0;
    if (ok && I.rec(p + "weights")) {
      B.weights = I.f(p + "weights", &n, &wr);
      B.n_basis = (int32_t)wr;
    }
    if (ok && has_full) {
      ok = I.fill_decoder(full[k], p + "intf_", nm);
      if (ok && srpc) ok = I.fill_decoder(gfull[k], p + "gamf_", nm);
    }
  }
  ddnm_artifacts a;
  std::memset(&a, 0, sizeof a);
  if (ok) {
    a.abi_version = DDNM_ABI_VERSION;
    a.map_kind = nm ? DDNM_MAP_AUTOENCODER : DDNM_MAP_LINEAR;
    a.activation = meta["activation"] == "sigmoid" ? DDNM_ACT_SIGMOID : DDNM_ACT_SWISH;
    a.gam_activation = meta["gam_activation"] == "sigmoid" ? DDNM_ACT_SIGMOID : DDNM_ACT_SWISH;
    a.constraint_mode = srpc ? DDNM_CON_SRPC : DDNM_CON_WFPC;
    a.nx = std::atoi(meta["nx"].c_str());
    a.ny = std::atoi(meta["ny"].c_str());
    a.nu = std::atof(meta["nu"].c_str());
    a.n_blocks = nb;
    a.n_c = std::atoi(meta["n_c"].c_str());
    a.blocks = blocks.data();
    if (I.rec("rbf_coeffs")) {
      if (meta["rbf_kernel"] != "thin_plate_spline") {
        ddnm_binio_free(b);
        return bfail(DDNM_EUNSUPPORTED, "only thin-plate-spline RBF initializers");
      }
      int64_t n = 0, rows = 0;
      a.rbf.y = I.f("rbf_y", &n, &rows);
      a.rbf.n_centers = (int32_t)rows;
      a.rbf.coeffs = I.f("rbf_coeffs");
      const int64_t* pw = I.i64("rbf_powers", &n);
      a.rbf.powers = pw;
      a.rbf.n_mono = (int32_t)(n / 2);
      const double* sh = I.f("rbf_shift");
      const double* sc = I.f("rbf_scale");
      const double* lo = I.f("rbf_lo");
      const double* hi = I.f("rbf_hi");
      ok = a.rbf.y && a.rbf.coeffs && pw && sh && sc && lo && hi;
      if (ok)
        for (int k = 0; k < 2; ++k) {
          a.rbf.shift[k] = sh[k]; a.rbf.scale[k] = sc[k]; a.rbf.lo[k] = lo[k]; a.rbf.hi[k] = hi[k];
        }
      a.rbf.epsilon = meta.count("rbf_epsilon") ? std::atof(meta["rbf_epsilon"].c_str()) : 1.0;
    }
  }
  if (!ok) {
    const std::string e = I.err;
    ddnm_binio_free(b);
    return bfail(DDNM_EFORMAT, std::string(path) + ": " + e);
  }
  ddnm_ctx* ctx = nullptr;
  rc = ddnm_ctx_create(device, &a, slots, &ctx);
  if (rc == 0 && has_full) {
    rc = ddnm_ctx_set_full_decoders(ctx, full.data(), srpc ? gfull.data() : nullptr);
    if (rc) ddnm_ctx_destroy(ctx);
  }
  ddnm_binio_free(b);
  if (rc) return bfail(rc, ddnm_last_error());
  *out = ctx;
  return 0;
}

}  // extern "C"
