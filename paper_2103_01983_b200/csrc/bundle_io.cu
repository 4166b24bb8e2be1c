// bundle_io.cu — PTMX matrices and OfflineBundle directories in the
// reference's on-disk layout, host code of the C ABI:
//   ptrom_ptmx_read / ptrom_ptmx_write      io.hpp:23-75 (read_matrix / write_matrix)
//   ptrom_bundle_open / _sizes / _export    bundle.cpp:96-141 (OfflineBundle::load)
//   ptrom_bundle_to_device                  → ptrom_basis, ptrom_gnat_op, ptrom_surrogate
// None of this needs a GPU except ptrom_bundle_to_device. index.json is read
// with a small streaming JSON reader: only the keys the loader needs are
// materialised (the membership lists of a 1M-body bundle hold ~1e7 ids), the
// "config" object is kept verbatim.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

thread_local std::string g_io_error;

struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ PTMX --
constexpr char kMagic[4] = {'P', 'T', 'M', 'X'};
constexpr uint32_t kVersion = 1;

struct Mat {
  uint64_t rows = 0, cols = 0;
  double dt = 0, t0 = 0;
  std::vector<double> data;  // column-major
};

// io.hpp:53-75 (same messages)
Mat read_ptmx(const std::string& path, bool with_data = true) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw io_error("read_matrix: cannot open " + path);
  char magic[4] = {};
  uint32_t version = 0;
  Mat m;
  in.read(magic, 4);
  in.read(reinterpret_cast<char*>(&version), 4);
  in.read(reinterpret_cast<char*>(&m.rows), 8);
  in.read(reinterpret_cast<char*>(&m.cols), 8);
  in.read(reinterpret_cast<char*>(&m.dt), 8);
  in.read(reinterpret_cast<char*>(&m.t0), 8);
  if (!in || std::memcmp(magic, kMagic, 4) != 0) throw io_error("read_matrix: " + path + " is not a matrix file");
  if (version != kVersion) throw io_error("read_matrix: unsupported version " + std::to_string(version));
  if (with_data) {
    m.data.resize(m.rows * m.cols);
    in.read(reinterpret_cast<char*>(m.data.data()), (std::streamsize)(8 * m.data.size()));
    if (!in) throw io_error("read_matrix: truncated file " + path);
  }
  return m;
}

// io.hpp:35-51
void write_ptmx(const std::string& path, uint64_t rows, uint64_t cols, double dt, double t0, const double* data) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw io_error("write_matrix: cannot open " + path);
  out.write(kMagic, 4);
  out.write(reinterpret_cast<const char*>(&kVersion), 4);
  out.write(reinterpret_cast<const char*>(&rows), 8);
  out.write(reinterpret_cast<const char*>(&cols), 8);
  out.write(reinterpret_cast<const char*>(&dt), 8);
  out.write(reinterpret_cast<const char*>(&t0), 8);
  out.write(reinterpret_cast<const char*>(data), (std::streamsize)(8 * rows * cols));
  if (!out) throw io_error("write_matrix: write failed for " + path);
}

// bundle.cpp:15-19 read_vector
std::vector<double> read_vector(const std::string& path) {
  Mat m = read_ptmx(path);
  if (m.cols != 1) throw io_error(path + ": expected a single column");
  return std::move(m.data);
}

// ------------------------------------------------------ streaming JSON --
struct Json {
  const char* p;
  const char* end;
  std::string where;

  [[noreturn]] void fail(const std::string& what) const {
    throw io_error("load_json: " + where + ": " + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool peek(char c) {
    ws();
    return p < end && *p == c;
  }
  void expect(char c) {
    ws();
    if (p >= end || *p != c) fail(std::string("expected '") + c + "'");
    ++p;
  }
  std::string str() {
    expect('"');
    std::string s;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= end) break;
        const char e = *p;
        s += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e;
        if (e == 'u') p += 4;  // keys and format strings here are ASCII
      } else {
        s += *p;
      }
      ++p;
    }
    expect('"');
    return s;
  }
  unsigned long long uinteger() {  // training hashes are full 64-bit
    ws();
    if (p >= end || *p < '0' || *p > '9') fail("expected an unsigned integer");
    unsigned long long v = 0;
    while (p < end && *p >= '0' && *p <= '9') v = v * 10 + (unsigned)(*p++ - '0');
    return v;
  }
  long long integer() {
    ws();
    if (end - p >= 4 && std::strncmp(p, "true", 4) == 0) {
      p += 4;
      return 1;
    }
    if (end - p >= 5 && std::strncmp(p, "false", 5) == 0) {
      p += 5;
      return 0;
    }
    const char* q = p;
    bool neg = false;
    if (q < end && *q == '-') {
      neg = true;
      ++q;
    }
    if (q >= end || *q < '0' || *q > '9') fail("expected an integer");
    long long v = 0;
    while (q < end && *q >= '0' && *q <= '9') v = v * 10 + (*q++ - '0');
    if (q < end && (*q == '.' || *q == 'e' || *q == 'E')) {  // integral doubles (e.g. 3.0)
      char* stop = nullptr;
      const double d = std::strtod(p, &stop);
      if (d != (double)(long long)d) fail("expected an integer");
      p = stop;
      return (long long)d;
    }
    p = q;
    return neg ? -v : v;
  }
  // Skips one value and returns its text span.
  std::pair<const char*, const char*> skip() {
    ws();
    const char* b = p;
    if (p >= end) fail("unexpected end");
    if (*p == '"') {
      str();
    } else if (*p == '{' || *p == '[') {
      int depth = 0;
      bool in_str = false;
      for (; p < end; ++p) {
        const char c = *p;
        if (in_str) {
          if (c == '\\') ++p;
          else if (c == '"') in_str = false;
        } else if (c == '"') {
          in_str = true;
        } else if (c == '{' || c == '[') {
          ++depth;
        } else if (c == '}' || c == ']') {
          if (--depth == 0) {
            ++p;
            break;
          }
        }
      }
    } else {
      while (p < end && *p != ',' && *p != '}' && *p != ']' && *p != ' ' && *p != '\n' && *p != '\r' && *p != '\t')
        ++p;
    }
    return {b, p};
  }
  template <class F>
  void object(F&& on_key) {
    expect('{');
    if (peek('}')) {
      ++p;
      return;
    }
    while (true) {
      const std::string k = str();
      expect(':');
      on_key(k);
      if (peek(',')) {
        ++p;
        continue;
      }
      expect('}');
      return;
    }
  }
  template <class F>
  void array(F&& on_item) {
    expect('[');
    if (peek(']')) {
      ++p;
      return;
    }
    while (true) {
      on_item();
      if (peek(',')) {
        ++p;
        continue;
      }
      expect(']');
      return;
    }
  }
  template <class T>
  std::vector<T> ints() {
    std::vector<T> v;
    array([&] { v.push_back((T)integer()); });
    return v;
  }
  // nested int lists → CSR (bundle.cpp parse_nested)
  void nested(std::vector<int64_t>& off, std::vector<int64_t>& flat) {
    off.assign(1, 0);
    flat.clear();
    array([&] {
      array([&] { flat.push_back(integer()); });
      off.push_back((int64_t)flat.size());
    });
  }
};

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw io_error("load_json: cannot open " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

template <class F>
int io_guarded(ptrom_ctx* ctx, F&& fn) {
  try {
    fn();
    g_io_error.clear();
    if (ctx) ctx->err.clear();
    return PTROM_OK;
  } catch (const ptrom::status_error& e) {
    g_io_error = e.what();
    if (ctx) ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_io_error = e.what();
    if (ctx) ctx->err = e.what();
    return PTROM_CONFIG_ERROR;  // io / format errors are the reference's config_error
  }
}

}  // namespace

// bundle.hpp:15-27 OfflineBundle, host side.
struct ptrom_bundle {
  Mat basis_phi, residual_phi, gnat_a, phi_tilde, direct_phi;
  std::vector<double> basis_sv, basis_xref, residual_sv, x0_tilde, gamma_tilde, direct_x0, direct_gamma;
  std::vector<int64_t> sample_ids, target_ids, direct_ids;
  std::vector<int32_t> cluster_node_ids;
  std::vector<int64_t> mem_off, mem_ids, cl_off, cl_list, d_off, d_list;
  std::vector<uint8_t> zero_gamma;
  std::vector<uint64_t> training_hashes;
  std::string config_json;
};

extern "C" {

const char* ptrom_io_last_error(void) { return g_io_error.c_str(); }

int ptrom_ptmx_read(ptrom_ctx* ctx, const char* path, uint64_t* rows, uint64_t* cols, double* dt, double* t0,
                    double* data, uint64_t capacity) {
  return io_guarded(ctx, [&] {
    if (!path) throw io_error("read_matrix: null path");
    Mat m = read_ptmx(path, data != nullptr);
    if (rows) *rows = m.rows;
    if (cols) *cols = m.cols;
    if (dt) *dt = m.dt;
    if (t0) *t0 = m.t0;
    if (data) {
      if (capacity < m.rows * m.cols) throw io_error("read_matrix: output buffer too small for " + std::string(path));
      std::memcpy(data, m.data.data(), 8 * m.data.size());
    }
  });
}

int ptrom_ptmx_write(ptrom_ctx* ctx, const char* path, uint64_t rows, uint64_t cols, double dt, double t0,
                     const double* data) {
  return io_guarded(ctx, [&] {
    if (!path || (!data && rows != 0 && cols != 0)) throw io_error("write_matrix: null argument");
    write_ptmx(path, rows, cols, dt, t0, data);
  });
}

// bundle.cpp:96-141 (same files, keys and error messages)
int ptrom_bundle_open(ptrom_ctx* ctx, const char* dir, ptrom_bundle** out) {
  return io_guarded(ctx, [&] {
    if (!dir || !out) throw io_error("bundle_open: null argument");
    const std::string root(dir);
    auto j = [&](const char* f) { return root + "/" + f; };
    const std::string text = slurp(j("index.json"));
    Json js{text.data(), text.data() + text.size(), j("index.json")};
    auto* b = new ptrom_bundle;
    try {
      std::string format;
      bool got_sample = false, got_clusters = false, got_targets = false, got_direct = false, got_config = false;
      js.object([&](const std::string& k) {
        if (k == "format") {
          js.ws();
          if (js.peek('"')) format = js.str();
          else js.skip();
        } else if (k == "config") {
          auto sp = js.skip();
          b->config_json.assign(sp.first, sp.second);
          got_config = true;
        } else if (k == "sample_ids") {
          b->sample_ids = js.ints<int64_t>();
          got_sample = true;
        } else if (k == "clusters") {
          got_clusters = true;
          bool node = false, mem = false, zero = false;
          js.object([&](const std::string& c) {
            if (c == "node_ids") {
              b->cluster_node_ids = js.ints<int32_t>();
              node = true;
            } else if (c == "membership") {
              js.nested(b->mem_off, b->mem_ids);
              mem = true;
            } else if (c == "zero_gamma") {
              for (long long z : js.ints<long long>()) b->zero_gamma.push_back(z != 0 ? 1 : 0);
              zero = true;
            } else {
              js.skip();
            }
          });
          if (!node || !mem || !zero) throw io_error(root + ": bundle index is missing a clusters key");
        } else if (k == "targets") {
          got_targets = true;
          bool ids = false, cl = false, dl = false;
          js.object([&](const std::string& t) {
            if (t == "ids") {
              b->target_ids = js.ints<int64_t>();
              ids = true;
            } else if (t == "clusters") {
              js.nested(b->cl_off, b->cl_list);
              cl = true;
            } else if (t == "direct") {
              js.nested(b->d_off, b->d_list);
              dl = true;
            } else {
              js.skip();
            }
          });
          if (!ids || !cl || !dl) throw io_error(root + ": bundle index is missing a targets key");
        } else if (k == "direct_ids") {
          b->direct_ids = js.ints<int64_t>();
          got_direct = true;
        } else if (k == "training_hashes") {
          js.array([&] { b->training_hashes.push_back((uint64_t)js.uinteger()); });
        } else {
          js.skip();
        }
      });
      if (format != "ptrom-bundle") throw io_error(root + ": not a bundle directory");
      if (!got_sample || !got_clusters || !got_targets || !got_direct || !got_config)
        throw io_error(root + ": bundle index is missing a required key");
      b->basis_phi = read_ptmx(j("basis_phi.ptmx"));
      b->basis_sv = read_vector(j("basis_sv.ptmx"));
      b->basis_xref = read_vector(j("basis_xref.ptmx"));
      b->residual_phi = read_ptmx(j("residual_phi.ptmx"));
      b->residual_sv = read_vector(j("residual_sv.ptmx"));
      b->gnat_a = read_ptmx(j("gnat_a.ptmx"));
      b->phi_tilde = read_ptmx(j("surrogate_phi.ptmx"));
      b->x0_tilde = read_vector(j("surrogate_x0.ptmx"));
      b->gamma_tilde = read_vector(j("surrogate_gamma.ptmx"));
      b->direct_phi = read_ptmx(j("direct_phi.ptmx"));
      b->direct_x0 = read_vector(j("direct_x0.ptmx"));
      b->direct_gamma = read_vector(j("direct_gamma.ptmx"));
      // shape checks (the reference finds these later, in the solver ctors)
      const uint64_t nd = b->basis_phi.rows, m = b->basis_phi.cols, nc = b->gamma_tilde.size();
      if (nd % 2) throw io_error("bundle: state dimension must be even");
      if (b->basis_xref.size() != nd || b->basis_sv.size() != m) throw io_error("bundle: basis shape mismatch");
      if (b->phi_tilde.rows != 2 * nc || b->x0_tilde.size() != 2 * nc)
        throw io_error("bundle: surrogate table shape mismatch");
      if (b->mem_off.size() != nc + 1 || b->zero_gamma.size() != nc)
        throw io_error("bundle: cluster membership count mismatch");
      if (b->cl_off.size() != b->target_ids.size() + 1 || b->d_off.size() != b->target_ids.size() + 1)
        throw io_error("bundle: per-target list count mismatch");
      if (b->gnat_a.cols != 2 * b->sample_ids.size())
        throw io_error("bundle: GNAT operator does not match the sample count");
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
  });
}

void ptrom_bundle_free(ptrom_bundle* b) { delete b; }

// sizes[0..10]: n_dofs, modes, residual modes, n_samples, GNAT rows (m_r),
// n_clusters, n_direct, n_targets, membership entries, cluster-list entries,
// direct-list entries.
int ptrom_bundle_sizes(const ptrom_bundle* b, int64_t* sizes) {
  if (!b || !sizes) return PTROM_CONFIG_ERROR;
  sizes[0] = (int64_t)b->basis_phi.rows;
  sizes[1] = (int64_t)b->basis_phi.cols;
  sizes[2] = (int64_t)b->residual_phi.cols;
  sizes[3] = (int64_t)b->sample_ids.size();
  sizes[4] = (int64_t)b->gnat_a.rows;
  sizes[5] = (int64_t)b->gamma_tilde.size();
  sizes[6] = (int64_t)b->direct_ids.size();
  sizes[7] = (int64_t)b->target_ids.size();
  sizes[8] = (int64_t)b->mem_ids.size();
  sizes[9] = (int64_t)b->cl_list.size();
  sizes[10] = (int64_t)b->d_list.size();
  return PTROM_OK;
}

// The ExperimentConfig JSON kept verbatim (control plane out of scope):
// copies up to cap bytes (NUL-terminated) and returns the full length.
int64_t ptrom_bundle_config_json(const ptrom_bundle* b, char* buf, int64_t cap) {
  if (!b) return -1;
  if (buf && cap > 0) {
    const size_t k = std::min<size_t>((size_t)cap - 1, b->config_json.size());
    std::memcpy(buf, b->config_json.data(), k);
    buf[k] = 0;
  }
  return (int64_t)b->config_json.size();
}

// Host copies of the bundle's arrays (NULL pointers skipped); matrices are
// column-major as in the PTMX files.
int ptrom_bundle_export(const ptrom_bundle* b, double* basis_phi, double* basis_sv, double* basis_xref,
                        double* residual_phi, double* residual_sv, double* gnat_a, int64_t* sample_ids,
                        double* phi_tilde, double* x0_tilde, double* gamma_tilde, int32_t* cluster_node_ids,
                        int64_t* mem_off, int64_t* mem_ids, uint8_t* zero_gamma, int64_t* target_ids,
                        int64_t* cl_off, int64_t* cl_list, int64_t* d_off, int64_t* d_list, int64_t* direct_ids,
                        double* direct_phi, double* direct_x0, double* direct_gamma) {
  if (!b) return PTROM_CONFIG_ERROR;
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(basis_phi, b->basis_phi.data);
  cp(basis_sv, b->basis_sv);
  cp(basis_xref, b->basis_xref);
  cp(residual_phi, b->residual_phi.data);
  cp(residual_sv, b->residual_sv);
  cp(gnat_a, b->gnat_a.data);
  cp(sample_ids, b->sample_ids);
  cp(phi_tilde, b->phi_tilde.data);
  cp(x0_tilde, b->x0_tilde);
  cp(gamma_tilde, b->gamma_tilde);
  cp(cluster_node_ids, b->cluster_node_ids);
  cp(mem_off, b->mem_off);
  cp(mem_ids, b->mem_ids);
  cp(zero_gamma, b->zero_gamma);
  cp(target_ids, b->target_ids);
  cp(cl_off, b->cl_off);
  cp(cl_list, b->cl_list);
  cp(d_off, b->d_off);
  cp(d_list, b->d_list);
  cp(direct_ids, b->direct_ids);
  cp(direct_phi, b->direct_phi.data);
  cp(direct_x0, b->direct_x0);
  cp(direct_gamma, b->direct_gamma);
  return PTROM_OK;
}

// → the device objects GnatSolver / hyperpair consume (rom.hpp:264-290).
int ptrom_bundle_to_device(ptrom_ctx* ctx, const ptrom_bundle* b, ptrom_basis** basis, ptrom_gnat_op** op,
                           ptrom_surrogate** sur) {
  if (!ctx) return PTROM_CONFIG_ERROR;
  if (!b || !basis || !op || !sur) {
    ctx->err = "bundle_to_device: null argument";
    return PTROM_CONFIG_ERROR;
  }
  *basis = nullptr;
  *op = nullptr;
  *sur = nullptr;
  int rc = ptrom_basis_create(ctx, (int64_t)b->basis_phi.rows, (int64_t)b->basis_phi.cols, b->basis_phi.data.data(),
                              b->basis_sv.data(), b->basis_xref.data(), basis);
  if (rc == PTROM_OK)
    rc = ptrom_gnat_op_create(ctx, *basis, (int64_t)b->sample_ids.size(), b->sample_ids.data(),
                              (int64_t)b->gnat_a.rows, b->gnat_a.data.data(), op);
  if (rc == PTROM_OK)
    rc = ptrom_surrogate_create(ctx, (int64_t)b->phi_tilde.cols, (int64_t)b->gamma_tilde.size(),
                                b->phi_tilde.data.data(), b->gamma_tilde.data(), b->x0_tilde.data(),
                                b->zero_gamma.data(), b->mem_off.data(), b->mem_ids.data(),
                                (int64_t)b->target_ids.size(), b->target_ids.data(), b->cl_off.data(),
                                b->cl_list.data(), (int64_t)b->direct_ids.size(), b->direct_ids.data(),
                                b->direct_phi.data.data(), b->direct_x0.data(), b->direct_gamma.data(),
                                b->d_off.data(), b->d_list.data(), sur);
  if (rc != PTROM_OK) {
    ptrom_surrogate_free(*sur);
    ptrom_gnat_op_free(*op);
    ptrom_basis_free(*basis);
    *basis = nullptr;
    *op = nullptr;
    *sur = nullptr;
  }
  return rc;
}

}  // extern "C"
