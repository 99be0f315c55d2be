// Data ingestion and synthetic generation.
//
//  * CTF1 tensor files, byte-exact with the reference (write_tensor /
//    read_tensor, io.cpp:30-77): "CTF1", u8 order, order x u64 LE dims, fp64
//    LE row-major payload.  Reads stream the payload straight into device
//    memory in 32 MiB chunks through a pinned staging buffer (fp64 -> fp32
//    conversion on the device), so a 16 GiB C5 tensor never needs a host
//    copy of itself.  Writes go the other way.
//  * COO text (read_coo, io.cpp:87-142) parsed into nonzeros for the sparse
//    path instead of being densified; same header/line grammar, same
//    line-numbered messages.
//  * trace CSV (write_trace, io.cpp:154-164): "iter,time_s,loss", %.17g.
//  * A counter-based generator for the BASELINE configs (new -- the
//    reference generators are noiseless, io.cpp:245-260): Philox4x32-10 keyed
//    by (seed, stream), uniforms (w >> 11) * 2^-53 like Rng::uniform01
//    (io.cpp:197-199), Gamma(k, theta) for integer k as theta * sum of k
//    -log1p(-U).  Any slab of X is generated in place on the device and
//    agrees with the host restatement (oracle/ntf_oracle.py, philox_*).
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "cp_kernels.cuh"
#include "engine.cuh"

namespace ntfg {

// ---- Philox4x32-10 ----------------------------------------------------------------
struct Philox {
  __host__ __device__ static inline void round(uint32_t (&c)[4], uint32_t (&k)[2]) {
    const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
    const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
    const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
    const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
    const uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
  // block `ctr` of stream `stream` under key `seed` -> two 64-bit words
  __host__ __device__ static inline void block(uint64_t seed, uint64_t stream, uint64_t ctr, uint64_t& w0,
                                               uint64_t& w1) {
    uint32_t c[4] = {uint32_t(ctr), uint32_t(ctr >> 32), uint32_t(stream), uint32_t(stream >> 32)};
    uint32_t k[2] = {uint32_t(seed), uint32_t(seed >> 32)};
    for (int r = 0; r < 10; ++r) round(c, k);
    w0 = (uint64_t(c[1]) << 32) | c[0];
    w1 = (uint64_t(c[3]) << 32) | c[2];
  }
  // uniform #j of (seed, stream) in [0, 1), 53 bits
  __host__ __device__ static inline double uniform(uint64_t seed, uint64_t stream, uint64_t j) {
    uint64_t w0, w1;
    block(seed, stream, j >> 1, w0, w1);
    return double(((j & 1) ? w1 : w0) >> 11) * 0x1.0p-53;
  }
};

constexpr uint64_t kStreamTruth = 1, kStreamInit = 2, kStreamNoise = 3;

// X(e) = CP(truth)(e) * Gamma(k, theta)(e) for the rows [row0, row1) of mode 0
template <typename T>
static __global__ void gen_cp_gamma_kernel(Geom g, int R, int64_t base, int64_t n, uint64_t seed, int k,
                                           double theta, T* out, const double* t0, const double* t1,
                                           const double* t2, const double* t3, const double* t4,
                                           const double* t5, const double* t6, const double* t7) {
  const double* tr[kMaxOrder] = {t0, t1, t2, t3, t4, t5, t6, t7};
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n; l += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = base + l;  // global linear (row-major) index
    int64_t idx[kMaxOrder];
    int64_t rem = e;
    for (int m = g.order - 1; m >= 0; --m) {
      idx[m] = rem % g.dims[m];
      rem /= g.dims[m];
    }
    double xh = 0.0;  // cp_reconstruct order: sum over r of prod over ascending m
    for (int r = 0; r < R; ++r) {
      double p = 1.0;
      for (int m = 0; m < g.order; ++m) p *= tr[m][idx[m] * R + r];
      xh += p;
    }
    double gs = 0.0;
    for (int i = 0; i < k; ++i) gs -= log1p(-Philox::uniform(seed, kStreamNoise, uint64_t(e) * k + i));
    out[l] = T(xh * (theta * gs));
  }
}

namespace {

void put_u64le(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}
uint64_t get_u64le(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}
bool little_endian() {
  const uint16_t one = 1;
  return *reinterpret_cast<const unsigned char*>(&one) == 1;
}

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() { if (f) std::fclose(f); }
};

constexpr size_t kChunk = size_t(4) << 20;  // doubles per staging chunk (32 MiB)

}  // namespace

// ---- CTF1 --------------------------------------------------------------------------
struct Ctf1Header {
  std::vector<uint64_t> dims;
  uint64_t entries = 1;
  long payload = 0;
};

static Ctf1Header ctf1_header(const char* path, uint64_t max_entries, File& f) {
  if (!f.f) throw Error(NTFG_ERR_FORMAT, std::string("cannot open: ") + path);
  unsigned char head[5];
  if (std::fread(head, 1, 5, f.f) != 5 || std::memcmp(head, "CTF1", 4) != 0)
    throw Error(NTFG_ERR_FORMAT, std::string("bad magic: not a CTF1 tensor file: ") + path);
  const size_t order = head[4];
  if (order == 0) throw Error(NTFG_ERR_FORMAT, "CTF1: zero tensor order");
  std::vector<unsigned char> d(8 * order);
  if (std::fread(d.data(), 1, d.size(), f.f) != d.size()) throw Error(NTFG_ERR_FORMAT, "CTF1: truncated header");
  Ctf1Header h;
  for (size_t n = 0; n < order; ++n) {
    const uint64_t v = get_u64le(d.data() + 8 * n);
    if (v == 0) throw Error(NTFG_ERR_FORMAT, "CTF1: zero dimension");
    if (max_entries && (v > max_entries || h.entries > max_entries / v))
      throw Error(NTFG_ERR_FORMAT, "CTF1: tensor exceeds the entry budget");
    if (!max_entries && h.entries > (uint64_t(1) << 62) / v) throw Error(NTFG_ERR_FORMAT, "CTF1: tensor too large");
    h.dims.push_back(v);
    h.entries *= v;
  }
  h.payload = long(5 + 8 * order);
  if (std::fseek(f.f, 0, SEEK_END) != 0) throw Error(NTFG_ERR_FORMAT, "CTF1: cannot seek");
  const long size = std::ftell(f.f);
  const uint64_t want = uint64_t(h.payload) + 8 * h.entries;
  if (uint64_t(size) != want)
    throw Error(NTFG_ERR_FORMAT, uint64_t(size) < want ? "CTF1: truncated payload" : "CTF1: trailing bytes");
  std::fseek(f.f, h.payload, SEEK_SET);
  return h;
}

void ctf1_header_api(const char* path, uint32_t* order, uint64_t* dims, uint32_t cap, uint64_t max_entries) {
  File f(path, "rb");
  const Ctf1Header h = ctf1_header(path, max_entries, f);
  *order = uint32_t(h.dims.size());
  if (dims) {
    if (h.dims.size() > cap) throw Error(NTFG_ERR_SHAPE, "CTF1: dims capacity too small for the tensor order");
    for (size_t n = 0; n < h.dims.size(); ++n) dims[n] = h.dims[n];
  }
}

void ctf1_read(Context* c, const char* path, void* dst, int dtype, int location, uint64_t max_entries) {
  if (!little_endian()) throw Error(NTFG_ERR_FORMAT, "CTF1 I/O assumes a little-endian host");
  File f(path, "rb");
  const Ctf1Header h = ctf1_header(path, max_entries, f);
  const uint64_t n = h.entries;
  if (location == NTFG_HOST) {
    if (dtype == 0) {
      if (std::fread(dst, 8, n, f.f) != n) throw Error(NTFG_ERR_FORMAT, "CTF1: truncated payload");
      return;
    }
    std::vector<double> buf(std::min<uint64_t>(n, kChunk));
    float* out = static_cast<float*>(dst);
    for (uint64_t b = 0; b < n; b += buf.size()) {
      const size_t len = size_t(std::min<uint64_t>(buf.size(), n - b));
      if (std::fread(buf.data(), 8, len, f.f) != len) throw Error(NTFG_ERR_FORMAT, "CTF1: truncated payload");
      for (size_t i = 0; i < len; ++i) out[b + i] = float(buf[i]);
    }
    return;
  }
  if (!c) throw Error(NTFG_ERR_INTERNAL, "CTF1 device read needs a context");
  // two pinned halves: read chunk i+1 from disk while chunk i is copied/converted
  const size_t chunk = size_t(std::min<uint64_t>(n, kChunk));
  double* pin = static_cast<double*>(c->pinned.get(2 * chunk * sizeof(double)));
  double* stage = dtype == 1 ? c->buf<double>("io.stage", 2 * chunk) : nullptr;
  cudaEvent_t done[2];
  for (auto& e : done) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  int half = 0;
  for (uint64_t b = 0; b < n; b += chunk, half ^= 1) {
    const size_t len = size_t(std::min<uint64_t>(chunk, n - b));
    double* hp = pin + size_t(half) * chunk;
    cuda_check(cudaEventSynchronize(done[half]), "cudaEventSynchronize");  // half free again
    if (std::fread(hp, 8, len, f.f) != len) throw Error(NTFG_ERR_FORMAT, "CTF1: truncated payload");
    if (dtype == 0) {
      cuda_check(cudaMemcpyAsync(static_cast<double*>(dst) + b, hp, len * 8, cudaMemcpyHostToDevice, c->stream),
                 "cudaMemcpyAsync");
    } else {
      double* sp = stage + size_t(half) * chunk;
      cuda_check(cudaMemcpyAsync(sp, hp, len * 8, cudaMemcpyHostToDevice, c->stream), "cudaMemcpyAsync");
      const int grid = int(std::min<int64_t>(ceil_div(int64_t(len), 256), 4096));
      convert_kernel<float, double><<<grid, 256, 0, c->stream>>>(sp, int64_t(len), static_cast<float*>(dst) + b);
      cuda_check(cudaGetLastError(), "convert_kernel");
    }
    cuda_check(cudaEventRecord(done[half], c->stream), "cudaEventRecord");
  }
  c->sync();
  for (auto& e : done) cudaEventDestroy(e);
}

void ctf1_write(Context* c, const char* path, uint32_t order, const uint64_t* dims, const void* src, int dtype,
                int location) {
  if (!little_endian()) throw Error(NTFG_ERR_FORMAT, "CTF1 I/O assumes a little-endian host");
  if (order == 0 || order > 255) throw Error(NTFG_ERR_FORMAT, "write_tensor: order must be in [1, 255]");
  uint64_t n = 1;
  for (uint32_t m = 0; m < order; ++m) n *= dims[m];
  File f(path, "wb");
  if (!f.f) throw Error(NTFG_ERR_FORMAT, std::string("cannot open for writing: ") + path);
  std::vector<unsigned char> head(5 + 8 * size_t(order));
  std::memcpy(head.data(), "CTF1", 4);
  head[4] = static_cast<unsigned char>(order);
  for (uint32_t m = 0; m < order; ++m) put_u64le(head.data() + 5 + 8 * m, dims[m]);
  if (std::fwrite(head.data(), 1, head.size(), f.f) != head.size())
    throw Error(NTFG_ERR_FORMAT, std::string("write failed: ") + path);
  const size_t chunk = size_t(std::min<uint64_t>(std::max<uint64_t>(n, 1), kChunk));
  std::vector<double> hostbuf;
  double* buf;
  double* stage = nullptr;
  if (location == NTFG_DEVICE) {
    if (!c) throw Error(NTFG_ERR_INTERNAL, "CTF1 device write needs a context");
    buf = static_cast<double*>(c->pinned.get(chunk * sizeof(double)));
    if (dtype == 1) stage = c->buf<double>("io.stage", chunk);
  } else {
    hostbuf.resize(chunk);
    buf = hostbuf.data();
  }
  for (uint64_t b = 0; b < n; b += chunk) {
    const size_t len = size_t(std::min<uint64_t>(chunk, n - b));
    if (location == NTFG_DEVICE) {
      if (dtype == 1) {
        const int grid = int(std::min<int64_t>(ceil_div(int64_t(len), 256), 4096));
        convert_kernel<double, float><<<grid, 256, 0, c->stream>>>(static_cast<const float*>(src) + b,
                                                                   int64_t(len), stage);
        cuda_check(cudaGetLastError(), "convert_kernel");
        cuda_check(cudaMemcpyAsync(buf, stage, len * 8, cudaMemcpyDeviceToHost, c->stream), "cudaMemcpyAsync");
      } else {
        cuda_check(cudaMemcpyAsync(buf, static_cast<const double*>(src) + b, len * 8, cudaMemcpyDeviceToHost,
                                   c->stream),
                   "cudaMemcpyAsync");
      }
      c->sync();
    } else if (dtype == 1) {
      for (size_t i = 0; i < len; ++i) buf[i] = double(static_cast<const float*>(src)[b + i]);
    } else {
      std::memcpy(buf, static_cast<const double*>(src) + b, len * 8);
    }
    if (std::fwrite(buf, 8, len, f.f) != len) throw Error(NTFG_ERR_FORMAT, std::string("write failed: ") + path);
  }
}

// ---- COO text ------------------------------------------------------------------------
static bool blank(const std::string& s) {
  for (unsigned char ch : s)
    if (!std::isspace(ch)) return false;
  return true;
}
static Error parse_error(const std::string& msg, size_t line) {
  return Error(NTFG_ERR_FORMAT, "line " + std::to_string(line) + ": " + msg);
}

// indices == nullptr: count only.  Values are raw (no floor: the reference's
// optional floor clamps the DENSE tensor, zeros included -- not a sparse op).
void coo_text_read(const char* path, uint32_t* order, uint64_t* dims, uint32_t cap, uint64_t* nnz,
                   int32_t* indices, double* values, uint64_t capacity, uint64_t max_entries) {
  std::ifstream is(path);
  if (!is) throw Error(NTFG_ERR_FORMAT, std::string("cannot open: ") + path);
  std::string line;
  size_t lineno = 0;
  std::vector<uint64_t> d;
  while (std::getline(is, line)) {
    ++lineno;
    if (blank(line)) continue;
    std::istringstream ss(line);
    std::string tag;
    ss >> tag;
    if (tag != "dims:") throw parse_error("expected `dims: I1 I2 ... IN`", lineno);
    uint64_t entries = 1;
    long long v = 0;
    while (ss >> v) {
      if (v <= 0) throw parse_error("dimensions must be positive", lineno);
      const uint64_t du = uint64_t(v);
      if (max_entries && (du > max_entries || entries > max_entries / du))
        throw parse_error("tensor exceeds the entry budget", lineno);
      entries *= du;
      d.push_back(du);
    }
    if (!ss.eof()) throw parse_error("malformed dimension list", lineno);
    if (d.empty()) throw parse_error("empty dimension list", lineno);
    break;
  }
  if (d.empty()) throw Error(NTFG_ERR_FORMAT, std::string("missing `dims:` header line: ") + path);
  if (d.size() > cap) throw Error(NTFG_ERR_SHAPE, "COO: dims capacity too small for the tensor order");
  if (d.size() > size_t(kMaxOrder)) throw Error(NTFG_ERR_SHAPE, "COO: tensor order above 8 is not supported");
  *order = uint32_t(d.size());
  for (size_t n = 0; n < d.size(); ++n) dims[n] = d[n];
  uint64_t count = 0;
  std::vector<long long> idx(d.size());
  while (std::getline(is, line)) {
    ++lineno;
    if (blank(line)) continue;
    std::istringstream ss(line);
    for (size_t n = 0; n < d.size(); ++n) {
      long long i = 0;
      if (!(ss >> i)) throw parse_error("malformed entry line", lineno);
      if (i < 0 || uint64_t(i) >= d[n]) throw parse_error("index out of range for mode " + std::to_string(n + 1), lineno);
      idx[n] = i;
    }
    double v = 0.0;
    if (!(ss >> v)) throw parse_error("malformed or missing value", lineno);
    std::string rest;
    if (ss >> rest) throw parse_error("trailing tokens after value", lineno);
    if (v < 0.0) throw parse_error("negative value", lineno);
    if (indices) {
      if (count >= capacity) throw Error(NTFG_ERR_SHAPE, "COO: capacity too small");
      for (size_t n = 0; n < d.size(); ++n) indices[count * d.size() + n] = int32_t(idx[n]);
      values[count] = v;
    }
    ++count;
  }
  *nnz = count;
}

// ---- trace CSV ----------------------------------------------------------------------
void trace_write(const char* path, const ntfg_trace_row* rows, uint64_t n) {
  File f(path, "w");
  if (!f.f) throw Error(NTFG_ERR_FORMAT, std::string("cannot open for writing: ") + path);
  std::fputs("iter,time_s,loss\n", f.f);
  for (uint64_t i = 0; i < n; ++i)
    std::fprintf(f.f, "%" PRIu64 ",%.17g,%.17g\n", uint64_t(rows[i].iter), rows[i].time_s, rows[i].loss);
  if (std::ferror(f.f)) throw Error(NTFG_ERR_FORMAT, std::string("write failed: ") + path);
}

// ---- generators ----------------------------------------------------------------------
void philox_uniforms(uint64_t seed, uint64_t stream, uint64_t offset, uint64_t n, double* out) {
  for (uint64_t j = 0; j < n; ++j) out[j] = Philox::uniform(seed, stream, offset + j);
}

// truth factors U[0,1) clamped to eps (random_matrix, io.cpp:202-208) from
// stream 1, factor n entry (i, r) = uniform #(off_n + i*R + r); init factors
// 0.1 + U from stream 2 (the BASELINE configs' U[0.1, 1.1) init).
void cp_factors_philox(uint32_t order, const uint64_t* dims, uint64_t rank, uint64_t seed, int which, double eps,
                       double* out) {
  uint64_t off = 0;
  const uint64_t stream = which == 0 ? kStreamTruth : kStreamInit;
  for (uint32_t m = 0; m < order; ++m) {
    for (uint64_t j = 0; j < dims[m] * rank; ++j) {
      const double u = Philox::uniform(seed, stream, off + j);
      out[off + j] = which == 0 ? (u < eps ? eps : u) : 0.1 + u;
    }
    off += dims[m] * rank;
  }
}

void generate_cp_gamma(Context& c, uint32_t order, const uint64_t* dims, uint64_t rank, uint64_t seed,
                       uint32_t k, double theta, uint64_t row0, uint64_t row1, void* dst, int dtype) {
  if (order < 1 || order > uint32_t(kMaxOrder)) throw Error(NTFG_ERR_SHAPE, "tensor order must be in [1, 8]");
  if (row0 > row1 || row1 > dims[0]) throw Error(NTFG_ERR_SHAPE, "generate: row range outside mode 0");
  if (k < 1 || !(theta > 0.0)) throw Error(NTFG_ERR_DOMAIN, "generate: gamma shape must be >= 1 and scale > 0");
  uint64_t F = 0;
  for (uint32_t m = 0; m < order; ++m) F += dims[m] * rank;
  std::vector<double> truth(F);
  cp_factors_philox(order, dims, rank, seed, 0, 1e-12, truth.data());
  double* dt = c.buf<double>("gen.truth", F);
  c.h2d(dt, truth.data(), F * sizeof(double));
  Geom g{};
  g.order = int(order);
  int64_t E = 1;
  for (uint32_t m = 0; m < order; ++m) {
    g.dims[m] = int64_t(dims[m]);
    E *= g.dims[m];
  }
  g.K = g.dims[order - 1];
  g.rows = E / g.K;
  const double* t[kMaxOrder] = {};
  uint64_t off = 0;
  for (uint32_t m = 0; m < order; ++m) {
    t[m] = dt + off;
    off += dims[m] * rank;
  }
  const int64_t per_row = E / g.dims[0];
  const int64_t n = int64_t(row1 - row0) * per_row;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), int64_t(c.sm_count) * 32)));
  const int64_t base = int64_t(row0) * per_row;
  if (dtype == 1)
    gen_cp_gamma_kernel<float><<<grid, 256, 0, c.stream>>>(g, int(rank), base, n, seed, int(k), theta,
                                                           static_cast<float*>(dst), t[0], t[1], t[2], t[3], t[4],
                                                           t[5], t[6], t[7]);
  else
    gen_cp_gamma_kernel<double><<<grid, 256, 0, c.stream>>>(g, int(rank), base, n, seed, int(k), theta,
                                                            static_cast<double*>(dst), t[0], t[1], t[2], t[3], t[4],
                                                            t[5], t[6], t[7]);
  cuda_check(cudaGetLastError(), "gen_cp_gamma_kernel");
  c.sync();
}

}  // namespace ntfg
