// evalio.cpp -- host-side measurement support (evalio.cpp / wire.cpp of the
// reference): the deterministic synthetic-data generator and the graph output
// file format.  Neither is on the timed path.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.hpp"

namespace knng_b200 {

namespace {

// Rng (rng.hpp:12-56) with the Box-Muller spare of next_gaussian.
struct HostRng {
  uint64_t state;
  float spare = 0.0f;
  bool have_spare = false;
  explicit HostRng(uint64_t s) : state(s) {}
  uint64_t next_u64() { return sm64_mix(state += kGamma); }
  float next_float() { return static_cast<float>(next_u64() >> 40) * 0x1.0p-24f; }
  float next_gaussian() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    float u1;
    do {
      u1 = next_float();
    } while (u1 <= 0.0f);
    const float u2 = next_float();
    const float r = std::sqrt(-2.0f * std::log(u1));
    const float a = 6.28318530717958647692f * u2;
    spare = r * std::sin(a);
    have_spare = true;
    return r * std::cos(a);
  }
};

constexpr uint32_t kMagic = 0x474E4E4Bu;  // "KNNG" wire.hpp:18
constexpr size_t kHeaderBytes = 22;       // wire.hpp:19

}  // namespace

// gen_random_dataset evalio.cpp:242-272 (same draws, same float ops).
void gen_random_dataset(uint64_t n, uint64_t dims, int dist, uint64_t seed, uint64_t clusters,
                        float* out) {
  require(n >= 1, "gen_random_dataset: n must be >= 1");
  require(dims >= 1, "gen_random_dataset: dims must be >= 1");
  HostRng rng(mix_seed(seed, 0xda7a5e7ull));
  const uint64_t total = n * dims;
  if (dist == 0) {
    for (uint64_t i = 0; i < total; ++i) out[i] = rng.next_float();
  } else if (dist == 1) {
    for (uint64_t i = 0; i < total; ++i) out[i] = rng.next_gaussian();
  } else {
    require(clusters >= 1, "gen_random_dataset: clustered needs clusters >= 1");
    std::vector<float> centers(clusters * dims);
    for (auto& v : centers) v = 5.0f * rng.next_gaussian();
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t c = i % clusters;
      for (uint64_t j = 0; j < dims; ++j)
        out[i * dims + j] = centers[c * dims + j] + rng.next_gaussian();
    }
  }
}

// save_graph evalio.cpp:274-276 = wire::serialize(KnnGraph) wire.cpp:76-82 +
// save_region wire.cpp:181-187.
void save_graph(const uint32_t* ids, const float* dists, uint64_t n, uint64_t k,
                const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("wire: cannot open for write: " + path);
  unsigned char h[kHeaderBytes];
  const uint8_t kind = 1, elem = 0;
  std::memcpy(h, &kMagic, 4);
  std::memcpy(h + 4, &kind, 1);
  std::memcpy(h + 5, &n, 8);
  std::memcpy(h + 13, &k, 8);
  std::memcpy(h + 21, &elem, 1);
  out.write(reinterpret_cast<const char*>(h), kHeaderBytes);
  out.write(reinterpret_cast<const char*>(ids), static_cast<std::streamsize>(n * k * 4));
  out.write(reinterpret_cast<const char*>(dists), static_cast<std::streamsize>(n * k * 4));
  if (!out) throw std::runtime_error("wire: write failed: " + path);
}

// peek_header wire.cpp:99-118 for a knng region file.
void load_graph_header(const std::string& path, uint64_t* n, uint64_t* k) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw std::runtime_error("wire: cannot open: " + path);
  const uint64_t size = static_cast<uint64_t>(in.tellg());
  in.seekg(0);
  if (size < kHeaderBytes) throw std::runtime_error("wire: region truncated before header end");
  unsigned char h[kHeaderBytes];
  in.read(reinterpret_cast<char*>(h), kHeaderBytes);
  uint32_t magic;
  std::memcpy(&magic, h, 4);
  if (magic != kMagic) throw std::runtime_error("wire: bad magic");
  if (h[4] > 3) throw std::runtime_error("wire: bad region kind");
  if (h[4] != 1) throw std::runtime_error("wire: expected knng region");
  if (h[21] > 2) throw std::runtime_error("wire: bad elem kind");
  std::memcpy(n, h + 5, 8);
  std::memcpy(k, h + 13, 8);
  if (size != kHeaderBytes + (*n) * (*k) * 8) throw std::runtime_error("wire: payload size mismatch");
}

void load_graph(const std::string& path, uint32_t* ids, float* dists, uint64_t n, uint64_t k) {
  uint64_t hn = 0, hk = 0;
  load_graph_header(path, &hn, &hk);
  require(hn == n && hk == k, "load_graph: output shape does not match the file");
  std::ifstream in(path, std::ios::binary);
  in.seekg(kHeaderBytes);
  in.read(reinterpret_cast<char*>(ids), static_cast<std::streamsize>(n * k * 4));
  in.read(reinterpret_cast<char*>(dists), static_cast<std::streamsize>(n * k * 4));
  if (!in) throw std::runtime_error("wire: read failed: " + path);
}

// ---------------------------------------------------------------------------
// .fvecs / .bvecs / .ivecs (read_vecs / write_vecs / read_ivecs / write_ivecs,
// evalio.cpp:31-123): per row a little-endian i32 dimension, then the row.
// ---------------------------------------------------------------------------
namespace {

// Walk the file row by row with the reference's checks (buffered stream);
// `row(i, payload, bytes)` receives each row's payload.
template <class RowFn>
void walk_vecs(const std::string& path, uint64_t esz, uint64_t* rows_out, uint64_t* dims_out,
               RowFn&& row) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw FormatError("cannot open: " + path);
  const uint64_t size = static_cast<uint64_t>(in.tellg());
  in.seekg(0);
  uint64_t rows = 0, dims = 0, pos = 0;
  std::vector<char> rowbuf;
  while (pos < size) {
    if (pos + 4 > size) throw FormatError(path + ": truncated dimension field");
    int32_t dim = 0;
    in.read(reinterpret_cast<char*>(&dim), 4);
    pos += 4;
    if (dim <= 0) throw FormatError(path + ": non-positive row dimension");
    if (rows == 0) {
      dims = static_cast<uint64_t>(dim);
      rowbuf.resize(dims * esz);
    } else if (static_cast<uint64_t>(dim) != dims) {
      throw FormatError(path + ": inconsistent row dimension " + std::to_string(dim) +
                        " (expected " + std::to_string(dims) + ")");
    }
    const uint64_t rb = dims * esz;
    if (pos + rb > size) throw FormatError(path + ": truncated row payload");
    in.read(rowbuf.data(), static_cast<std::streamsize>(rb));
    if (!in) throw FormatError("read failed: " + path);
    row(rows, rowbuf.data(), rb);
    pos += rb;
    ++rows;
  }
  *rows_out = rows;
  *dims_out = dims;
}

}  // namespace

void vecs_shape(const std::string& path, uint64_t esz, uint64_t* rows, uint64_t* dims) {
  walk_vecs(path, esz, rows, dims, [](uint64_t, const char*, uint64_t) {});
}

// Rows land in `out` (host), or stream to device memory through two pinned
// staging buffers (the file read overlaps the previous buffer's copy).
void read_vecs(const std::string& path, uint64_t esz, void* out, uint64_t rows, uint64_t dims,
               const Runner* dev_runner) {
  uint64_t fr = 0, fd = 0;
  vecs_shape(path, esz, &fr, &fd);
  require(fr == rows && fd == dims, "read_vecs: output shape does not match the file");
  const uint64_t rb = dims * esz;
  if (!dev_runner) {
    char* o = static_cast<char*>(out);
    walk_vecs(path, esz, &fr, &fd,
              [&](uint64_t i, const char* p, uint64_t n) { std::memcpy(o + i * rb, p, n); });
    return;
  }
  const Runner& r = *dev_runner;
  DeviceGuard g(r.device);
  const uint64_t per = std::max<uint64_t>(1, (uint64_t{32} << 20) / rb);  // rows per buffer
  HBuf<char> stage[2];
  stage[0].alloc(per * rb);
  stage[1].alloc(per * rb);
  cudaEvent_t done[2];
  KNNG_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  KNNG_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  int b = 0;
  uint64_t fill = 0, first = 0;
  char* o = static_cast<char*>(out);
  auto flush = [&]() {
    if (!fill) return;
    KNNG_CUDA(cudaMemcpyAsync(o + first * rb, stage[b].p, fill * rb, cudaMemcpyHostToDevice,
                              r.stream));
    KNNG_CUDA(cudaEventRecord(done[b], r.stream));
    b ^= 1;
    KNNG_CUDA(cudaEventSynchronize(done[b]));  // the other buffer's copy is finished
    first += fill;
    fill = 0;
  };
  KNNG_CUDA(cudaEventRecord(done[1], r.stream));
  walk_vecs(path, esz, &fr, &fd, [&](uint64_t, const char* p, uint64_t n) {
    std::memcpy(stage[b].p + fill * rb, p, n);
    if (++fill == per) flush();
  });
  flush();
  KNNG_CUDA(cudaStreamSynchronize(r.stream));
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
}

void write_vecs(const std::string& path, const void* data, uint64_t rows, uint64_t dims,
                uint64_t esz) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw FormatError("cannot open for write: " + path);
  const int32_t dim = static_cast<int32_t>(dims);
  const char* p = static_cast<const char*>(data);
  for (uint64_t i = 0; i < rows; ++i) {
    out.write(reinterpret_cast<const char*>(&dim), 4);
    out.write(p + i * dims * esz, static_cast<std::streamsize>(dims * esz));
  }
  if (!out) throw FormatError("write failed: " + path);
}

}  // namespace knng_b200
