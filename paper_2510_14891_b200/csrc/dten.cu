// DTEN v1 ingest straight into device memory.
//
// Format (cpkern dtensor.py:334-382, little endian): "DTEN", u32 version = 1,
// u32 d, u64 dims[d], u32 element type = 1 (float64), then the N float64
// values first mode fastest.  The header is validated with the reference's
// rules and messages map to its FormatError (CPK_ERR_FORMAT).
//
// A slab [lo, hi) along `mode` of the file's tensor is a set of `outer`
// contiguous runs of (hi - lo) * inner values (inner = prod of the faster
// modes' extents, outer = prod of the slower ones), and concatenating the
// runs in file order is exactly the slab's own first-mode-fastest layout.
// So the loader preads runs into pinned staging buffers with a few reader
// threads and streams each full buffer to the device with cudaMemcpyAsync
// while the next one fills (double buffering on the caller's stream): the
// sharded CP-ALS driver loads only its own rows, the whole tensor never
// passes through pageable host memory, and there is no redistribution step
// (the one the paper found dominant).
#include "common.cuh"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace cpk {
namespace {

constexpr char kMagic[4] = {'D', 'T', 'E', 'N'};
constexpr uint32_t kVersion = 1, kFloat64 = 1;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

bool pread_all(int fd, void* buf, size_t n, int64_t off) {
  char* p = static_cast<char*>(buf);
  while (n > 0) {
    const ssize_t r = pread(fd, p, n, off);
    if (r <= 0) return false;
    p += r;
    n -= size_t(r);
    off += r;
  }
  return true;
}

// dtensor._read_dten_meta (dtensor.py:359-382)
int read_header(int fd, int* d, int64_t* dims, int64_t* data_offset, int64_t* file_bytes) {
  unsigned char head[12];
  if (!pread_all(fd, head, 12, 0)) return fail(CPK_ERR_FORMAT, "truncated DTEN header");
  uint32_t version, nd;
  memcpy(&version, head + 4, 4);
  memcpy(&nd, head + 8, 4);
  if (memcmp(head, kMagic, 4) != 0) {
    char shown[20] = {0}, *q = shown;  // Python bytes repr of the 4 magic bytes
    for (int i = 0; i < 4; ++i) {
      const unsigned char c = head[i];
      if (c >= 32 && c < 127 && c != '\\' && c != '\'') *q++ = char(c);
      else q += snprintf(q, 5, "\\x%02x", c);
    }
    return fail(CPK_ERR_FORMAT, "bad magic b'%s', expected b'DTEN'", shown);
  }
  if (version != kVersion) return fail(CPK_ERR_FORMAT, "unsupported DTEN version %u", version);
  if (nd < 1 || nd > 64) return fail(CPK_ERR_FORMAT, "implausible mode count %u", nd);
  std::vector<unsigned char> raw(8 * nd + 4);
  if (!pread_all(fd, raw.data(), raw.size(), 12)) return fail(CPK_ERR_FORMAT, "truncated DTEN dimension block");
  uint32_t etype;
  memcpy(&etype, raw.data() + 8 * nd, 4);
  if (etype != kFloat64) return fail(CPK_ERR_FORMAT, "unsupported element-type code %u", etype);
  // the shape as Python prints a tuple, for messages that match the reference's
  std::string shape = "(";
  for (uint32_t m = 0; m < nd; ++m) {
    uint64_t e;
    memcpy(&e, raw.data() + 8 * m, 8);
    shape += std::to_string(e) + (m + 1 < nd ? ", " : (nd == 1 ? ",)" : ")"));
  }
  int64_t n = 1;
  for (uint32_t m = 0; m < nd; ++m) {
    uint64_t e;
    memcpy(&e, raw.data() + 8 * m, 8);
    if (e < 1)
      return fail(CPK_ERR_FORMAT, "bad shape in DTEN header: every extent must be >= 1, got %s", shape.c_str());
    if (e > uint64_t(INT64_MAX) / uint64_t(n))
      return fail(CPK_ERR_FORMAT, "bad shape in DTEN header: volume overflows int64");
    dims[m] = int64_t(e);
    n *= int64_t(e);
  }
  struct stat st;
  if (fstat(fd, &st) != 0) return fail(CPK_ERR_FORMAT, "cannot stat DTEN file");
  *d = int(nd);
  *data_offset = 12 + 8 * int64_t(nd) + 4;
  *file_bytes = int64_t(st.st_size);
  const int64_t payload = *file_bytes - *data_offset;
  if (payload != 8 * n)
    return fail(CPK_ERR_FORMAT, "payload holds %lld bytes, shape %s needs %lld", (long long)payload, shape.c_str(),
                (long long)(8 * n));
  return CPK_OK;
}

}  // namespace
}  // namespace cpk

using namespace cpk;

extern "C" int cpk_dten_read_header(const char* path, int* d, int64_t* dims) {
  if (!path || !d || !dims) return fail(CPK_ERR_PARAM, "NULL argument");
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return fail(CPK_ERR_FORMAT, "cannot open %s", path);
  int64_t off, bytes;
  return read_header(f.fd, d, dims, &off, &bytes);
}

extern "C" int cpk_dten_load_slab_f64(const char* path, int mode, int64_t lo, int64_t hi, double* dst,
                                      int64_t dst_elems, int threads, void* stream) {
  if (!path || !dst) return fail(CPK_ERR_PARAM, "NULL argument");
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return fail(CPK_ERR_FORMAT, "cannot open %s", path);
  int d;
  int64_t dims[CPK_DTEN_MAX_MODES], data_off, file_bytes;
  int rc = read_header(f.fd, &d, dims, &data_off, &file_bytes);
  if (rc) return rc;
  if (mode < 0 || mode >= d) return fail(CPK_ERR_INDEX, "mode %d out of range [0, %d]", mode, d - 1);
  if (lo < 0 || hi < lo || hi > dims[mode])
    return fail(CPK_ERR_PARAM, "slab [%lld, %lld) outside [0, %lld)", (long long)lo, (long long)hi,
                (long long)dims[mode]);
  int64_t inner = 1, outer = 1;
  for (int m = 0; m < mode; ++m) inner *= dims[m];
  for (int m = mode + 1; m < d; ++m) outer *= dims[m];
  const int64_t run = (hi - lo) * inner;  // values per contiguous run
  if (dst_elems != run * outer)
    return fail(CPK_ERR_SHAPE, "destination holds %lld values, slab needs %lld", (long long)dst_elems,
                (long long)(run * outer));
  if (run == 0 || outer == 0) return CPK_OK;
  cudaStream_t st = as_stream(stream);

  // staging: two pinned buffers; each is filled with whole runs when they
  // fit, else with pieces of one run
  const int64_t kStage = int64_t(64) << 20;  // bytes per buffer
  const int64_t stage_vals = std::max<int64_t>(1, kStage / 8);
  double* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  for (int i = 0; i < 2; ++i) {
    if (cudaHostAlloc(&buf[i], size_t(stage_vals) * 8, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) {
      for (int j = 0; j <= i; ++j) {
        if (buf[j]) cudaFreeHost(buf[j]);
        if (done[j]) cudaEventDestroy(done[j]);
      }
      return fail(CPK_ERR_RESOURCE, "cannot allocate pinned staging buffers");
    }
  }
  const int hw = int(std::thread::hardware_concurrency());
  const int nthreads = std::max(1, std::min(threads > 0 ? threads : std::max(8, hw), 32));
  const int64_t total = run * outer;  // values to move
  int64_t moved = 0;
  int which = 0;
  bool io_ok = true;
  while (moved < total && io_ok) {
    const int64_t take = std::min(stage_vals, total - moved);
    double* b = buf[which];
    if (cudaEventSynchronize(done[which]) != cudaSuccess) {  // previous copy out of this buffer
      io_ok = false;
      break;
    }
    // values [moved, moved + take) of the slab: split across reader threads
    // by value range; each maps slab offsets back to file offsets run by run
    std::atomic<bool> ok{true};
    auto read_range = [&](int64_t a, int64_t z) {
      while (a < z && ok.load(std::memory_order_relaxed)) {
        const int64_t o = a / run, w = a % run;  // run index, offset within it
        const int64_t n = std::min(z - a, run - w);
        const int64_t file_val = o * dims[mode] * inner + lo * inner + w;
        if (!pread_all(f.fd, b + (a - moved), size_t(n) * 8, data_off + 8 * file_val)) ok = false;
        a += n;
      }
    };
    const int64_t per = (take + nthreads - 1) / nthreads;
    std::vector<std::thread> pool;
    for (int t = 1; t < nthreads && int64_t(t) * per < take; ++t)
      pool.emplace_back(read_range, moved + t * per, moved + std::min(take, (t + 1) * per));
    read_range(moved, moved + std::min(take, per));
    for (auto& th : pool) th.join();
    if (!ok) {
      io_ok = false;
      break;
    }
    if (cudaMemcpyAsync(dst + moved, b, size_t(take) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(done[which], st) != cudaSuccess) {
      io_ok = false;
      break;
    }
    moved += take;
    which ^= 1;
  }
  // the staging buffers are freed only after the last copies have drained
  for (int i = 0; i < 2; ++i) {
    cudaEventSynchronize(done[i]);
    cudaEventDestroy(done[i]);
    cudaFreeHost(buf[i]);
  }
  if (!io_ok) {
    if (moved < total && cudaGetLastError() == cudaSuccess) return fail(CPK_ERR_FORMAT, "short read from %s", path);
    return fail(CPK_ERR_CUDA, "staging copy failed");
  }
  return check_launch("dten load");
}
