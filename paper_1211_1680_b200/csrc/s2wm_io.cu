// S2WM file I/O (reference: mapio.py) with device-side payloads.
//
// Layout (mapio.py:1-15), all little-endian:
//   0  4  magic "S2WM"
//   4  4  version (u32) = 1
//   8  1  scheme (u8): 0 = GL, 1 = MW
//   9  4  band-limit L (u32)
//   13 1  kind (u8): 0 = real map, 1 = complex map, 2 = harmonic coefficients
//   14 8  payload_count (u64)
// followed by payload_count float64 (real maps) or (re, im) float64 pairs.
//
// Device payloads stream through two pinned staging buffers: file reads of
// chunk i+1 overlap the host->device copy of chunk i (and symmetrically for
// writes), so a 537 MB L = 4096 complex map moves at disk/PCIe speed without
// a pageable bounce.  Writing the same payload twice yields byte-identical
// files (mapio.py:15).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "s2w.h"
#include "s2w_internal.h"

namespace {

constexpr size_t kHeader = 22;
constexpr size_t kChunk = 32u << 20;  // staging chunk (bytes)

static_assert(sizeof(double) == 8, "float64 payload");

bool little_endian() {
  const uint16_t v = 1;
  uint8_t b;
  std::memcpy(&b, &v, 1);
  return b == 1;
}

void put_u32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put_u64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint32_t get_u32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
  return v;
}
uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
  cudaError_t init(size_t bytes) {
    for (int i = 0; i < 2; ++i) {
      cudaError_t e = cudaHostAlloc(&p[i], bytes, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
};

}  // namespace

extern "C" {

int s2w_s2wm_read_header(const char* path, int* scheme, int* L, int* kind, long long* count) {
  if (!path || !scheme || !L || !kind || !count) return s2w::io_fail(S2W_EPARAM, "null argument");
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return s2w::io_fail(S2W_EIO, "%s: cannot open for reading", path);
  uint8_t h[kHeader];
  const size_t got = fread(h, 1, kHeader, fh.f);
  if (got < kHeader)
    return s2w::io_fail(S2W_EFORMAT_TRUNCATED, "%s: shorter than the %zu-byte header", path, kHeader);
  if (std::memcmp(h, "S2WM", 4) != 0)
    return s2w::io_fail(S2W_EFORMAT_MAGIC, "%s: not an S2WM file (magic %.4s)", path, (const char*)h);
  const uint32_t version = get_u32(h + 4);
  if (version != 1) return s2w::io_fail(S2W_EFORMAT_VERSION, "%s: unsupported version %u", path, version);
  *scheme = h[8];
  *L = (int)get_u32(h + 9);
  *kind = h[13];
  *count = (long long)get_u64(h + 14);
  return S2W_OK;
}

int s2w_s2wm_read_payload(const char* path, long long count, int complex_payload, void* dst,
                          int dst_device, void* stream) {
  if (!path || !dst || count < 0) return s2w::io_fail(S2W_EPARAM, "invalid argument");
  if (!little_endian()) return s2w::io_fail(S2W_EINTERNAL, "big-endian hosts are not supported");
  File fh;
  fh.f = fopen(path, "rb");
  if (!fh.f) return s2w::io_fail(S2W_EIO, "%s: cannot open for reading", path);
  if (fseek(fh.f, 0, SEEK_END) != 0) return s2w::io_fail(S2W_EIO, "%s: seek failed", path);
  const long long size = ftell(fh.f);
  const long long item = complex_payload ? 16 : 8;
  const long long expected = count * item;
  const long long body = size - (long long)kHeader;
  if (body != expected)
    return s2w::io_fail(S2W_EFORMAT_TRUNCATED, "%s: payload holds %lld bytes, expected %lld", path,
                        body, expected);
  if (fseek(fh.f, (long)kHeader, SEEK_SET) != 0) return s2w::io_fail(S2W_EIO, "%s: seek failed", path);
  if (!dst_device) {
    if (fread(dst, 1, (size_t)expected, fh.f) != (size_t)expected)
      return s2w::io_fail(S2W_EIO, "%s: read failed", path);
    return S2W_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Pinned pin;
  const size_t chunk = (size_t)std::min<long long>((long long)kChunk, std::max<long long>(expected, 1));
  if (pin.init(chunk) != cudaSuccess) return s2w::io_fail(S2W_ENOMEM, "pinned staging allocation failed");
  long long off = 0;
  int b = 0;
  while (off < expected) {
    const size_t n = (size_t)std::min<long long>((long long)chunk, expected - off);
    // the copy that last used this buffer must have finished
    if (cudaEventSynchronize(pin.ev[b]) != cudaSuccess)
      return s2w::io_fail(S2W_ECUDA, "staging event failed");
    if (fread(pin.p[b], 1, n, fh.f) != n) return s2w::io_fail(S2W_EIO, "%s: read failed", path);
    if (cudaMemcpyAsync((char*)dst + off, pin.p[b], n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(pin.ev[b], st) != cudaSuccess)
      return s2w::io_fail(S2W_ECUDA, "host-to-device copy failed");
    off += (long long)n;
    b ^= 1;
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return s2w::io_fail(S2W_ECUDA, "stream sync failed");
  return S2W_OK;
}

int s2w_s2wm_write(const char* path, int scheme, int L, int kind, long long count,
                   int complex_payload, const void* src, int src_device, void* stream) {
  if (!path || !src || count < 1) return s2w::io_fail(S2W_EPARAM, "refusing to write an empty payload");
  if (scheme < 0 || scheme > 255 || kind < 0 || kind > 255 || L < 0)
    return s2w::io_fail(S2W_EPARAM, "invalid header field");
  if (!little_endian()) return s2w::io_fail(S2W_EINTERNAL, "big-endian hosts are not supported");
  uint8_t h[kHeader];
  std::memcpy(h, "S2WM", 4);
  put_u32(h + 4, 1);
  h[8] = (uint8_t)scheme;
  put_u32(h + 9, (uint32_t)L);
  h[13] = (uint8_t)kind;
  put_u64(h + 14, (uint64_t)count);
  File fh;
  fh.f = fopen(path, "wb");
  if (!fh.f) return s2w::io_fail(S2W_EIO, "writing %s: cannot open", path);
  if (fwrite(h, 1, kHeader, fh.f) != kHeader) return s2w::io_fail(S2W_EIO, "writing %s: short write", path);
  const long long bytes = count * (complex_payload ? 16 : 8);
  if (!src_device) {
    if (fwrite(src, 1, (size_t)bytes, fh.f) != (size_t)bytes)
      return s2w::io_fail(S2W_EIO, "writing %s: short write", path);
    return S2W_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Pinned pin;
  const size_t chunk = (size_t)std::min<long long>((long long)kChunk, bytes);
  if (pin.init(chunk) != cudaSuccess) return s2w::io_fail(S2W_ENOMEM, "pinned staging allocation failed");
  // prime: copy chunk 0; then, while chunk i is written to the file, chunk i+1 is copied
  long long off = 0;
  int b = 0;
  size_t n = (size_t)std::min<long long>((long long)chunk, bytes);
  if (cudaMemcpyAsync(pin.p[b], src, n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaEventRecord(pin.ev[b], st) != cudaSuccess)
    return s2w::io_fail(S2W_ECUDA, "device-to-host copy failed");
  while (off < bytes) {
    const long long next = off + (long long)n;
    size_t nn = 0;
    if (next < bytes) {
      nn = (size_t)std::min<long long>((long long)chunk, bytes - next);
      if (cudaMemcpyAsync(pin.p[b ^ 1], (const char*)src + next, nn, cudaMemcpyDeviceToHost, st) !=
              cudaSuccess ||
          cudaEventRecord(pin.ev[b ^ 1], st) != cudaSuccess)
        return s2w::io_fail(S2W_ECUDA, "device-to-host copy failed");
    }
    if (cudaEventSynchronize(pin.ev[b]) != cudaSuccess)
      return s2w::io_fail(S2W_ECUDA, "staging event failed");
    if (fwrite(pin.p[b], 1, n, fh.f) != n) return s2w::io_fail(S2W_EIO, "writing %s: short write", path);
    off = next;
    n = nn;
    b ^= 1;
  }
  return S2W_OK;
}

}  // extern "C"
