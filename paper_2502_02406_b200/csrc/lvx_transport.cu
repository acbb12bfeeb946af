// Copy-engine peer transport for the ring schedulers (replaces the reference's
// buffered send / blocking FIFO recv of cluster.py:173-220 and
// WorkerContext.send/recv at cluster.py:227-264).
//
// Every rank owns one "arena": a device allocation whose layout is identical
// on all ranks (the host scheduler lays it out from global shapes).  A hop is
//   * one or more 2-D cudaMemcpyAsync from local memory straight into the
//     SAME offset of a peer's arena (pushed by this GPU's copy engine over
//     NVLink 5 / NVSwitch: no SM is used, so the attention kernels keep all
//     148 SMs while the hop is in flight), then
//   * a stream-ordered 32-bit flag write into the peer's arena
//     (cuStreamWriteValue32, which fences the preceding copies), which the
//     peer's compute stream waits on with cuStreamWaitValue32 (GEQ).
// Nothing on this path synchronises a host thread.
//
// Peers are mapped once: by CUDA IPC for one process per GPU
// (lvx_peer_export / lvx_peer_open), or by plain pointers when several ranks
// share one process and GPU (lvx_peer_attach: the thread-rank mode used to run
// n-rank protocols on one device).
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <new>

#include "lvx_common.cuh"

namespace {

typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

PFN_write32 write32() {
  static PFN_write32 fn = driver_fn<PFN_write32>("cuStreamWriteValue32");
  return fn;
}
PFN_wait32 wait32() {
  static PFN_wait32 fn = driver_fn<PFN_wait32>("cuStreamWaitValue32");
  return fn;
}

}  // namespace

struct lvx_peer_map {
  char* base;                       // this rank's arena (cudaMalloc, owned)
  uint64_t bytes;
  int rank, n;
  char* peer[LVX_MAX_PEERS];        // arena base of each peer as mapped here
  void* ipc_base[LVX_MAX_PEERS];    // cudaIpcOpenMemHandle results (to close)
};

extern "C" {

int lvx_peer_create(uint64_t bytes, int rank, int n, lvx_peer_map** out) {
  if (!out || bytes == 0 || n < 1 || n > LVX_MAX_PEERS || rank < 0 || rank >= n)
    return LVX_EINVAL;
  void* base = nullptr;
  if (cudaMalloc(&base, bytes) != cudaSuccess) return LVX_ECUDA;
  if (cudaMemset(base, 0, bytes) != cudaSuccess) {
    cudaFree(base);
    return LVX_ECUDA;
  }
  lvx_peer_map* m = new (std::nothrow) lvx_peer_map;
  if (!m) {
    cudaFree(base);
    return LVX_ECUDA;
  }
  memset(m, 0, sizeof(*m));
  m->base = static_cast<char*>(base);
  m->bytes = bytes;
  m->rank = rank;
  m->n = n;
  m->peer[rank] = m->base;
  *out = m;
  return LVX_OK;
}

int lvx_peer_destroy(lvx_peer_map* m) {
  if (!m) return LVX_OK;
  int st = LVX_OK;
  for (int p = 0; p < LVX_MAX_PEERS; ++p)
    if (m->ipc_base[p] && cudaIpcCloseMemHandle(m->ipc_base[p]) != cudaSuccess) st = LVX_ECUDA;
  if (cudaFree(m->base) != cudaSuccess) st = LVX_ECUDA;
  delete m;
  return st;
}

void* lvx_peer_base(const lvx_peer_map* m) { return m ? m->base : nullptr; }

uint64_t lvx_peer_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int lvx_peer_export(const lvx_peer_map* m, void* handle) {
  if (!m || !handle) return LVX_EINVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, m->base) != cudaSuccess) return LVX_ECUDA;
  memcpy(handle, &h, sizeof(h));
  return LVX_OK;
}

int lvx_peer_open(lvx_peer_map* m, int peer, const void* handle) {
  if (!m || !handle || peer < 0 || peer >= m->n || peer == m->rank) return LVX_EINVAL;
  if (m->ipc_base[peer]) return LVX_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return LVX_ECUDA;
  m->ipc_base[peer] = p;
  m->peer[peer] = static_cast<char*>(p);
  return LVX_OK;
}

int lvx_peer_attach(lvx_peer_map* m, int peer, const lvx_peer_map* other) {
  if (!m || !other || peer < 0 || peer >= m->n || other->bytes != m->bytes) return LVX_EINVAL;
  m->peer[peer] = other->base;
  return LVX_OK;
}

int lvx_peer_put(const lvx_peer_map* m, int peer, uint64_t dst_off, uint64_t dst_pitch,
                 const void* src, uint64_t src_pitch, uint64_t width, uint64_t height,
                 void* stream) {
  if (!m || peer < 0 || peer >= m->n || !m->peer[peer]) return LVX_EINVAL;
  if (width == 0 || height == 0) return LVX_OK;
  if (!src) return LVX_EINVAL;
  if (height > 1 && (dst_pitch < width || src_pitch < width)) return LVX_EINVAL;
  const uint64_t span = (height - 1) * dst_pitch + width;
  if (dst_off + span > m->bytes) return LVX_EINVAL;
  char* dst = m->peer[peer] + dst_off;
  auto st = static_cast<cudaStream_t>(stream);
  cudaError_t e = height == 1
                      ? cudaMemcpyAsync(dst, src, width, cudaMemcpyDeviceToDevice, st)
                      : cudaMemcpy2DAsync(dst, dst_pitch, src, src_pitch, width, height,
                                          cudaMemcpyDeviceToDevice, st);
  return e == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

int lvx_peer_signal(const lvx_peer_map* m, int peer, uint64_t flag_off, uint32_t value,
                    void* stream) {
  if (!m || peer < 0 || peer >= m->n || !m->peer[peer]) return LVX_EINVAL;
  if ((flag_off & 3) || flag_off + 4 > m->bytes) return LVX_EINVAL;
  auto fn = write32();
  if (!fn) return LVX_ECUDA;
  const CUdeviceptr p = reinterpret_cast<CUdeviceptr>(m->peer[peer] + flag_off);
  return fn(static_cast<CUstream>(stream), p, value, CU_STREAM_WRITE_VALUE_DEFAULT) ==
                 CUDA_SUCCESS
             ? LVX_OK
             : LVX_ECUDA;
}

int lvx_peer_wait(const lvx_peer_map* m, uint64_t flag_off, uint32_t value, void* stream) {
  if (!m || (flag_off & 3) || flag_off + 4 > m->bytes) return LVX_EINVAL;
  auto fn = wait32();
  if (!fn) return LVX_ECUDA;
  const CUdeviceptr p = reinterpret_cast<CUdeviceptr>(m->base + flag_off);
  return fn(static_cast<CUstream>(stream), p, value, CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
             ? LVX_OK
             : LVX_ECUDA;
}

// A dedicated non-blocking stream (torch's streams come from a fixed pool of
// 32 per device handed out round-robin, so two live torch.cuda.Stream objects
// can be the same CUDA stream; ranks sharing a GPU need streams of their own).
int lvx_stream_create(void** out) {
  if (!out) return LVX_EINVAL;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return LVX_ECUDA;
  *out = st;
  return LVX_OK;
}

int lvx_stream_destroy(void* stream) {
  if (!stream) return LVX_OK;
  return cudaStreamDestroy(static_cast<cudaStream_t>(stream)) == cudaSuccess ? LVX_OK : LVX_ECUDA;
}

}  // extern "C"
