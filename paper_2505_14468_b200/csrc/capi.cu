// C ABI plumbing: status strings, device attributes, and the P1 artifact pre-loader
// (pinned host -> HBM on a side stream; single host read fanned out over NVLink by NCCL).
//
// Replaces the reference's modelled load of a PreloadPlan GPU placement,
// `usable_at_ms = now + load_from_container_ms | load_cold_ms`
// (/root/reference/pkg/src/slorasim/engine.py:1040-1053, ArtifactSpec core.py:56-78), with
// real transfers whose measured time calibrates ArtifactSpec.load_from_container_ms.
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace slx {
int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}
}  // namespace slx

using namespace slx;

extern "C" const char* slx_status_string(int status) {
  switch (status) {
    case SLX_OK: return "ok";
    case SLX_ERR_INVALID: return "invalid argument or shape";
    case SLX_ERR_ALIGN: return "misaligned pointer or leading dimension";
    case SLX_ERR_UNSUPPORTED: return "shape outside the kernel envelope";
    case SLX_ERR_WORKSPACE: return "workspace missing or too small";
    case SLX_ERR_CUDA: return "CUDA error";
    case SLX_ERR_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

extern "C" int slx_abi_version(void) { return SLX_ABI_VERSION; }

extern "C" int slx_device_sm_count(int* out) {
  SLX_CHECK_ARG(out != nullptr);
  *out = sm_count();
  return SLX_OK;
}

// ------------------------------------------------------------------ P1 pre-loader
extern "C" int slx_host_register(void* ptr, size_t bytes) {
  SLX_CHECK_ARG(ptr && bytes > 0);
  return cudaHostRegister(ptr, bytes, cudaHostRegisterPortable) == cudaSuccess ? SLX_OK
                                                                                : SLX_ERR_CUDA;
}

extern "C" int slx_host_unregister(void* ptr) {
  SLX_CHECK_ARG(ptr != nullptr);
  return cudaHostUnregister(ptr) == cudaSuccess ? SLX_OK : SLX_ERR_CUDA;
}

extern "C" int slx_preload_h2d(void* dst_dev, const void* src_pinned, size_t bytes,
                               size_t chunk_bytes, void* stream, void* done_event) {
  SLX_CHECK_ARG(dst_dev && src_pinned && chunk_bytes > 0);
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t off = 0; off < bytes; off += chunk_bytes) {
    const size_t n = bytes - off < chunk_bytes ? bytes - off : chunk_bytes;
    if (cudaMemcpyAsync((char*)dst_dev + off, (const char*)src_pinned + off, n,
                        cudaMemcpyHostToDevice, s) != cudaSuccess)
      return SLX_ERR_CUDA;
  }
  if (done_event && cudaEventRecord((cudaEvent_t)done_event, s) != cudaSuccess) return SLX_ERR_CUDA;
  return SLX_OK;
}

extern "C" int slx_offload_d2h(void* dst_pinned, const void* src_dev, size_t bytes,
                               size_t chunk_bytes, void* stream, void* done_event) {
  SLX_CHECK_ARG(dst_pinned && src_dev && chunk_bytes > 0);
  cudaStream_t s = (cudaStream_t)stream;
  for (size_t off = 0; off < bytes; off += chunk_bytes) {
    const size_t n = bytes - off < chunk_bytes ? bytes - off : chunk_bytes;
    if (cudaMemcpyAsync((char*)dst_pinned + off, (const char*)src_dev + off, n,
                        cudaMemcpyDeviceToHost, s) != cudaSuccess)
      return SLX_ERR_CUDA;
  }
  if (done_event && cudaEventRecord((cudaEvent_t)done_event, s) != cudaSuccess) return SLX_ERR_CUDA;
  return SLX_OK;
}

extern "C" int slx_nccl_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

extern "C" int slx_nccl_get_unique_id(void* out_id) {
  SLX_CHECK_ARG(out_id != nullptr);
  return ncclGetUniqueId((ncclUniqueId*)out_id) == ncclSuccess ? SLX_OK : SLX_ERR_NCCL;
}

extern "C" int slx_nccl_comm_init(void** comm, int nranks, const void* id, int rank) {
  SLX_CHECK_ARG(comm && id && nranks > 0 && rank >= 0 && rank < nranks);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, nranks, uid, rank) != ncclSuccess) return SLX_ERR_NCCL;
  *comm = (void*)c;
  return SLX_OK;
}

extern "C" int slx_nccl_comm_destroy(void* comm) {
  SLX_CHECK_ARG(comm != nullptr);
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? SLX_OK : SLX_ERR_NCCL;
}

extern "C" int slx_bcast(void* buf, size_t bytes, int root, void* comm, void* stream) {
  SLX_CHECK_ARG(buf && comm);
  return ncclBroadcast(buf, buf, bytes, ncclChar, root, (ncclComm_t)comm, (cudaStream_t)stream) ==
                 ncclSuccess
             ? SLX_OK
             : SLX_ERR_NCCL;
}

// Pipelined: chunk i is copied H2D on copy_stream (root only) while chunk i-1 is
// broadcast on comm_stream; an event per chunk orders the broadcast after its copy.
extern "C" int slx_preload_bcast(void* dst_dev, const void* src_pinned, size_t bytes,
                                 size_t chunk_bytes, int root, void* comm, void* copy_stream,
                                 void* comm_stream) {
  SLX_CHECK_ARG(dst_dev && comm && chunk_bytes > 0);
  int rank = 0;
  if (ncclCommUserRank((ncclComm_t)comm, &rank) != ncclSuccess) return SLX_ERR_NCCL;
  const bool is_root = rank == root;
  if (is_root) SLX_CHECK_ARG(src_pinned != nullptr);
  cudaStream_t cs = (cudaStream_t)copy_stream, ns = (cudaStream_t)comm_stream;
  const size_t n_chunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  cudaEvent_t ev[2];
  for (int i = 0; i < 2; ++i)
    if (cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) return SLX_ERR_CUDA;
  int status = SLX_OK;
  for (size_t c = 0; c < n_chunks && status == SLX_OK; ++c) {
    const size_t off = c * chunk_bytes;
    const size_t n = bytes - off < chunk_bytes ? bytes - off : chunk_bytes;
    char* dst = (char*)dst_dev + off;
    if (is_root) {
      if (cudaMemcpyAsync(dst, (const char*)src_pinned + off, n, cudaMemcpyHostToDevice, cs) !=
              cudaSuccess ||
          cudaEventRecord(ev[c & 1], cs) != cudaSuccess ||
          cudaStreamWaitEvent(ns, ev[c & 1], 0) != cudaSuccess) {
        status = SLX_ERR_CUDA;
        break;
      }
    }
    if (ncclBroadcast(dst, dst, n, ncclChar, root, (ncclComm_t)comm, ns) != ncclSuccess)
      status = SLX_ERR_NCCL;
  }
  // events are consumed by already-enqueued waits; destroying them now is legal
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return status;
}
