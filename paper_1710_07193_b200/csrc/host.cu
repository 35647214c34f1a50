// Host-side orchestration of the C ABI (include/dctf.h):
//   * dctf_filter_frames_host — a frame batch from / to host buffers: the
//     frames stream through a 3-slot device ring in chunks, H2D copy, the
//     batch kernel and D2H copy of consecutive chunks overlapped on three
//     streams (filter_image's host-buffer contract, image.hpp:210-225, for a
//     video of frames);
//   * the multi-device entries: a dctf_multi holds one
//     replica of a plan per device; blocks never exchange data
//     (image.hpp:205-209), so an image is split into contiguous block-row
//     bands and a frame batch into contiguous frame ranges, one host thread
//     and stream per replica, no data-path collective. The only collective is
//     the optional all-gather of device-resident results (NCCL, loaded at
//     run time; NVLink / NVSwitch between GPUs of one box).
// Streams, events and scratch are per call / per host thread, so concurrent
// calls on one plan from several threads do not serialise on plan state.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

using dctf::set_error;

struct dctf_multi {
  std::vector<dctf_plan*> replicas;  // one per entry of devices
  std::vector<int> devices;
};

namespace {

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Three non-blocking streams (H2D, compute, D2H) and an event pool per host
// thread and device, created on first use and kept for the thread's life.
struct IoStreams {
  cudaStream_t s[3] = {};
  cudaEvent_t ev[32] = {};
};
dctf_status io_streams(int device, IoStreams*& out) {
  thread_local std::vector<IoStreams*> per_dev;
  if (device < 0 || device >= 1024) return set_error(DCTF_INVALID_ARGUMENT, "bad device ordinal");
  if (per_dev.size() <= static_cast<size_t>(device)) per_dev.resize(device + 1, nullptr);
  if (!per_dev[device]) {
    auto* io = new IoStreams();
    for (auto& st : io->s)
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return set_error(DCTF_CUDA_ERROR, "cudaStreamCreate");
    for (auto& e : io->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        return set_error(DCTF_CUDA_ERROR, "cudaEventCreate");
    per_dev[device] = io;
    // keep the per-call ring allocations of the host entries cached in the
    // device's stream-ordered pool instead of returning them at every sync
    static std::once_flag pool_once[64];
    if (device < 64)
      std::call_once(pool_once[device], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
          uint64_t thr = ~0ull;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
      });
  }
  out = per_dev[device];
  return DCTF_OK;
}

dctf_status check_frames(const dctf_plan* const* plans, int nplans, const int* pof, int nframes, int w, int h,
                         size_t pitch, size_t frame_stride) {
  if (!plans || nplans < 1 || !pof || nframes < 0) return set_error(DCTF_INVALID_ARGUMENT, "bad plan list");
  if (w < 0 || h < 0) return set_error(DCTF_INVALID_ARGUMENT, "image dimensions must be >= 0");
  if (h > 0 && pitch < static_cast<size_t>(w)) return set_error(DCTF_INVALID_ARGUMENT, "pitch < width");
  if (nframes > 1 && frame_stride < pitch * static_cast<size_t>(h))
    return set_error(DCTF_INVALID_ARGUMENT, "frame_stride smaller than one frame");
  for (int i = 0; i < nplans; ++i) {
    if (!plans[i]) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
    if (plans[i]->n != plans[0]->n || plans[i]->device != plans[0]->device)
      return set_error(DCTF_INVALID_ARGUMENT, "plans must share n and device");
  }
  for (int f = 0; f < nframes; ++f)
    if (pof[f] < 0 || pof[f] >= nplans) return set_error(DCTF_INVALID_ARGUMENT, "plan_of_frame index out of range");
  return DCTF_OK;
}

// Generic 3-stage pipeline over host chunks: chunk c's H2D copy (copy_in),
// device work (run) and D2H copy (copy_out) on the calling thread's three
// streams of `dev`, through a ring of up to 3 device slots of slot_bytes for
// input and output each (allocated per call, stream-ordered). Synchronous.
template <typename In, typename Run, typename Out>
dctf_status host_pipeline(int dev, int nch, size_t slot_bytes, In copy_in, Run run, Out copy_out) {
  if (nch <= 0) return DCTF_OK;
  DevGuard guard(dev);
  IoStreams* io = nullptr;
  dctf_status s = io_streams(dev, io);
  if (s != DCTF_OK) return s;
  const int slots = std::min(3, nch);
  uint8_t* dbuf = nullptr;
  cudaStream_t s_in = io->s[0], s_run = io->s[1], s_out = io->s[2];
  // the ring, then a per-call NaN flag (quantize_sample's throw, reported as
  // DCTF_NAN_ENCOUNTERED; the plan's own flag belongs to the device entries)
  const size_t ring = ((2 * slots * slot_bytes + 255) / 256) * 256;
  if (cudaMallocAsync(reinterpret_cast<void**>(&dbuf), ring + 256, s_run) != cudaSuccess)
    return set_error(DCTF_CUDA_ERROR, "host pipeline: device ring allocation failed");
  int* d_nan = reinterpret_cast<int*>(dbuf + ring);
  cudaMemsetAsync(d_nan, 0, sizeof(int), s_run);
  dctf::NanScope nan_scope(d_nan);
  int nan_seen = 0;
  cudaEventRecord(io->ev[31], s_run);
  cudaStreamWaitEvent(s_in, io->ev[31], 0);
  cudaEvent_t* ev_in = io->ev;        // [slot] input chunk landed
  cudaEvent_t* ev_run = io->ev + 3;   // [slot] device work done (input slot free, output ready)
  cudaEvent_t* ev_out = io->ev + 6;   // [slot] D2H done (output slot free)
  for (int c = 0; c < nch && s == DCTF_OK; ++c) {
    const int slot = c % slots;
    uint8_t* din = dbuf + slot * slot_bytes;
    uint8_t* dout = dbuf + (slots + slot) * slot_bytes;
    if (c >= slots) cudaStreamWaitEvent(s_in, ev_run[slot], 0);  // work c - slots has read this input slot
    cudaError_t e = copy_in(c, din, s_in);
    if (e != cudaSuccess) {
      s = set_error(DCTF_CUDA_ERROR, std::string("host pipeline H2D: ") + cudaGetErrorString(e));
      break;
    }
    cudaEventRecord(ev_in[slot], s_in);
    cudaStreamWaitEvent(s_run, ev_in[slot], 0);
    if (c >= slots) cudaStreamWaitEvent(s_run, ev_out[slot], 0);  // D2H c - slots drained this output slot
    s = run(c, din, dout, s_run);
    if (s != DCTF_OK) break;
    cudaEventRecord(ev_run[slot], s_run);
    cudaStreamWaitEvent(s_out, ev_run[slot], 0);
    e = copy_out(c, dout, s_out);
    if (e != cudaSuccess) {
      s = set_error(DCTF_CUDA_ERROR, std::string("host pipeline D2H: ") + cudaGetErrorString(e));
      break;
    }
    cudaEventRecord(ev_out[slot], s_out);
  }
  // the ring is released once every stream has finished with it
  cudaEventRecord(io->ev[29], s_in);
  cudaEventRecord(io->ev[30], s_out);
  cudaStreamWaitEvent(s_run, io->ev[29], 0);
  cudaStreamWaitEvent(s_run, io->ev[30], 0);
  cudaMemcpyAsync(&nan_seen, d_nan, sizeof(int), cudaMemcpyDeviceToHost, s_run);
  cudaFreeAsync(dbuf, s_run);
  const cudaError_t e = cudaStreamSynchronize(s_run);
  cudaStreamSynchronize(s_in);
  cudaStreamSynchronize(s_out);
  if (s == DCTF_OK && e != cudaSuccess) s = set_error(DCTF_CUDA_ERROR, std::string("host pipeline: ") + cudaGetErrorString(e));
  if (s == DCTF_OK && nan_seen) s = set_error(DCTF_NAN_ENCOUNTERED, "quantize: NaN sample");
  return s;
}

// h x w u8 rows (src pitch -> dst pitch), n images spaced by the strides.
cudaError_t copy_images(uint8_t* dst, size_t dst_stride, size_t dst_pitch, const uint8_t* src, size_t src_stride,
                        size_t src_pitch, int w, int h, int n, cudaMemcpyKind kind, cudaStream_t st) {
  if (dst_pitch == src_pitch && dst_pitch == static_cast<size_t>(w) &&
      (n == 1 || (dst_stride == src_stride && dst_stride == dst_pitch * h)))
    return cudaMemcpyAsync(dst, src, dst_pitch * h * n, kind, st);
  for (int i = 0; i < n; ++i) {
    const cudaError_t e =
        cudaMemcpy2DAsync(dst + i * dst_stride, dst_pitch, src + i * src_stride, src_pitch, w, h, kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Host frames [0, nframes) -> device ring -> batch kernel -> host, chunks of
// whole frames (~32 MiB: per-chunk host work is ~20 us, so config 5 runs at
// 92 % of the concurrent H2D + D2H bound with 32 MiB chunks against 86 % with
// 8 MiB; ramped chunk sizes and deeper rings measured no better,
// scripts/e2e_chunks.py). Caller validated the arguments.
dctf_status frames_host(const dctf_plan* const* plans, int nplans, const int* pof, const uint8_t* h_in,
                        uint8_t* h_out, int nframes, int w, int h, size_t pitch, size_t frame_stride,
                        int* launches) {
  *launches = 0;
  if (nframes == 0 || w == 0 || h == 0) return DCTF_OK;
  const size_t dpitch = (static_cast<size_t>(w) + 15) & ~size_t(15);
  const size_t fbytes = dpitch * static_cast<size_t>(h);
  const int cf = static_cast<int>(std::max<size_t>(1, std::min<size_t>(nframes, (size_t(32) << 20) / fbytes)));
  const int nch = (nframes + cf - 1) / cf;
  auto count = [&](int c) { return std::min(cf, nframes - c * cf); };
  return host_pipeline(
      plans[0]->device, nch, fbytes * cf,
      [&](int c, uint8_t* din, cudaStream_t st) {
        return copy_images(din, fbytes, dpitch, h_in + c * cf * frame_stride, frame_stride, pitch, w, h, count(c),
                           cudaMemcpyHostToDevice, st);
      },
      [&](int c, uint8_t* din, uint8_t* dout, cudaStream_t st) {
        dctf::reset_launches();
        const dctf_status x = dctf::filter_frames_device(plans, nplans, pof + c * cf, din, dout, count(c), w, h,
                                                         dpitch, fbytes, st);
        *launches += dctf_last_launch_count();
        return x;
      },
      [&](int c, uint8_t* dout, cudaStream_t st) {
        return copy_images(h_out + c * cf * frame_stride, frame_stride, pitch, dout, fbytes, dpitch, w, h, count(c),
                           cudaMemcpyDeviceToHost, st);
      });
}

}  // namespace

namespace dctf {
// The calling thread's compute stream on `device` (created once per thread
// and device) and a grow-only device scratch buffer of this thread on it:
// the per-block host entries (forward / inverse / filter_coeffs / convolve
// on host BlockMatrix batches) reuse both instead of creating a stream and
// allocating per call.
dctf_status thread_scratch(int device, size_t bytes, cudaStream_t* st, void** buf) {
  IoStreams* io = nullptr;
  const dctf_status s = io_streams(device, io);
  if (s != DCTF_OK) return s;
  *st = io->s[1];
  struct Scratch {
    std::vector<std::pair<void*, size_t>> per_dev;
    ~Scratch() {
      for (auto& b : per_dev)
        if (b.first) cudaFree(b.first);
    }
  };
  thread_local Scratch scratch;
  if (scratch.per_dev.size() <= static_cast<size_t>(device)) scratch.per_dev.resize(device + 1, {nullptr, 0});
  auto& b = scratch.per_dev[device];
  if (b.second < bytes) {
    if (b.first) {
      cudaStreamSynchronize(*st);
      cudaFree(b.first);
    }
    b = {nullptr, 0};
    const size_t want = std::max(bytes, size_t(1) << 20);
    if (cudaMalloc(&b.first, want) != cudaSuccess) return set_error(DCTF_CUDA_ERROR, "host scratch allocation failed");
    b.second = want;
  }
  *buf = b.first;
  return DCTF_OK;
}

// One image from / to host buffers through the copy-engine pipeline: bands of
// whole block rows (~16 MiB) are independent images (blocks never cross a
// band; the ragged bottom band replicates the image's last row exactly as
// tile() does). Per-call scratch and per-thread streams: concurrent callers
// on one plan do not serialise.
dctf_status image_host_copy(const dctf_plan* p, const uint8_t* h_in, uint8_t* h_out, int w, int h, size_t pitch,
                            int* launches) {
  *launches = 0;
  if (w == 0 || h == 0) return DCTF_OK;
  const int n = p->n, bh = (h + n - 1) / n;
  const size_t dpitch = (static_cast<size_t>(w) + 15) & ~size_t(15);
  const int brows = static_cast<int>(std::max<size_t>(1, std::min<size_t>(bh, (size_t(16) << 20) / (dpitch * n))));
  const int nch = (bh + brows - 1) / brows;
  auto rows = [&](int c) { return std::min(h, (c + 1) * brows * n) - c * brows * n; };
  return host_pipeline(
      p->device, nch, dpitch * brows * n,
      [&](int c, uint8_t* din, cudaStream_t st) {
        return copy_images(din, 0, dpitch, h_in + size_t(c) * brows * n * pitch, 0, pitch, w, rows(c), 1,
                           cudaMemcpyHostToDevice, st);
      },
      [&](int c, uint8_t* din, uint8_t* dout, cudaStream_t st) {
        dctf::reset_launches();
        const dctf_status x = filter_image_device(p, din, dout, w, rows(c), dpitch, 0, 1, nullptr, st);
        *launches += dctf_last_launch_count();
        return x;
      },
      [&](int c, uint8_t* dout, cudaStream_t st) {
        return copy_images(h_out + size_t(c) * brows * n * pitch, 0, pitch, dout, 0, dpitch, w, rows(c), 1,
                           cudaMemcpyDeviceToHost, st);
      });
}
}  // namespace dctf

namespace {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the optional gather is the only user).
struct NcclApi {
  typedef int (*InitAll)(void**, int, const int*);
  typedef int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
  typedef int (*Simple)();
  typedef int (*Destroy)(void*);
  typedef const char* (*ErrStr)(int);
  InitAll init_all = nullptr;
  AllGather all_gather = nullptr;
  Simple group_start = nullptr, group_end = nullptr;
  Destroy destroy = nullptr;
  ErrStr err = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.init_all = reinterpret_cast<NcclApi::InitAll>(dlsym(h, "ncclCommInitAll"));
    api.all_gather = reinterpret_cast<NcclApi::AllGather>(dlsym(h, "ncclAllGather"));
    api.group_start = reinterpret_cast<NcclApi::Simple>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<NcclApi::Simple>(dlsym(h, "ncclGroupEnd"));
    api.destroy = reinterpret_cast<NcclApi::Destroy>(dlsym(h, "ncclCommDestroy"));
    api.err = reinterpret_cast<NcclApi::ErrStr>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.init_all && api.all_gather && api.group_start && api.group_end && api.destroy && api.err;
  });
  return api;
}

// Runs fn(r) for every replica r on its own host thread (device set).
template <typename Fn>
dctf_status fan_out(const std::vector<int>& devices, Fn fn) {
  const int n = static_cast<int>(devices.size());
  std::vector<dctf_status> st(n, DCTF_OK);
  std::vector<std::string> msg(n);
  auto body = [&](int r) {
    DevGuard g(devices[r]);
    cudaFree(nullptr);  // make the device's primary context current on this thread (driver-API calls follow)
    st[r] = fn(r);
    if (st[r] != DCTF_OK) msg[r] = dctf_last_error_message();
  };
  if (n == 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (int r = 0; r < n; ++r) pool.emplace_back(body, r);
    for (auto& t : pool) t.join();
  }
  for (int r = 0; r < n; ++r)
    if (st[r] != DCTF_OK) return set_error(st[r], "replica " + std::to_string(r) + ": " + msg[r]);
  return DCTF_OK;
}

// Contiguous shard r of [0, total) over n replicas (sizes differ by at most 1).
inline int shard_lo(int total, int n, int r) { return static_cast<int>(static_cast<long long>(total) * r / n); }

dctf_status check_multi_list(const dctf_multi* const* ms, int nplans) {
  if (!ms || nplans < 1) return set_error(DCTF_INVALID_ARGUMENT, "bad plan list");
  for (int i = 0; i < nplans; ++i) {
    if (!ms[i]) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
    if (ms[i]->devices != ms[0]->devices) return set_error(DCTF_INVALID_ARGUMENT, "plans must share devices");
  }
  return DCTF_OK;
}

}  // namespace

extern "C" {

dctf_status dctf_filter_frames_host(const dctf_plan* const* plans, int nplans, const int* h_plan_of_frame,
                                    const uint8_t* h_in, uint8_t* h_out, int nframes, int width, int height,
                                    size_t pitch, size_t frame_stride) {
  dctf::NvtxRange nvtx_range("dctf_filter_frames_host");
  dctf::reset_launches();
  dctf_status s = check_frames(plans, nplans, h_plan_of_frame, nframes, width, height, pitch, frame_stride);
  if (s != DCTF_OK) return s;
  if (nframes > 0 && width > 0 && height > 0 && (!h_in || !h_out))
    return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  int launches = 0;
  s = frames_host(plans, nplans, h_plan_of_frame, h_in, h_out, nframes, width, height, pitch, frame_stride,
                  &launches);
  dctf::reset_launches();
  dctf::add_launches(launches);
  return s;
}

dctf_status dctf_multi_create(const double* h_weights, int kr, int kc, int n, int padding, int precision,
                              const int* devices, int ndevices, dctf_multi** out) {
  dctf::NvtxRange nvtx_range("dctf_multi_create");
  if (!out || !devices || ndevices < 1) return set_error(DCTF_INVALID_ARGUMENT, "bad device list");
  *out = nullptr;
  auto* m = new dctf_multi();
  m->devices.assign(devices, devices + ndevices);
  for (int r = 0; r < ndevices; ++r) {
    dctf_plan* p = nullptr;
    const dctf_status s = dctf_plan_create(h_weights, kr, kc, n, padding, precision, devices[r], &p);
    if (s != DCTF_OK) {
      const std::string msg = dctf_last_error_message();
      dctf_multi_destroy(m);
      return set_error(s, msg);
    }
    m->replicas.push_back(p);
  }
  *out = m;
  return DCTF_OK;
}

dctf_status dctf_multi_destroy(dctf_multi* m) {
  if (!m) return DCTF_OK;
  for (dctf_plan* p : m->replicas) dctf_plan_destroy(p);
  delete m;
  return DCTF_OK;
}

dctf_status dctf_multi_info(const dctf_multi* m, int* ndevices, const dctf_plan** replica0) {
  if (!m) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  if (ndevices) *ndevices = static_cast<int>(m->replicas.size());
  if (replica0) *replica0 = m->replicas[0];
  return DCTF_OK;
}

dctf_status dctf_multi_replica(const dctf_multi* m, int r, const dctf_plan** out) {
  if (!m || !out || r < 0 || r >= static_cast<int>(m->replicas.size()))
    return set_error(DCTF_INVALID_ARGUMENT, "bad replica index");
  *out = m->replicas[r];
  return DCTF_OK;
}

dctf_status dctf_filter_image_host_multi(const dctf_multi* m, const uint8_t* h_in, uint8_t* h_out, int width,
                                         int height, size_t pitch) {
  dctf::NvtxRange nvtx_range("dctf_filter_image_host_multi");
  dctf::reset_launches();
  if (!m) return set_error(DCTF_INVALID_ARGUMENT, "plan is NULL");
  if (width < 0 || height < 0) return set_error(DCTF_INVALID_ARGUMENT, "image dimensions must be >= 0");
  if (height > 0 && pitch < static_cast<size_t>(width)) return set_error(DCTF_INVALID_ARGUMENT, "pitch < width");
  if (width == 0 || height == 0) return DCTF_OK;
  if (!h_in || !h_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  const int nrep = static_cast<int>(m->replicas.size()), n = m->replicas[0]->n;
  const int bh = (height + n - 1) / n;
  // block-row band r; a band is an image of its own (rows are whole blocks,
  // except the ragged last band, whose edge replication tile() applies
  // identically inside it)
  std::vector<int> nl(nrep, 0);
  const dctf_status s = fan_out(m->devices, [&](int r) {
    const int b0 = shard_lo(bh, nrep, r), b1 = shard_lo(bh, nrep, r + 1);
    if (b1 <= b0) return DCTF_OK;
    const int y0 = b0 * n, rows = std::min(height, b1 * n) - y0;
    const dctf_status st = dctf_filter_image_host(m->replicas[r], h_in + y0 * pitch, h_out + y0 * pitch, width,
                                                  rows, pitch);
    nl[r] = dctf_last_launch_count();
    return st;
  });
  dctf::reset_launches();
  for (int v : nl) dctf::add_launches(v);
  return s;
}

dctf_status dctf_filter_frames_host_multi(const dctf_multi* const* ms, int nplans, const int* h_plan_of_frame,
                                          const uint8_t* h_in, uint8_t* h_out, int nframes, int width, int height,
                                          size_t pitch, size_t frame_stride) {
  dctf::NvtxRange nvtx_range("dctf_filter_frames_host_multi");
  dctf::reset_launches();
  dctf_status s = check_multi_list(ms, nplans);
  if (s != DCTF_OK) return s;
  const int nrep = static_cast<int>(ms[0]->replicas.size());
  std::vector<std::vector<const dctf_plan*>> per(nrep);
  for (int r = 0; r < nrep; ++r)
    for (int i = 0; i < nplans; ++i) per[r].push_back(ms[i]->replicas[r]);
  s = check_frames(per[0].data(), nplans, h_plan_of_frame, nframes, width, height, pitch, frame_stride);
  if (s != DCTF_OK) return s;
  if (nframes > 0 && width > 0 && height > 0 && (!h_in || !h_out))
    return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
  std::vector<int> nl(nrep, 0);
  s = fan_out(ms[0]->devices, [&](int r) {
    const int f0 = shard_lo(nframes, nrep, r), f1 = shard_lo(nframes, nrep, r + 1);
    return frames_host(per[r].data(), nplans, h_plan_of_frame + f0, h_in + f0 * frame_stride,
                       h_out + f0 * frame_stride, f1 - f0, width, height, pitch, frame_stride, &nl[r]);
  });
  dctf::reset_launches();
  for (int v : nl) dctf::add_launches(v);
  return s;
}

dctf_status dctf_filter_frames_u8_multi(const dctf_multi* const* ms, int nplans, const int* h_plan_of_frame,
                                        const uint8_t* const* d_in, uint8_t* const* d_out, int nframes, int width,
                                        int height, size_t pitch, size_t frame_stride, uint8_t* const* d_gather,
                                        void* const* streams) {
  dctf::NvtxRange nvtx_range("dctf_filter_frames_u8_multi");
  dctf::reset_launches();
  dctf_status s = check_multi_list(ms, nplans);
  if (s != DCTF_OK) return s;
  if (!d_in || !d_out) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer list");
  const int nrep = static_cast<int>(ms[0]->replicas.size());
  std::vector<std::vector<const dctf_plan*>> per(nrep);
  for (int r = 0; r < nrep; ++r)
    for (int i = 0; i < nplans; ++i) per[r].push_back(ms[i]->replicas[r]);
  s = check_frames(per[0].data(), nplans, h_plan_of_frame, nframes, width, height, pitch, frame_stride);
  if (s != DCTF_OK) return s;
  if (d_gather && nframes % nrep != 0)
    return set_error(DCTF_INVALID_ARGUMENT, "gather needs equal shards (nframes % ndevices == 0)");
  std::vector<int> nl(nrep, 0);
  s = fan_out(ms[0]->devices, [&](int r) {
    const int f0 = shard_lo(nframes, nrep, r), f1 = shard_lo(nframes, nrep, r + 1);
    if (f1 <= f0 || width == 0 || height == 0) return DCTF_OK;
    if (!d_in[r] || !d_out[r]) return set_error(DCTF_INVALID_ARGUMENT, "NULL buffer");
    dctf::reset_launches();
    const cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[r]) : nullptr;
    const dctf_status x = dctf::filter_frames_device(per[r].data(), nplans, h_plan_of_frame + f0, d_in[r], d_out[r],
                                                     f1 - f0, width, height, pitch, frame_stride, st);
    nl[r] = dctf_last_launch_count();
    return x;
  });
  dctf::reset_launches();
  for (int v : nl) dctf::add_launches(v);
  if (s != DCTF_OK || !d_gather || nframes == 0) return s;
  // optional all-gather of the equal shards: d_gather[r] receives all frames
  const NcclApi& api = nccl();
  if (!api.ok) return set_error(DCTF_UNSUPPORTED, "gather: libnccl.so.2 not loadable");
  for (int r = 0; r < nrep; ++r)
    for (int q = 0; q < r; ++q)
      if (ms[0]->devices[q] == ms[0]->devices[r])
        return set_error(DCTF_UNSUPPORTED, "gather: NCCL needs distinct devices per replica");
  std::vector<void*> comms(nrep, nullptr);
  int rc = api.init_all(comms.data(), nrep, ms[0]->devices.data());
  if (rc != 0) return set_error(DCTF_CUDA_ERROR, std::string("ncclCommInitAll: ") + api.err(rc));
  const size_t shard = static_cast<size_t>(nframes / nrep) * frame_stride;
  api.group_start();
  for (int r = 0; r < nrep && rc == 0; ++r) {
    DevGuard g(ms[0]->devices[r]);
    const cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[r]) : nullptr;
    rc = api.all_gather(d_out[r], d_gather[r], shard, /*ncclUint8*/ 1, comms[r], st);
  }
  const int rc2 = api.group_end();
  for (int r = 0; r < nrep; ++r) {
    DevGuard g(ms[0]->devices[r]);
    const cudaStream_t st = streams ? static_cast<cudaStream_t>(streams[r]) : nullptr;
    cudaStreamSynchronize(st);
    api.destroy(comms[r]);
  }
  if (rc != 0 || rc2 != 0) return set_error(DCTF_CUDA_ERROR, std::string("ncclAllGather: ") + api.err(rc ? rc : rc2));
  return DCTF_OK;
}

}  // extern "C"
