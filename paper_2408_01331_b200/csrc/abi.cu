// C-ABI plumbing: error state, the per-step schedule prologue and the batch gather.
#include <cstring>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace hnn {

static thread_local std::string g_last_error;

void set_error(const char* where, const char* what) {
  g_last_error = std::string(where) + ": " + what;
}

int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(where, cudaGetErrorString(e));
    return HNN_ERR_CUDA;
  }
  return HNN_OK;
}

// sched row block `*counter` -> cur, then advance.  One block; n_models*12 words.
__global__ void step_begin_kernel(const hnn_step_row* __restrict__ sched, int32_t* counter,
                                  hnn_step_row* __restrict__ cur, int n_models) {
  hnn::pdl_wait();
  const int step = *counter;
  const int words = n_models * int(sizeof(hnn_step_row) / 4);
  const int32_t* src = reinterpret_cast<const int32_t*>(sched + size_t(step) * n_models);
  int32_t* dst = reinterpret_cast<int32_t*>(cur);
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) *counter = step + 1;
}

// One warp per (row, problem), 8 rows per block: dst row r <- src row perm[perm_base + r]; rows
// >= R zero-filled.  A warp's float4 loads of its row are all in flight together (a block per
// row left one permutation lookup + one short copy per 128 threads: 2 TB/s).
constexpr int GATHER_ROWS = 8;

__global__ void __launch_bounds__(32 * GATHER_ROWS) gather_rows_kernel(const hnn_gather_problem* __restrict__ probs,
                                                                       const hnn_step_row* __restrict__ cur) {
  hnn::pdl_wait();
  const hnn_gather_problem& p = probs[blockIdx.y];
  const int lane = threadIdx.x % 32;
  const int r = blockIdx.x * GATHER_ROWS + threadIdx.x / 32;
  if (r >= p.cap || !cur[p.model].active) return;
  const int rows = cur[p.model].rows;
  float* dst = p.dst_x + size_t(r) * p.ld_dst;
  if (r >= rows) {
    for (int i = lane; i < p.ld_dst; i += 32) dst[i] = 0.0f;
    if (lane == 0) p.dst_y[r] = 0;
    return;
  }
  const int src_row = p.perm[cur[p.model].perm_base + r];
  const float* src = p.src_x + size_t(src_row) * p.sample;
  const bool vec = ((p.sample & 3) == 0) && ((p.ld_dst & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(p.src_x) & 15) == 0) && ((reinterpret_cast<uintptr_t>(p.dst_x) & 15) == 0);
  if (vec) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = p.sample / 4;
    int i = lane;
    for (; i + 224 < n4; i += 256) {  // 8 independent 16-byte loads per lane per round
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(s4 + i + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) d4[i + 32 * u] = v[u];
    }
    {  // the rest (an MNIST row: 196 float4 = 6.1 per lane) in one round as well
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = i + 32 * u < n4 ? __ldg(s4 + i + 32 * u) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + 32 * u < n4) d4[i + 32 * u] = v[u];
    }
  } else {
    for (int i = lane; i < p.sample; i += 32) dst[i] = __ldg(src + i);
  }
  for (int i = p.sample + lane; i < p.ld_dst; i += 32) dst[i] = 0.0f;
  if (lane == 0) p.dst_y[r] = p.src_y[src_row];
}

}  // namespace hnn

extern "C" {

const char* hnn_last_error(void) { return hnn::g_last_error.c_str(); }

const char* hnn_version(void) { return "hnn_b200 1.0 sm_100a"; }

int hnn_struct_size(const char* name) {
  if (!name) return -1;
  if (!strcmp(name, "hnn_step_row")) return sizeof(hnn_step_row);
  if (!strcmp(name, "hnn_model_status")) return sizeof(hnn_model_status);
  if (!strcmp(name, "hnn_gather_problem")) return sizeof(hnn_gather_problem);
  if (!strcmp(name, "hnn_gemm_problem")) return sizeof(hnn_gemm_problem);
  if (!strcmp(name, "hnn_conv_problem")) return sizeof(hnn_conv_problem);
  if (!strcmp(name, "hnn_pool_problem")) return sizeof(hnn_pool_problem);
  if (!strcmp(name, "hnn_relu_problem")) return sizeof(hnn_relu_problem);
  if (!strcmp(name, "hnn_sce_problem")) return sizeof(hnn_sce_problem);
  if (!strcmp(name, "hnn_opt_segment")) return sizeof(hnn_opt_segment);
  if (!strcmp(name, "hnn_host_gather_item")) return sizeof(hnn_host_gather_item);
  if (!strcmp(name, "hnn_hostfed_io")) return sizeof(hnn_hostfed_io);
  if (!strcmp(name, "hnn_tail_problem")) return sizeof(hnn_tail_problem);
  if (!strcmp(name, "hnn_convtc_problem")) return sizeof(hnn_convtc_problem);
  if (!strcmp(name, "hnn_embed_problem")) return sizeof(hnn_embed_problem);
  return -1;
}

int hnn_step_begin(const hnn_step_row* sched, int32_t* counter, hnn_step_row* cur, int n_models, void* stream) {
  HNN_REQUIRE(sched && counter && cur && n_models > 0, "hnn_step_begin", "null pointer or empty model set");
  hnn::launch_pdl(hnn::step_begin_kernel, dim3(1), dim3(256), 0, hnn::as_stream(stream), sched, counter, cur, n_models);
  return hnn::check_launch("hnn_step_begin");
}

int hnn_gather_rows(const hnn_gather_problem* probs, int nprob, int max_cap, const hnn_step_row* cur,
                    void* stream) {
  HNN_REQUIRE(probs && cur && nprob > 0 && max_cap > 0, "hnn_gather_rows", "bad arguments");
  HNN_REQUIRE(nprob <= 65535, "hnn_gather_rows", "too many problems");
  dim3 grid((max_cap + hnn::GATHER_ROWS - 1) / hnn::GATHER_ROWS, nprob);
  hnn::launch_pdl(hnn::gather_rows_kernel, dim3(grid), dim3(32 * hnn::GATHER_ROWS), 0, hnn::as_stream(stream), probs, cur);
  return hnn::check_launch("hnn_gather_rows");
}

int hnn_host_gather_rows(float* dst_x, int64_t ld_dst, int32_t* dst_y, const float* src_x, int64_t ld_src,
                         const float* src_y, const int64_t* idx, int64_t n, int64_t cols) {
  HNN_REQUIRE(dst_x && dst_y && src_x && src_y && (idx || n == 0) && n >= 0 && cols >= 0 && ld_dst >= cols &&
                  ld_src >= cols,
              "hnn_host_gather_rows", "bad arguments");
  const size_t bytes = size_t(cols) * sizeof(float);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = idx[r];
    std::memcpy(dst_x + r * ld_dst, src_x + i * ld_src, bytes);
    dst_y[r] = static_cast<int32_t>(src_y[i]);
  }
  return HNN_OK;
}

}  // extern "C"

// Persistent host worker pool for the loader's per-step gather: spawning and joining threads per
// call cost ~0.1 ms per step (the bound of the small configs' end-to-end step).  One job at a time
// (a mutex serialises callers); the caller runs piece 0..n-1 alongside the workers.
namespace {
struct HostPool {
  std::mutex run_m, m;
  std::condition_variable cv, done_cv;
  std::vector<std::thread> workers;
  std::function<void(int)> job;
  int pieces = 0, remaining = 0;
  std::atomic<int> next{0};
  uint64_t gen = 0;

  void pieces_loop() {
    for (int i; (i = next.fetch_add(1)) < pieces;) {
      job(i);
      std::lock_guard<std::mutex> lk(m);
      if (--remaining == 0) done_cv.notify_all();
    }
  }
  void worker() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m);
    for (;;) {
      cv.wait(lk, [&] { return gen != seen; });
      seen = gen;
      lk.unlock();
      pieces_loop();
      lk.lock();
    }
  }
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> serial(run_m);
    {
      std::unique_lock<std::mutex> lk(m);
      while (int(workers.size()) < n - 1) {
        workers.emplace_back([this] { worker(); });
        workers.back().detach();  // (never joined: idle workers must not block process exit)
      }
      job = fn;
      pieces = n;
      remaining = n;
      next.store(0);
      ++gen;
    }
    cv.notify_all();
    pieces_loop();
    std::unique_lock<std::mutex> lk(m);
    done_cv.wait(lk, [&] { return remaining == 0; });
  }
};
HostPool& host_pool() {
  static HostPool* p = new HostPool();  // (leaked on purpose: no destructor runs at exit)
  return *p;
}
}  // namespace

static void host_pool_run(int n, const std::function<void(int)>& fn) { host_pool().run(n, fn); }

extern "C" {

int hnn_host_gather_batch(const hnn_host_gather_item* items, int n_items, int threads) {
  HNN_REQUIRE(items && n_items >= 0 && threads >= 1 && threads <= 64, "hnn_host_gather_batch", "bad arguments");
  std::vector<int64_t> start(size_t(n_items) + 1, 0);  // prefix sums of the rows each item writes
  for (int i = 0; i < n_items; ++i) {
    const hnn_host_gather_item& it = items[i];
    HNN_REQUIRE(it.dst_x && it.dst_y && it.src_x && it.src_y && (it.idx || it.n == 0) && it.n >= 0 &&
                    it.cap >= it.n && it.cols >= 0 && it.ld_dst >= it.cols && it.ld_src >= it.cols,
                "hnn_host_gather_batch", "bad item");
    start[i + 1] = start[i] + it.cap;
  }
  const int64_t total = start[n_items];
  auto work = [&](int64_t r0, int64_t r1) {
    int i = int(std::upper_bound(start.begin(), start.end(), r0) - start.begin()) - 1;
    for (int64_t g = r0; g < r1;) {
      while (g >= start[i + 1]) ++i;
      const hnn_host_gather_item& it = items[i];
      const int64_t end = std::min(r1, start[i + 1]);
      for (; g < end; ++g) {
        const int64_t r = g - start[i];
        float* dst = it.dst_x + r * it.ld_dst;
        if (r < it.n) {
          const int64_t j = it.idx[r];
          std::memcpy(dst, it.src_x + j * it.ld_src, size_t(it.cols) * sizeof(float));
          it.dst_y[r] = static_cast<int32_t>(it.src_y[j]);
        } else {
          std::memset(dst, 0, size_t(it.cols) * sizeof(float));
          it.dst_y[r] = 0;
        }
      }
    }
  };
  const int nt = int(std::min<int64_t>(threads, std::max<int64_t>(1, total / 64)));
  if (nt <= 1) {
    work(0, total);
    return HNN_OK;
  }
  host_pool_run(nt, [&](int t) { work(total * t / nt, total * (t + 1) / nt); });
  return HNN_OK;
}

// ---------------------------------------------------------------- host-fed step (one native call)
// The public host-fed step's stream work without per-step Python (train.HostFedStepper, fast path):
// copy stream: wait until staging slot k is free, H2D of the pinned batch into it, record ready[k];
// compute stream: wait ready[k], move the staged batch into the arenas, record free[k], launch the
// captured step graph, D2H the per-model outputs.  Events live in the context.
struct HostFed {
  cudaEvent_t ready[2], free_[2];
  bool used[2];
};

int hnn_hostfed_create(void** out) {
  HNN_REQUIRE(out, "hnn_hostfed_create", "null output");
  HostFed* h = new HostFed();
  for (int k = 0; k < 2; ++k) {
    if (cudaEventCreateWithFlags(&h->ready[k], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->free_[k], cudaEventDisableTiming) != cudaSuccess) {
      hnn::set_error("hnn_hostfed_create", "cudaEventCreate failed");
      delete h;
      return HNN_ERR_CUDA;
    }
    h->used[k] = false;
  }
  *out = h;
  return HNN_OK;
}

int hnn_hostfed_destroy(void* ctx) {
  HostFed* h = static_cast<HostFed*>(ctx);
  if (!h) return HNN_OK;
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(h->ready[k]);
    cudaEventDestroy(h->free_[k]);
  }
  delete h;
  return HNN_OK;
}

int hnn_hostfed_step(void* ctx, int slot, const hnn_hostfed_io* io, void* graph_exec, void* compute_stream,
                     void* copy_stream, void** copied_event) {
  HostFed* h = static_cast<HostFed*>(ctx);
  HNN_REQUIRE(h && io && graph_exec && (slot == 0 || slot == 1), "hnn_hostfed_step", "bad arguments");
  cudaStream_t cs = hnn::as_stream(compute_stream), xs = hnn::as_stream(copy_stream);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
  };
  if (h->used[slot]) ok(cudaStreamWaitEvent(xs, h->free_[slot], 0));  // step t-2 moved its batch out
  ok(cudaMemcpyAsync(io->stage_x, io->host_x, size_t(io->x_bytes), cudaMemcpyHostToDevice, xs));
  ok(cudaMemcpyAsync(io->stage_y, io->host_y, size_t(io->y_bytes), cudaMemcpyHostToDevice, xs));
  ok(cudaEventRecord(h->ready[slot], xs));
  ok(cudaStreamWaitEvent(cs, h->ready[slot], 0));
  ok(cudaMemcpyAsync(io->arena_x, io->stage_x, size_t(io->x_bytes), cudaMemcpyDeviceToDevice, cs));
  ok(cudaMemcpyAsync(io->arena_y, io->stage_y, size_t(io->y_bytes), cudaMemcpyDeviceToDevice, cs));
  ok(cudaEventRecord(h->free_[slot], cs));
  h->used[slot] = true;
  ok(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), cs));
  for (int i = 0; i < 2; ++i)
    if (io->out_bytes[i] > 0)
      ok(cudaMemcpyAsync(io->out_host[i], io->out_dev[i], size_t(io->out_bytes[i]), cudaMemcpyDeviceToHost, cs));
  if (copied_event) *copied_event = h->ready[slot];
  if (e != cudaSuccess) {
    hnn::set_error("hnn_hostfed_step", cudaGetErrorString(e));
    return HNN_ERR_CUDA;
  }
  return HNN_OK;
}

int hnn_event_synchronize(void* event) {
  HNN_REQUIRE(event, "hnn_event_synchronize", "null event");
  const cudaError_t e = cudaEventSynchronize(static_cast<cudaEvent_t>(event));
  if (e != cudaSuccess) {
    hnn::set_error("hnn_event_synchronize", cudaGetErrorString(e));
    return HNN_ERR_CUDA;
  }
  return HNN_OK;
}

}  // extern "C"
