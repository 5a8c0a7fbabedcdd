// C ABI (include/tacho_b200.h): host flattener, device context and the
// analysis helpers. No exception crosses this file's extern "C" functions.
#include "../../include/tacho_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <new>
#include <string>

#include "device/device_api.hpp"
#include "host/flow_plan.hpp"
#include "host/plan.hpp"
#include "host/sparse.hpp"

namespace {

thread_local std::string g_plan_error;
thread_local std::string g_tch_error;

tcb::CsrMatrix csr_from_view(const tcg_csr_view* v, bool need_values) {
  if (!v || v->n < 0 || v->nnz < 0 || (!v->row_ptr && v->n > 0))
    throw std::invalid_argument("csr view: null or negative sizes");
  tcb::CsrMatrix m;
  m.nrows = m.ncols = v->n;
  m.row_ptr.assign(v->row_ptr, v->row_ptr + v->n + 1);
  if (v->nnz > 0) {
    if (!v->col_idx) throw std::invalid_argument("csr view: null col_idx");
    m.col_idx.assign(v->col_idx, v->col_idx + v->nnz);
  }
  if (v->values && v->nnz > 0)
    m.values.assign(v->values, v->values + v->nnz);
  else if (need_values && v->nnz > 0)
    throw std::invalid_argument("csr view: values required");
  else
    m.values.assign(static_cast<std::size_t>(v->nnz), 1.0);
  if (v->n == 0 && m.row_ptr.empty()) m.row_ptr.assign(1, 0);
  tcb::validate_csr(m);
  return m;
}

void view_of(const tcb::CsrMatrix& m, tcg_csr_view* out) {
  out->n = m.nrows;
  out->nnz = m.nnz();
  out->row_ptr = m.row_ptr.data();
  out->col_idx = m.col_idx.data();
  out->values = m.values.data();
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Device blocks of the arenas, kept for reuse after a context frees them (a
// one-shot call allocates and frees a few hundred MB to ~2 GB each time;
// cudaMalloc / cudaFree of that much took 10-300 ms on B200 boxes). A request
// takes a cached block of at least its size and at most 25% larger; at most
// 8 GB stay cached per device; TCG_DEVICE_CACHE=0 turns the cache off. A
// block is only returned once its stream's work is done (callers synchronise).
struct DeviceCache {
  std::mutex mu;
  std::map<int, std::multimap<size_t, void*>> free_blocks;  // device -> size -> block
  std::map<void*, std::pair<int, size_t>> size_of;          // block -> (device, bytes)
  std::map<int, size_t> cached;
  static constexpr size_t kCap = size_t{8} << 30;
};
DeviceCache& device_cache() {
  static DeviceCache* c = new DeviceCache();  // never destroyed: blocks live until the process exits
  return *c;
}
bool cache_on() {
  static const bool on = [] {
    const char* e = std::getenv("TCG_DEVICE_CACHE");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

cudaError_t dev_alloc(int device, void** p, size_t bytes) {
  bytes = align_up(std::max<size_t>(bytes, 1), size_t{1} << 20);
  DeviceCache& dc = device_cache();
  if (cache_on()) {
    std::lock_guard<std::mutex> lock(dc.mu);
    auto& fl = dc.free_blocks[device];
    auto it = fl.lower_bound(bytes);
    if (it != fl.end() && it->first <= bytes + bytes / 4) {
      *p = it->second;
      dc.cached[device] -= it->first;
      fl.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation && cache_on()) {  // give the cached blocks back and retry
    cudaGetLastError();
    std::lock_guard<std::mutex> lock(dc.mu);
    for (auto& kv : dc.free_blocks[device]) {
      cudaFree(kv.second);
      dc.size_of.erase(kv.second);
    }
    dc.free_blocks[device].clear();
    dc.cached[device] = 0;
    e = cudaMalloc(p, bytes);
  }
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lock(dc.mu);
    dc.size_of[*p] = {device, bytes};
  }
  return e;
}

void dev_free(void* p) {
  if (!p) return;
  DeviceCache& dc = device_cache();
  std::lock_guard<std::mutex> lock(dc.mu);
  auto it = dc.size_of.find(p);
  if (it == dc.size_of.end() || !cache_on()) {
    if (it != dc.size_of.end()) dc.size_of.erase(it);
    cudaFree(p);
    return;
  }
  const int device = it->second.first;
  const size_t bytes = it->second.second;
  auto& fl = dc.free_blocks[device];
  while (dc.cached[device] + bytes > DeviceCache::kCap && !fl.empty()) {  // make room: largest first
    auto big = std::prev(fl.end());
    dc.cached[device] -= big->first;
    dc.size_of.erase(big->second);
    cudaFree(big->second);
    fl.erase(big);
  }
  if (bytes > DeviceCache::kCap) {
    dc.size_of.erase(it);
    cudaFree(p);
    return;
  }
  fl.emplace(bytes, p);
  dc.cached[device] += bytes;
}

}  // namespace

// A plan holds the lean value-flow plan (flow_plan.hpp: initial values and
// the schedule, O(nnz) host work; U's transposed index and the update
// programs are built on the device by tcg_upload) and, only when asked for,
// the full task-DAG plan (plan.hpp: block layout, the reference's DAG, the
// task executors' tables, sharded parts), built from the lean plan's copy of
// the pattern.
struct tcg_plan {
  tcb::FlowPlan flow;
  tcb::RangeList ranges;
  mutable std::unique_ptr<tcb::Plan> full;
  std::map<std::int32_t, tcb::FlowPart> parts;  // tcg_plan_part_problem results
  std::vector<std::int32_t> part_owner;         // the owner table of the last part problem
};

namespace {
// the full task-DAG plan (built on first use)
tcb::Plan& full_plan(const tcg_plan* plan) {
  if (!plan->full) {
    tcb::PlanOptions po;
    if (const char* e = std::getenv("TCG_CTA_COST")) po.cta_cost = std::max(1.0, std::atof(e));
    if (const char* e = std::getenv("TCG_MAX_WIDTH")) po.max_width = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("TCG_DEP_WIDE_COST")) po.dep_wide_cost = std::max(1.0, std::atof(e));
    plan->full = std::make_unique<tcb::Plan>(
        tcb::build_plan(tcb::flow_plan_pattern(plan->flow),
                        std::vector<double>(plan->flow.values.begin(), plan->flow.values.end()), plan->ranges,
                        true, po));
  }
  return *plan->full;
}

tcb::CsrRef ref_of(const tcg_csr_view* v) {
  if (!v || v->n < 0 || v->nnz < 0 || (!v->row_ptr && v->n > 0))
    throw std::invalid_argument("csr view: null or negative sizes");
  static const int64_t zero = 0;
  tcb::CsrRef r;
  r.n = v->n;
  r.nnz = v->nnz;
  r.row_ptr = v->row_ptr ? v->row_ptr : &zero;
  r.col_idx = v->col_idx;
  r.values = v->values;
  return r;
}
}  // namespace

struct tcg_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  // end to end with a pinned output: best whole-call ms of a copy after the
  // launch (0), the drain CTAs (1) and the chunked copies (2) over the first
  // calls of a problem and batch size (taking turns)
  float drain_ms[3] = {-1.f, -1.f, -1.f};
  int drain_calls = 0;
  // chunked download (run_flow, mode 2): chunk starts (host, nchunks + 1), device
  // counters (units per chunk, and the working copy), host-mapped flags
  int nchunks = 0;
  bool chunks_ready = false;
  std::vector<std::int64_t> chunk_start;
  int* chunk_units = nullptr;
  int* chunk_left = nullptr;
  int* chunk_flag = nullptr;    // pinned, mapped
  int* chunk_flag_d = nullptr;  // its device address
  int chunk_seq = 0;
  void* arena = nullptr;
  size_t arena_bytes = 0;
  tcbdev::Ctrl* host_ctrl = nullptr;
  // arena carve-out
  int* cols = nullptr;
  double* vals = nullptr;
  double* vals0 = nullptr;
  int4* tasks = nullptr;
  int4* items = nullptr;
  int4* srcs = nullptr;
  int4* succ = nullptr;  // 4 int4 per edge (kSuccWords)
  int* indeg = nullptr;
  int* indeg0 = nullptr;
  int* queue = nullptr;
  int* roots = nullptr;
  int* claim = nullptr;
  int* fin = nullptr;
  int* iflag = nullptr;
  int4* slot_rec = nullptr;
  int2* upd = nullptr;
  bool has_programs = false;
  int4* flow_rec = nullptr;  // value-flow schedule (mode 5)
  int* flow_item = nullptr;
  int* a_map = nullptr;      // device init_factor_values (in the arena)
  // pipelined batches end to end (run_flow_chunked): copy streams, per-chunk
  // events and status words
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  tcbdev::Ctrl* host_ctrls = nullptr;
  int host_ctrls_len = 0;
  double* a_stage = nullptr; // staging for A's values (separate allocation, grown on demand)
  unsigned* drain_done = nullptr;  // end-to-end drain: groups copied per 2,048 values
  std::int64_t drain_len = 0;
  std::int64_t nnz_a = 0, a_stage_len = 0;
  double** peers = nullptr;  // sharded runs: device table of every part's U (own included)
  int npeers = 0;
  std::vector<void*> ipc_opened;  // peer arenas mapped by tcg_ipc_open
  int* m_flags = nullptr;    // per member: breakdown latch, row (2 ints) + pivot (below)
  double* m_pivot = nullptr;
  // batch of value sets sharing the pattern (mode 5); separate allocation
  int nbatch = 1;
  void* batch_arena = nullptr;
  double* bvals = nullptr;   // nbatch x nnz working values
  double* bvals0 = nullptr;  // nbatch x nnz initial values
  double* ba = nullptr;      // nbatch x nnz prelude snapshot
  int* bm_flags = nullptr;
  double* bm_pivot = nullptr;
  int4* flow_slot = nullptr;
  int2* flow_upd = nullptr;
  int* flow_ub = nullptr;      // per coordinate: first product in flow_upd (nnz + 1), in prog_arena
  void* prog_arena = nullptr;  // device-built (m, o) pairs (their count is known after the count pass)
  double prog_build_ms = 0.0;
  int ub_total = 0;            // host source of flow_ub[nnz]
  int flow_depth = 0;          // longest chain of the schedule built on the device (0: built on the host)  // device time of the last program build
  double* flow_a = nullptr;  // snapshot of the input values
  std::int64_t nflow = 0, nflow_upd = 0;
  bool has_flow = false;
  std::int64_t nslots = 0, nupdates = 0;
  tcbdev::Ctrl* ctrl = nullptr;
  unsigned long long* trace = nullptr;
  // problem shape
  std::int64_t ntab = 0;  // tasks with device tables (modes 1/2: the task-DAG plan was uploaded)
  std::int64_t n = 0, nnz = 0, ntasks = 0, nitems = 0, nsrc = 0, nedges = 0, nroots = 0;
  std::int64_t qcap = 0;
  int epoch = 0;
  int max_target_len = 0, max_flag_rows = 0;
  bool uploaded = false;
  // the working values equal their restore copy (after upload, set_values,
  // restore): mode 5 then reads its input from the copy instead of
  // snapshotting the working values first
  bool pristine = false;
  tcg_options opt{};
  std::string err;
};

#define TCG_CUDA_TRY(ctx, call)                                              \
  do {                                                                       \
    cudaError_t e__ = (call);                                                \
    if (e__ != cudaSuccess) {                                                \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e__);      \
      return TCG_CUDA;                                                       \
    }                                                                        \
  } while (0)

extern "C" {

// ---------------------------------------------------------------- plan ----

tcg_status tcg_plan_build(const tcg_csr_view* a_permuted, const tcg_csr_view* pattern,
                          int32_t nranges, const int32_t* range_bounds, tcg_plan** out) {
  if (!out) return TCG_INVALID;
  *out = nullptr;
  try {
    const tcb::CsrRef a = ref_of(a_permuted), u = ref_of(pattern);
    if (nranges < 0 || (nranges > 0 && !range_bounds))
      throw std::invalid_argument("range list: null bounds");
    auto p = std::make_unique<tcg_plan>();
    for (int32_t r = 0; r < nranges; ++r) p->ranges.ranges.push_back({range_bounds[r], range_bounds[r + 1]});
    // the schedule is built on the device at upload unless TCG_HOST_SCHEDULE asks for the host
    const char* hs = std::getenv("TCG_HOST_SCHEDULE");
    p->flow = tcb::build_flow_plan(a, u, p->ranges, hs && std::atoi(hs) != 0);
    *out = p.release();
    return TCG_OK;
  } catch (const std::bad_alloc&) {
    g_plan_error = "out of host memory";
    return TCG_INVALID;
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
}

tcg_status tcg_plan_schedule(tcg_plan* plan) {
  if (!plan) return TCG_INVALID;
  try {
    tcb::flow_plan_schedule(plan->flow);
    return TCG_OK;
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
}

tcg_status tcg_plan_expand(tcg_plan* plan) {
  if (!plan) return TCG_INVALID;
  try {
    full_plan(plan);
    return TCG_OK;
  } catch (const std::bad_alloc&) {
    g_plan_error = "out of host memory";
    return TCG_INVALID;
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
}

void tcg_plan_free(tcg_plan* plan) { delete plan; }
const char* tcg_plan_error(void) { return g_plan_error.c_str(); }

tcg_status tcg_plan_problem(const tcg_plan* plan, tcg_problem* o) {
  if (!plan || !o) return TCG_INVALID;
  *o = tcg_problem{};
  const tcb::FlowPlan& F = plan->flow;
  o->n = F.n;
  o->nnz = F.nnz;
  o->col_idx = F.cols.data();
  o->values = F.values.data();
  o->nnz_a = F.a_map.empty() ? 0 : F.nnz_a;
  o->a_map = F.a_map.empty() ? nullptr : F.a_map.data();
  o->ntasks = F.stats.tasks[0] + F.stats.tasks[1] + F.stats.tasks[2] + F.stats.tasks[3];
  // the value-flow schedule with device-built programs (the default executor)
  o->nflow = F.stats.units;
  o->flow_rec = F.scheduled ? F.rec.data() : nullptr;  // else the device builds the schedule
  o->flow_item = F.scheduled ? F.unit.data() : nullptr;
  o->u_first = F.ufirst.data();
  o->u_tb = F.u_tb.data();
  o->u_len = F.u_len.data();
  o->u_row = F.u_row.data();
  o->flow_devprog = 1;
  o->u_row_ptr = F.row_ptr.data();
  o->flow_part = -1;
  if (!plan->full) return TCG_OK;
  // the task executors' tables (modes 1, 2) when the full plan exists
  const tcb::Plan& P = *plan->full;
  o->ntasks = static_cast<int64_t>(P.node_kind.size());
  o->task_rec = P.task_rec.data();
  o->nitems = static_cast<int64_t>(P.item_rec.size() / tcb::kItemWords);
  o->item_rec = P.item_rec.data();
  o->nsources = static_cast<int64_t>(P.src_rec.size() / tcb::kSrcWords);
  o->src_rec = P.src_rec.data();
  o->nedges = static_cast<int64_t>(P.succ.size());
  o->succ = P.succ.data();
  o->succ_rec = P.succ_rec.data();
  o->indeg = P.indeg.data();
  o->nroots = static_cast<int64_t>(P.roots.size());
  o->roots = P.roots.data();
  o->max_target_len = P.stats.max_target_len;
  o->max_flag_rows = P.stats.max_flag_rows;
  o->nhelpers = P.stats.helpers;
  o->nslots = static_cast<int64_t>(P.slot_rec.size() / 4);
  o->slot_rec = P.slot_rec.data();
  o->nupdates = static_cast<int64_t>(P.upd.size() / 2);
  o->upd = P.upd.data();
  return TCG_OK;
}

tcg_status tcg_plan_part_problem(tcg_plan* plan, int32_t nparts, const int32_t* part_of_row, int32_t part,
                                 tcg_problem* o, int64_t* remote_operands) {
  if (!plan || !o || !part_of_row) return TCG_INVALID;
  try {
    tcb::flow_plan_schedule(plan->flow);  // a part is a slice of the global schedule
    std::vector<std::int32_t> own(part_of_row, part_of_row + plan->flow.n);
    plan->parts[part] = tcb::build_flow_part(plan->flow, own, nparts, part);
    plan->part_owner = std::move(own);
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
  const tcb::FlowPart& F = plan->parts[part];
  *o = tcg_problem{};
  const tcb::FlowPlan& P = plan->flow;
  // only the value-flow tables describe a part: no task executor
  o->n = P.n;
  o->nnz = P.nnz;
  o->col_idx = P.cols.data();
  o->values = P.values.data();
  o->ntasks = P.stats.tasks[0] + P.stats.tasks[1] + P.stats.tasks[2] + P.stats.tasks[3];
  o->nflow = F.rows;
  o->flow_rec = F.rec.data();
  o->flow_item = F.unit.data();
  o->flow_devprog = 1;
  o->u_row_ptr = P.row_ptr.data();
  o->flow_part = part;
  o->part_of_row = plan->part_owner.data();
  if (remote_operands) *remote_operands = F.remote_sources;
  return TCG_OK;
}

tcg_status tcg_plan_get_stats(const tcg_plan* plan, tcg_plan_stats* o) {
  if (!plan || !o) return TCG_INVALID;
  *o = tcg_plan_stats{};
  const tcb::FlowPlanStats& f = plan->flow.stats;
  for (int k = 0; k < 4; ++k) o->tasks[k] = f.tasks[k];
  o->nblocks_rows = f.nblock_rows;
  o->nblocks = f.nblocks;
  o->block_build_seconds = f.block_build_seconds;
  o->plan_seconds = f.plan_seconds;
  o->flow_rows = f.units;
  o->flow_depth = f.depth;
  o->host_threads = f.threads;
  o->full_plan = plan->full ? 1 : 0;
  if (!plan->full) return TCG_OK;
  // the task-DAG statistics exist once the full plan does
  const tcb::PlanStats& s = plan->full->stats;
  o->edges = s.edges;
  o->items = s.items;
  o->sources = s.sources;
  o->pairs = s.pairs;
  o->empty_tasks = s.empty_tasks;
  o->max_target_len = s.max_target_len;
  o->max_flag_rows = s.max_flag_rows;
  o->dag_depth = s.dag_depth;
  o->max_width = s.max_width;
  o->helpers = s.helpers;
  o->updates = s.updates;
  o->full_plan_seconds = s.plan_seconds + s.block_build_seconds;
  return TCG_OK;
}

tcg_status tcg_plan_dag(const tcg_plan* plan, int64_t* nnodes, const int32_t** kind,
                        const int32_t** block_row, const int32_t** block_col, int64_t* nedges,
                        const int32_t** edge_from, const int32_t** edge_to) {
  if (!plan) return TCG_INVALID;
  try {
    const tcb::Plan& P = full_plan(plan);
    if (nnodes) *nnodes = static_cast<int64_t>(P.node_kind.size());
    if (kind) *kind = P.node_kind.data();
    if (block_row) *block_row = P.node_i.data();
    if (block_col) *block_col = P.node_j.data();
    if (nedges) *nedges = static_cast<int64_t>(P.edge_from.size());
    if (edge_from) *edge_from = P.edge_from.data();
    if (edge_to) *edge_to = P.edge_to.data();
    return TCG_OK;
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
}

tcg_status tcg_plan_blocks(const tcg_plan* plan, int32_t* m, const int64_t** brow_ptr,
                           int64_t* nblocks, const int32_t** bcol_idx) {
  if (!plan) return TCG_INVALID;
  try {
    const tcb::BlockLayout& B = full_plan(plan).blocks;
    if (m) *m = B.m;
    if (brow_ptr) *brow_ptr = B.brow_ptr.data();
    if (nblocks) *nblocks = B.nblocks();
    if (bcol_idx) *bcol_idx = B.bcol_idx.data();
    return TCG_OK;
  } catch (const std::exception& e) {
    g_plan_error = e.what();
    return TCG_INVALID;
  }
}

// -------------------------------------------------------------- device ----

tcg_status tcg_create(int device, tcg_ctx** out) {
  if (!out) return TCG_INVALID;
  *out = nullptr;
  auto c = std::make_unique<tcg_ctx>();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev2);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev3, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&c->host_ctrl), sizeof(tcbdev::Ctrl));
  if (e != cudaSuccess) {
    g_plan_error = std::string("tcg_create: ") + cudaGetErrorString(e);
    tcg_destroy(c.release());
    return TCG_CUDA;
  }
  *out = c.release();
  return TCG_OK;
}

void tcg_destroy(tcg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);  // before any block goes back to the cache
  if (c->d2h_stream) cudaStreamSynchronize(c->d2h_stream);
  if (c->h2d_stream) cudaStreamSynchronize(c->h2d_stream);
  dev_free(c->batch_arena);
  dev_free(c->prog_arena);
  if (c->a_stage) cudaFree(c->a_stage);
  if (c->drain_done) cudaFree(c->drain_done);
  if (c->chunk_units) cudaFree(c->chunk_units);
  if (c->chunk_flag) cudaFreeHost(c->chunk_flag);
  if (c->peers) cudaFree(c->peers);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  dev_free(c->arena);
  if (c->host_ctrl) cudaFreeHost(c->host_ctrl);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev2) cudaEventDestroy(c->ev2);
  if (c->ev3) cudaEventDestroy(c->ev3);
  for (cudaEvent_t e : c->chunk_ev) cudaEventDestroy(e);
  if (c->host_ctrls) cudaFreeHost(c->host_ctrls);
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* tcg_last_error(const tcg_ctx* c) {
  if (!c) return g_plan_error.c_str();
  return c->err.c_str();
}

tcg_status tcg_set_options(tcg_ctx* c, const tcg_options* opt) {
  if (!c || !opt) return TCG_INVALID;
  const int t = opt->threads_per_cta;
  if (t != 0 && t != 128 && t != 256 && t != 512 && t != 384 && t != 768) {
    c->err = "threads_per_cta must be 128, 256 or 512 (or 384, 768 in mode 5)";
    return TCG_INVALID;
  }
  c->opt = *opt;
  return TCG_OK;
}

}  // extern "C"

// The value-flow update programs built on the device (flow_program.cu): U's
// transposed index by a radix sort, a count pass, a scan, the (m, o) pairs'
// own allocation, a fill pass. Scratch: one temporary allocation for the
// index, the counts and the 32-bit offsets in the working values, the 64-bit
// scan in the input snapshot (both rewritten before any factorization).
static tcg_status build_programs(tcg_ctx* c, const tcg_problem* p) {
  const std::int64_t n = p->n, nnz = p->nnz, ns = nnz - n;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* tmp = nullptr;
  size_t scan_bytes = 0, sort_bytes = 0;
  TCG_CUDA_TRY(c, tcbdev::flow_program_scan(nullptr, nullptr, nullptr, nnz, nullptr, nullptr, &scan_bytes,
                                            c->sm_count, c->stream));
  TCG_CUDA_TRY(c, tcbdev::flow_transpose(static_cast<int>(n), static_cast<int>(nnz), nullptr, nullptr, nullptr,
                                         nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &sort_bytes,
                                         c->sm_count, c->stream));
  // the schedule on the device when the plan has none (tcg_plan_build's default)
  const bool dev_sched = !p->flow_rec;
  const std::int64_t U = dev_sched ? p->nflow : 0;
  size_t sched_bytes = 0;
  tcbdev::SchedParams S{};
  S.nunits = static_cast<int>(U);
  if (dev_sched)
    TCG_CUDA_TRY(c, tcbdev::flow_schedule(S, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                          &sched_bytes, c->sm_count, c->stream));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + std::max<size_t>(bytes, 1), 256);
    return at;
  };
  const size_t o_rp = take(sizeof(int) * (n + 1)), o_cp = take(sizeof(int) * (n + 1));
  const size_t o_key = take(sizeof(int) * nnz), o_pos = take(sizeof(int) * nnz), o_rid = take(sizeof(int) * nnz);
  const size_t o_keys = take(sizeof(int) * nnz), o_poss = take(sizeof(int) * nnz), o_cs = take(sizeof(int) * ns);
  const size_t o_ctr = take(sizeof(int) * 2), o_tot = take(sizeof(long long));
  const size_t o_own = take(p->flow_part >= 0 ? sizeof(int) * n : 0);
  const size_t o_tmp = take(std::max({scan_bytes, sort_bytes, sched_bytes}));
  const size_t o_uf = take(dev_sched ? sizeof(int) * (n + 1) : 0), o_utb = take(sizeof(int) * U),
               o_ulen = take(sizeof(int) * U), o_urow = take(sizeof(int) * U), o_lvl = take(sizeof(int) * U),
               o_hgt = take(sizeof(int) * U), o_acc = take(sizeof(int) * U), o_ids = take(sizeof(int) * (U + 1)),
               o_ord = take(sizeof(int) * (U + 1)), o_skey = take(sizeof(long long) * U), o_skey2 = take(sizeof(long long) * U),
               o_words = take(sizeof(int) * 2), o_uc0 = take(sizeof(int) * U), o_uc1 = take(sizeof(int) * U),
               o_acc2 = take(sizeof(int) * U);
  TCG_CUDA_TRY(c, dev_alloc(c->device, &tmp, off));
  struct Free {
    void* p;
    cudaStream_t st;
    ~Free() {
      cudaStreamSynchronize(st);  // (an early return may leave work on the stream)
      dev_free(p);
    }
  } free_tmp{tmp, c->stream};
  char* b = static_cast<char*>(tmp);
  int* row_ptr = reinterpret_cast<int*>(b + o_rp);
  int* col_ptr = reinterpret_cast<int*>(b + o_cp);
  int* col_pos = reinterpret_cast<int*>(b + o_poss);
  int* col_src = reinterpret_cast<int*>(b + o_cs);
  tcbdev::ProgParams q{};
  q.n = static_cast<int>(n);
  q.row_ptr = row_ptr;
  q.cols = c->cols;
  q.col_ptr = col_ptr;
  q.col_src = col_src;
  q.col_pos = col_pos;
  q.next_row = reinterpret_cast<int*>(b + o_ctr);
  int* count = reinterpret_cast<int*>(c->vals);   // nnz ints (of 2 nnz)
  int* ub32 = count + nnz;                         // nnz ints
  long long* ub64 = reinterpret_cast<long long*>(c->flow_a);
  long long* total_d = reinterpret_cast<long long*>(b + o_tot);
  q.count = count;
  q.ub = ub32;
  q.slot = c->flow_slot;
  TCG_CUDA_TRY(c, cudaMemcpyAsync(row_ptr, p->u_row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaMemsetAsync(q.next_row, 0, sizeof(int) * 2, c->stream));
  TCG_CUDA_TRY(c, cudaEventCreate(&e0));
  TCG_CUDA_TRY(c, cudaEventCreate(&e1));
  struct Ev {
    cudaEvent_t a, b;
    ~Ev() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } evs{e0, e1};
  TCG_CUDA_TRY(c, cudaEventRecord(e0, c->stream));
  TCG_CUDA_TRY(c, tcbdev::flow_transpose(static_cast<int>(n), static_cast<int>(nnz), row_ptr, c->cols,
                                         reinterpret_cast<int*>(b + o_key), reinterpret_cast<int*>(b + o_pos),
                                         reinterpret_cast<int*>(b + o_rid), reinterpret_cast<int*>(b + o_keys),
                                         col_pos, col_ptr, col_src, b + o_tmp, &sort_bytes, c->sm_count, c->stream));
  const bool say = std::getenv("TCG_PLAN_TIMES") != nullptr;
  auto wall = [&](const char* what) {  // host wall time of the stream's work so far (TCG_PLAN_TIMES)
    static thread_local std::chrono::steady_clock::time_point last;
    if (!say) return;
    cudaStreamSynchronize(c->stream);
    const auto now = std::chrono::steady_clock::now();
    if (what) std::fprintf(stderr, "upload %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  };
  wall(nullptr);
  if (dev_sched && U > 0) {
    auto ip = [&](size_t o) { return reinterpret_cast<int*>(b + o); };
    TCG_CUDA_TRY(c, cudaMemcpyAsync(ip(o_uf), p->u_first, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(ip(o_utb), p->u_tb, sizeof(int) * U, cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(ip(o_ulen), p->u_len, sizeof(int) * U, cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(ip(o_urow), p->u_row, sizeof(int) * U, cudaMemcpyHostToDevice, c->stream));
    wall("units H2D");
    S.n = static_cast<int>(n);
    S.nnz = nnz;
    S.slack_pct = tcb::flow_slack_pct(n, nnz, U);
    S.row_ptr = row_ptr;
    S.cols = c->cols;
    S.col_ptr = col_ptr;
    S.col_src = col_src;
    S.col_pos = col_pos;
    S.ufirst = ip(o_uf);
    S.u_tb = ip(o_utb);
    S.u_len = ip(o_ulen);
    S.uc0 = ip(o_uc0);
    S.uc1 = ip(o_uc1);
    S.level = ip(o_lvl);
    S.height = ip(o_hgt);
    S.acc = ip(o_acc);
    S.acc2 = ip(o_acc2);
    S.depth = ip(o_words);
    S.error = ip(o_words) + 1;
    S.timeout_ns = static_cast<unsigned long long>((c->opt.timeout_s > 0 ? c->opt.timeout_s : 30.0) * 1e9);
    TCG_CUDA_TRY(c, tcbdev::flow_schedule(S, ip(o_urow), c->flow_rec, c->flow_item,
                                          reinterpret_cast<unsigned long long*>(b + o_skey),
                                          reinterpret_cast<unsigned long long*>(b + o_skey2), ip(o_ids), ip(o_ord),
                                          b + o_tmp, &sched_bytes, c->sm_count, c->stream));
    wall("schedule");
    int words[2] = {0, 0};
    TCG_CUDA_TRY(c, cudaMemcpyAsync(words, ip(o_words), sizeof(words), cudaMemcpyDeviceToHost, c->stream));
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (words[1]) {
      c->err = "tcg_upload: device watchdog expired while building the schedule";
      return TCG_TIMEOUT;
    }
    c->flow_depth = words[0];
  }
  TCG_CUDA_TRY(c, tcbdev::flow_program_count(q, c->sm_count, c->stream));
  TCG_CUDA_TRY(c, tcbdev::flow_program_scan(count, ub64, ub32, nnz, total_d, b + o_tmp, &scan_bytes,
                                            c->sm_count, c->stream));
  long long total = 0;
  TCG_CUDA_TRY(c, cudaMemcpyAsync(&total, total_d, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (total > 0x7fffffffLL) {
    c->err = "tcg_upload: more than 2^31 products in the update programs";
    return TCG_INVALID;
  }
  // [(m, o) pairs][per-coordinate offsets, nnz + 1] (the offsets for the product-parallel rows)
  const size_t upd_bytes = align_up(sizeof(int2) * std::max<long long>(total, 1), 256);
  TCG_CUDA_TRY(c, dev_alloc(c->device, &c->prog_arena, upd_bytes + sizeof(int) * (nnz + 1)));
  c->flow_upd = static_cast<int2*>(c->prog_arena);
  c->flow_ub = reinterpret_cast<int*>(static_cast<char*>(c->prog_arena) + upd_bytes);
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->flow_ub, ub32, sizeof(int) * nnz, cudaMemcpyDeviceToDevice, c->stream));
  c->ub_total = static_cast<int>(total);
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->flow_ub + nnz, &c->ub_total, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  q.upd = c->flow_upd;
  TCG_CUDA_TRY(c, tcbdev::flow_program_fill(q, c->sm_count, c->stream));
  if (p->flow_part >= 0) {  // a part: operands of other parts' rows through the peer table
    int* owner = reinterpret_cast<int*>(b + o_own);
    TCG_CUDA_TRY(c, cudaMemcpyAsync(owner, p->part_of_row, sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, tcbdev::flow_program_remote_rewrite(nnz, reinterpret_cast<int*>(b + o_rid), owner, p->flow_part,
                                                        c->flow_slot, c->flow_upd, c->sm_count, c->stream));
  }
  TCG_CUDA_TRY(c, cudaEventRecord(e1, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  TCG_CUDA_TRY(c, cudaEventElapsedTime(&ms, e0, e1));
  c->prog_build_ms = ms;
  c->nflow_upd = total;
  return TCG_OK;
}

extern "C" {

tcg_status tcg_upload(tcg_ctx* c, const tcg_problem* p) {
  if (!c || !p) return TCG_INVALID;
  if (p->n < 0 || p->nnz < 0 || p->ntasks < 0 || p->nitems < 0 || p->nsources < 0 ||
      p->nedges < 0 || p->nroots < 0 || p->nhelpers < 0 || p->nnz > 0x7fffffffLL ||
      p->ntasks + p->nhelpers >= 0x40000000LL || p->nflow < 0 || p->nflow > 0x7fffffffLL ||
      (p->flow_devprog && p->nnz < p->n)) {
    c->err = "tcg_upload: invalid problem sizes";
    return TCG_INVALID;
  }
  // the task tables exist only with the task-DAG plan (tcg_plan_expand); the count stays
  // for the statistics either way
  const std::int64_t ntab = p->task_rec ? p->ntasks : 0;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->arena) {
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    dev_free(c->arena);
    c->arena = nullptr;
    c->uploaded = false;
  }
  if (c->batch_arena) {
    dev_free(c->batch_arena);
    c->batch_arena = nullptr;
  }
  if (c->prog_arena) {
    dev_free(c->prog_arena);
    c->prog_arena = nullptr;
  }
  c->flow_ub = nullptr;  // lives in prog_arena (device-built programs only)
  c->nbatch = 1;
  // one arena: [cols][vals][vals0][tasks][items][srcs][succ][indeg][indeg0][queue][roots]
  //            [claim][fin][iflag][ctrl][trace]
  const std::int64_t qcap = ntab + (ntab ? p->nhelpers : 0);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + std::max<size_t>(bytes, 1), 256);
    return at;
  };
  const size_t o_cols = take(sizeof(int) * p->nnz);
  const size_t o_vals = take(sizeof(double) * p->nnz);
  const size_t o_vals0 = take(sizeof(double) * p->nnz);
  const size_t o_tasks = take(sizeof(int) * 12 * ntab);
  const size_t o_items = take(sizeof(int) * 8 * p->nitems);
  const size_t o_srcs = take(sizeof(int) * 4 * p->nsources);
  const size_t o_succ = take(sizeof(int4) * 4 * p->nedges);
  const size_t o_indeg = take(sizeof(int) * ntab);
  const size_t o_indeg0 = take(sizeof(int) * ntab);
  const size_t o_queue = take(sizeof(int) * qcap);
  const size_t o_roots = take(sizeof(int) * p->nroots);
  const size_t o_claim = take(sizeof(int) * ntab);
  const size_t o_fin = take(sizeof(int) * ntab);
  const size_t o_iflag = take(sizeof(int) * p->nitems);
  const bool programs = p->nslots > 0 && p->slot_rec && (p->nupdates == 0 || p->upd);
  const size_t o_slot = take(programs ? sizeof(int4) * p->nslots : 0);
  const size_t o_upd = take(programs ? sizeof(int) * 2 * p->nupdates : 0);
  const bool devprog = p->flow_devprog && p->u_row_ptr;
  const bool dev_sched = devprog && !p->flow_rec && p->u_first && p->u_tb && p->u_len && p->u_row &&
                         p->flow_part < 0;
  const bool flow = p->nflow > 0 && ((p->flow_rec && p->flow_item) || dev_sched) &&
                    (devprog || (p->flow_slot && (p->nflow_upd == 0 || p->flow_upd)));
  if (p->flow_part >= 0 && (!devprog || !p->part_of_row || p->nnz >= (1LL << tcb::kRemoteShift))) {
    c->err = "tcg_upload: a part needs device-built programs, its owner table and U below 2^25 entries";
    return TCG_INVALID;
  }
  const size_t o_frec = take(flow ? sizeof(int4) * p->nflow : 0);
  const size_t o_fitem = take(flow ? sizeof(int) * p->nflow : 0);
  const size_t o_fslot = take(flow ? sizeof(int4) * p->nnz : 0);
  const size_t o_fupd = take(flow && !devprog ? sizeof(int2) * p->nflow_upd : 0);
  const size_t o_fa = take(flow ? sizeof(double) * p->nnz : 0);
  const bool amap = p->nnz_a > 0 && p->a_map;
  const size_t o_amap = take(amap ? sizeof(int) * p->nnz : 0);
  const size_t o_mflags = take(sizeof(int) * 2);
  const size_t o_mpivot = take(sizeof(double));
  const size_t o_ctrl = take(sizeof(tcbdev::Ctrl));
  const size_t o_trace = take(sizeof(unsigned long long) * (2 * ntab + 4 * std::max(p->nitems, p->nflow)));
  TCG_CUDA_TRY(c, dev_alloc(c->device, &c->arena, off));
  c->arena_bytes = off;
  char* base = static_cast<char*>(c->arena);
  c->cols = reinterpret_cast<int*>(base + o_cols);
  c->vals = reinterpret_cast<double*>(base + o_vals);
  c->vals0 = reinterpret_cast<double*>(base + o_vals0);
  c->tasks = reinterpret_cast<int4*>(base + o_tasks);
  c->items = reinterpret_cast<int4*>(base + o_items);
  c->srcs = reinterpret_cast<int4*>(base + o_srcs);
  c->succ = reinterpret_cast<int4*>(base + o_succ);
  c->indeg = reinterpret_cast<int*>(base + o_indeg);
  c->indeg0 = reinterpret_cast<int*>(base + o_indeg0);
  c->queue = reinterpret_cast<int*>(base + o_queue);
  c->roots = reinterpret_cast<int*>(base + o_roots);
  c->claim = reinterpret_cast<int*>(base + o_claim);
  c->fin = reinterpret_cast<int*>(base + o_fin);
  c->iflag = reinterpret_cast<int*>(base + o_iflag);
  c->slot_rec = reinterpret_cast<int4*>(base + o_slot);
  c->upd = reinterpret_cast<int2*>(base + o_upd);
  c->has_programs = programs;
  c->flow_rec = reinterpret_cast<int4*>(base + o_frec);
  c->flow_item = reinterpret_cast<int*>(base + o_fitem);
  c->a_map = amap ? reinterpret_cast<int*>(base + o_amap) : nullptr;
  c->nnz_a = amap ? p->nnz_a : 0;
  c->m_flags = reinterpret_cast<int*>(base + o_mflags);
  c->m_pivot = reinterpret_cast<double*>(base + o_mpivot);
  c->flow_slot = reinterpret_cast<int4*>(base + o_fslot);
  c->flow_upd = reinterpret_cast<int2*>(base + o_fupd);
  c->flow_a = reinterpret_cast<double*>(base + o_fa);
  c->nflow = flow ? p->nflow : 0;
  c->nflow_upd = flow && !devprog ? p->nflow_upd : 0;
  c->has_flow = flow;

  c->nslots = programs ? p->nslots : 0;
  c->nupdates = programs ? p->nupdates : 0;
  c->ctrl = reinterpret_cast<tcbdev::Ctrl*>(base + o_ctrl);
  c->trace = reinterpret_cast<unsigned long long*>(base + o_trace);
  auto put = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
  };
  TCG_CUDA_TRY(c, put(c->cols, p->col_idx, sizeof(int) * p->nnz));
  TCG_CUDA_TRY(c, put(c->vals0, p->values, sizeof(double) * p->nnz));
  TCG_CUDA_TRY(c, put(c->tasks, p->task_rec, sizeof(int) * 12 * ntab));
  TCG_CUDA_TRY(c, put(c->items, p->item_rec, sizeof(int) * 8 * p->nitems));
  TCG_CUDA_TRY(c, put(c->srcs, p->src_rec, sizeof(int) * 4 * p->nsources));
  if (p->nedges > 0 && !p->succ_rec) {
    c->err = "tcg_upload: succ_rec is required";
    return TCG_INVALID;
  }
  TCG_CUDA_TRY(c, put(c->succ, p->succ_rec, sizeof(int4) * 4 * p->nedges));
  TCG_CUDA_TRY(c, put(c->indeg0, p->indeg, sizeof(int) * ntab));
  TCG_CUDA_TRY(c, put(c->roots, p->roots, sizeof(int) * p->nroots));
  if (programs) {
    TCG_CUDA_TRY(c, put(c->slot_rec, p->slot_rec, sizeof(int4) * p->nslots));
    TCG_CUDA_TRY(c, put(c->upd, p->upd, sizeof(int) * 2 * p->nupdates));
  }
  c->flow_depth = 0;
  if (flow) {
    if (!dev_sched) {
      TCG_CUDA_TRY(c, put(c->flow_rec, p->flow_rec, sizeof(int4) * p->nflow));
      TCG_CUDA_TRY(c, put(c->flow_item, p->flow_item, sizeof(int) * p->nflow));
    }
    if (!devprog) {
      TCG_CUDA_TRY(c, put(c->flow_slot, p->flow_slot, sizeof(int4) * p->nnz));
      TCG_CUDA_TRY(c, put(c->flow_upd, p->flow_upd, sizeof(int2) * p->nflow_upd));
    }
  }
  if (amap) TCG_CUDA_TRY(c, put(c->a_map, p->a_map, sizeof(int) * p->nnz));
  if (p->nitems > 0)
    TCG_CUDA_TRY(c, cudaMemsetAsync(c->iflag, 0, sizeof(int) * p->nitems, c->stream));
  if (flow && devprog) {
    const tcg_status st = build_programs(c, p);
    if (st != TCG_OK) return st;
  }
  if (p->nnz > 0)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->vals, c->vals0, sizeof(double) * p->nnz,
                                    cudaMemcpyDeviceToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->n = p->n;
  c->nnz = p->nnz;
  c->ntasks = p->ntasks;
  c->ntab = ntab;
  c->nitems = p->nitems;
  c->nsrc = p->nsources;
  c->nedges = p->nedges;
  c->nroots = p->nroots;
  c->qcap = qcap;
  c->epoch = 0;
  c->max_target_len = p->max_target_len;
  c->max_flag_rows = p->max_flag_rows;
  c->uploaded = true;
  c->chunks_ready = false;
  c->drain_ms[0] = c->drain_ms[1] = c->drain_ms[2] = -1.f;
  c->drain_calls = 0;
  c->pristine = true;
  return TCG_OK;
}

tcg_status tcg_set_values(tcg_ctx* c, const double* values) {
  if (!c || !c->uploaded || (!values && c->nnz > 0)) return TCG_INVALID;
  if (c->nnz == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->vals0, values, sizeof(double) * c->nnz,
                                  cudaMemcpyHostToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->vals, c->vals0, sizeof(double) * c->nnz,
                                  cudaMemcpyDeviceToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->pristine = true;
  return TCG_OK;
}

tcg_status tcg_restore(tcg_ctx* c) {
  if (!c || !c->uploaded) return TCG_INVALID;
  if (c->nnz == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->nbatch > 1)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->bvals, c->bvals0, sizeof(double) * c->nnz * c->nbatch,
                                    cudaMemcpyDeviceToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->vals, c->vals0, sizeof(double) * c->nnz,
                                  cudaMemcpyDeviceToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->pristine = true;
  return TCG_OK;
}

// The chunks of the chunked download (run_flow, mode 2): up to 64 ranges of U
// of at least 512 KB, cut at unit starts; a unit at tb lies in chunk
// tb * nchunks / nnz. Built once per upload from the schedule's records.
static tcg_status prepare_chunks(tcg_ctx* c) {
  if (c->chunks_ready) return TCG_OK;
  constexpr int kMaxChunks = 64;
  std::int64_t least = 512 << 10;  // bytes per chunk at least (TCG_D2H_CHUNK_KB)
  if (const char* e = std::getenv("TCG_D2H_CHUNK_KB")) least = std::max<std::int64_t>(1, std::atoll(e)) << 10;
  const int n = static_cast<int>(std::min<std::int64_t>(kMaxChunks, c->nnz * 8 / least));
  c->nchunks = n >= 4 ? n : 0;
  c->chunks_ready = true;
  if (!c->nchunks) return TCG_OK;
  if (!c->chunk_units) {
    TCG_CUDA_TRY(c, cudaMalloc(&c->chunk_units, sizeof(int) * 3 * kMaxChunks));
    c->chunk_left = c->chunk_units + kMaxChunks;
    TCG_CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->chunk_flag), sizeof(int) * kMaxChunks, cudaHostAllocMapped));
    std::memset(c->chunk_flag, 0, sizeof(int) * kMaxChunks);
    TCG_CUDA_TRY(c, cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->chunk_flag_d), c->chunk_flag, 0));
  }
  int* start_d = c->chunk_units + 2 * kMaxChunks;
  TCG_CUDA_TRY(c, tcbdev::launch_chunk_setup(c->flow_rec, static_cast<int>(c->nflow), c->nnz, c->nchunks, start_d,
                                             c->chunk_units, c->sm_count, c->stream));
  int start[kMaxChunks];
  TCG_CUDA_TRY(c, cudaMemcpyAsync(start, start_d, sizeof(int) * c->nchunks, cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->chunk_start.assign(static_cast<size_t>(c->nchunks) + 1, c->nnz);
  for (int k = 0; k < c->nchunks; ++k) {
    if (start[k] == 0x7f7f7f7f || (k == 0 && start[k] != 0)) {  // a range without a unit start: no chunks
      c->nchunks = 0;
      return TCG_OK;
    }
    c->chunk_start[static_cast<size_t>(k)] = start[k];
  }
  return TCG_OK;
}

// Product-parallel rows (flow_pp_kernel.cu) where programs are short (mean
// products per coordinate <= 4: C1, C2, C5, C6): a row's products spread over
// a group of wpr warps, nb batches of kp per thread and chunk. One warp per
// row for large schedules, two for small ones (B200: C1 0.044 -> 0.040, C2
// 0.395 -> 0.364, C5 0.168 -> 0.134, C6 1.725 -> 1.424, the C5 batch 1.816 ->
// 1.412 ms). Long programs (C3, C4) stay on the per-lane kernel.
// TCG_FLOW_PP=0 turns it off; TCG_FLOW_PP=wpr,kp,nb,minb,d[,backoff] picks a variant.
static bool pick_pp(const tcg_ctx* c, double mean, int* w, int* k, int* n, int* m, int* d, int* b) {
  if (!c->flow_ub) return false;
  if (c->opt.threads_per_cta != 0 && c->opt.threads_per_cta != 256) return false;  // 256-thread CTAs only
  if (const char* e = std::getenv("TCG_FLOW_PP")) {
    *b = -1;
    const int got = std::sscanf(e, "%d,%d,%d,%d,%d,%d", w, k, n, m, d, b);
    return got >= 5 && *w > 0;
  }
  if (mean > 4.0) return false;
  const long long positions = c->nflow * c->nbatch;
  // Between the small matrices (a few units per warp: the group's parallel products win) and the
  // large ones (hundreds of units per warp: throughput) the chain binds, and the per-lane kernel
  // with its warp-wide settle of the last batch is the faster one. B200, 7-point Laplacians IC(1),
  // per-lane / product-parallel ms: 40^3 (64 K units) 0.173 / 0.187, 56^3 (176 K) 0.270 / 0.311,
  // 64^3 (C2, 262 K) 0.343 / 0.361, 80^3 (512 K) 0.539 / 0.529, 96^3 (885 K) 0.813 / 0.751,
  // 128^3 (C6) 1.67 / 1.43; C5 (33 K) 0.146 / 0.136, C1 (13 K) 0.052 / 0.043.
  if (c->nbatch == 1 && positions > 48000 && positions <= 400000) return false;
  if (positions <= 200000) {
    *w = 2, *k = 2, *n = 2, *m = 3, *d = 1;
  } else {
    *w = 1, *k = 2, *n = 1, *m = 4, *d = 2;
  }
  *b = 0;
  return true;
}

// Value-flow execution (mode 5, flow_kernel.cu): prelude (snapshot the
// input, mark the output unwritten, reset the status words) + one persistent
// launch; both inside the timed region.
// host_in/host_out (tcg_factor_host): upload, factor and download on the
// launch stream.
static tcg_status run_flow(tcg_ctx* c, tcg_stats& S, int threads, const double* host_in = nullptr,
                           double* host_out = nullptr, int phase = 0, const double* host_a = nullptr) {
  // the value-flow kernels run 256-thread CTAs of whole warps (tcg_options.threads_per_cta
  // applies to the task executors, lanes_per_row is kept for the ABI and ignored)
  threads = 256;
  // gather batch from the mean products per coordinate (flow_kernel.cu variants)
  const double mean = c->nnz > 0 ? static_cast<double>(c->nflow_upd) / static_cast<double>(c->nnz) : 0.0;
  // short programs: one product in flight per lane where the chain binds (B200, KB 1 vs 2: C2
  // 0.402 -> 0.390, C5 0.183 -> 0.168 ms), two where each warp runs hundreds of rows back to
  // back and the per-row gather sets the pace (C6, 2.1 M rows: 1.711 vs 1.734 ms)
  const bool one_local = c->nbatch == 1 && !c->opt.trace && c->npeers <= 1;  // the single-matrix kernels
  int kb = mean <= 4.0 ? (one_local && c->nflow <= 1000000 ? 1 : 2) : 3;
  int minb = threads == 128 ? 6 : threads == 384 ? 2 : threads == 256 ? 3 : 1;
  if (const char* e = std::getenv("TCG_FLOW_KB")) kb = std::atoi(e);
  // short programs: 5 CTAs per SM of the single-matrix kernel (48 registers, no spills;
  // B200: C1 0.049 -> 0.043, C2 0.415 -> 0.402, C5 0.188 -> 0.181, C6 1.79 -> 1.71 ms);
  // with KB = 3 the fifth CTA costs more than it hides (C3 4.03 -> 4.15, C4 1.47 -> 1.60)
  if (threads == 256 && kb <= 2 && one_local) minb = 5;
  if (const char* e = std::getenv("TCG_FLOW_MINB")) minb = std::atoi(e);
  int remote = c->npeers > 1 ? 1 : 0;  // sharded: operands of other parts via peers
  if (const char* e = std::getenv("TCG_FLOW_REMOTE")) remote = std::atoi(e) ? 1 : remote;
  bool pipe = true;  // the per-lane kernel (factor_flow_pipe), unless the product-parallel one runs
  // the member / trace arithmetic; sharded runs use those variants too (their remote reads exist there)
  int extras = (c->nbatch > 1 || c->opt.trace || remote) ? 1 : 0;
  if (const char* e = std::getenv("TCG_FLOW_EXTRAS")) extras = std::atoi(e) ? 1 : extras;
  // end to end: CTAs of the launch copy the factor to the host as it becomes
  // final (the D2H overlaps the factorization); needs a pinned, mapped buffer
  double* drain_out = nullptr;
  // drain CTAs: 8, or 4 where long programs keep L2 busy (B200, end to end: C2 0.82 ms at 4-8,
  // C4 4.09 at 8 / 4.47 at 4, C6 5.45 at 8 / 6.02 at 4, C3 (24.8 products per coordinate)
  // 4.57 at 4 / 4.93 at 8; 16-32 no better anywhere)
  int drain_ctas = mean > 16.0 ? 4 : 8;
  if (const char* e = std::getenv("TCG_DRAIN_CTAS")) drain_ctas = std::max(1, std::atoi(e));
  bool drain = host_out && pipe && !remote && !c->opt.trace && c->nflow > 0 && phase == 0;
  bool chunks = drain && c->nbatch == 1;
  bool out_pinned = false;
  if (drain) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, host_out) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
        attr.devicePointer) {
      drain_out = static_cast<double*>(attr.devicePointer);
      out_pinned = true;
    } else {
      cudaGetLastError();
    }
    // 16-byte accesses on both sides (flow_kernel.cu drain_values)
    drain = drain_out != nullptr && reinterpret_cast<std::uintptr_t>(drain_out) % 16 == 0 &&
            reinterpret_cast<std::uintptr_t>(c->nbatch > 1 ? c->bvals : c->vals) % 16 == 0;
  }
  // chunked copies: the copy engine takes each chunk of U to the (pinned) host
  // buffer as soon as its last unit has run, beside the rest of the launch
  if (chunks && out_pinned) {
    const tcg_status cs = prepare_chunks(c);
    if (cs != TCG_OK) return cs;
    chunks = c->nchunks > 0;
    if (chunks && !c->d2h_stream) TCG_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
  } else {
    chunks = false;
  }
  // How the factor should leave depends on the host: zero-copy writes from
  // the SMs (the drain CTAs) ran at ~40 GB/s on some B200 boxes (C2 end to end
  // 1.02 -> 0.82 ms) and far slower on others (1.03 -> 1.44 ms); the copy
  // engine runs at PCIe speed everywhere, after the launch (mode 0) or chunk
  // by chunk beside it (mode 2). Unless TCG_DRAIN decides (0 / 1 / 2), the
  // first calls of a problem take turns (the very first call of a buffer pays
  // one-time costs, so each mode keeps its best of 3), later calls take the fastest.
  int dmode = 0;
  bool calibrating = false;
  if (const char* e = std::getenv("TCG_DRAIN")) {
    const int v = std::atoi(e);
    dmode = (v == 1 && drain) ? 1 : (v == 2 && chunks) ? 2 : 0;
  } else if (drain || chunks) {
    int cand[3], nc = 0;
    cand[nc++] = 0;
    if (drain) cand[nc++] = 1;
    if (chunks) cand[nc++] = 2;
    if (c->drain_calls < 3 * nc) {
      dmode = cand[c->drain_calls % nc];
      calibrating = true;
    } else {
      for (int i = 1; i < nc; ++i)
        if (c->drain_ms[cand[i]] >= 0.f && c->drain_ms[cand[i]] < c->drain_ms[dmode]) dmode = cand[i];
    }
  }
  drain = dmode == 1;
  chunks = dmode == 2;
  // the 5-CTA kernel exists for one local matrix (with or without the drain)
  if (minb == 5 && (remote || extras || !pipe || kb > 2)) minb = 3;
  int occ = 0;
  // poll back-off for long programs (flow_kernel.cu Ctx): thousands of lanes
  // poll the lines the critical rows write; sleeping between polls frees them
  // (the sleep only follows a poll that still saw kUnset). B200, fixed
  // back-off sweep with a compiled variant for every value -- __nanosleep
  // rounds its argument into coarse steps, so 300-500 ns and 520-1600 ns each
  // measure as one value: C3 (24.8 products per coordinate) 4.01 / 2.91 / 2.76
  // / 2.66 / 2.60 / 3.23 ms at 0 / 100 / 200 / 300-500 / 520-1600 / 2400; C4
  // (12.4) 1.49 / 1.31 / 1.30 / 1.31 / 1.32 / 1.45 at 0 / 100 / 150-250 / 400 /
  // 600-1000 / 1600. (Two shorter sleeps in a row are worse than one: C3 2.74
  // at 200 + 200, 2.82 at 400 + 600.) With the last batch settled warp-wide
  // (flow_slot_conv) C4 takes 1.23 ms at 100 and 1.25 at 200.
  // The longer step pays only where many rows wait at once (C3: 73 units per
  // warp); with a few units per warp the chain itself binds and the shorter
  // sleep wins (s27, 2.4 units per warp: 0.88 ms at 400, 0.90 at 600; elast6
  // 0.35 / 0.43).
  const bool crowded = c->nflow >= 32LL * 32 * c->sm_count;
  int backoff = kb >= 3 ? (mean >= 16.0 ? (crowded ? 600 : 400) : 100) : 0;
  if (const char* e = std::getenv("TCG_FLOW_BACKOFF")) backoff = std::atoi(e);
  int pp_w = 0, pp_k = 0, pp_n = 0, pp_m = 0, pp_d = 0, pp_b = -1;
  bool pp = !remote && !c->opt.trace && phase == 0 && pick_pp(c, mean, &pp_w, &pp_k, &pp_n, &pp_m, &pp_d, &pp_b);
  if (pp) {
    if (pp_b < 0) pp_b = backoff;
    size_t pp_smem = 0;
    cudaError_t pe = tcbdev::pp_occupancy(pp_w, pp_k, pp_n, pp_m, extras, dmode, pp_b, pp_d, &occ, &pp_smem);
    if (pe != cudaSuccess && dmode) {
      cudaGetLastError();
      drain = chunks = false;
      dmode = 0;
      pe = tcbdev::pp_occupancy(pp_w, pp_k, pp_n, pp_m, extras, 0, pp_b, pp_d, &occ, &pp_smem);
    }
    if (pe != cudaSuccess) {
      cudaGetLastError();
      pp = false;
    }
  }
  if (!pp) {
    pipe = true;
    cudaError_t oe = tcbdev::pipe_occupancy(threads, kb, minb, remote, extras, &occ, dmode, backoff);
    if (oe != cudaSuccess && dmode) {  // no such variant: a copy after the launch
      cudaGetLastError();
      drain = chunks = false;
      dmode = 0;
      oe = tcbdev::pipe_occupancy(threads, kb, minb, remote, extras, &occ, 0, backoff);
    }
    // a back-off asked for by name must exist: a silent fall-back to none once made
    // every value above 400 ns of a sweep measure as 0
    if (std::getenv("TCG_FLOW_BACKOFF") && backoff > 0 && oe == cudaSuccess &&
        !tcbdev::pipe_variant_exists(threads, kb, minb, remote, extras, dmode, backoff)) {
      c->err = "no value-flow kernel variant with a " + std::to_string(backoff) +
               " ns back-off for this launch (TCG_FLOW_BACKOFF; see TCG_PIPE_VARIANTS)";
      return TCG_INVALID;
    }
    if (oe == cudaErrorInvalidValue) {
      cudaGetLastError();
      c->err = "no value-flow kernel variant for KB " + std::to_string(kb) + ", " + std::to_string(minb) +
               " CTAs/SM (TCG_FLOW_KB / TCG_FLOW_MINB)";
      return TCG_INVALID;
    }
    TCG_CUDA_TRY(c, oe);
  }
  if (occ < 1) {
    c->err = "value-flow kernel does not fit on an SM";
    return TCG_INVALID;
  }
  if (c->opt.ctas_per_sm > 0) occ = std::min(occ, c->opt.ctas_per_sm);
  if (const char* e = std::getenv("TCG_FLOW_CTAS")) occ = std::max(1, std::min(occ, std::atoi(e)));
  const int grid = std::max(1, occ * c->sm_count);
  if (drain && grid <= drain_ctas) {
    drain = false;
    dmode = 0;
  }
  const bool batch = c->nbatch > 1;
  if (static_cast<int64_t>(c->nflow) * c->nbatch > 0x7fffffffLL) {
    c->err = "value-flow batch: rows x members beyond 2^31";
    return TCG_INVALID;
  }
  double* const vals = batch ? c->bvals : c->vals;
  tcbdev::FlowPrepParams q{};
  q.vals = vals;
  q.a = batch ? c->ba : c->flow_a;
  // host_a: the device init below writes the restore copy too, which then
  // serves as the kernel's input
  const bool from_copy = (c->pristine && !host_in) || host_a;
  if (from_copy) q.a = batch ? c->bvals0 : c->vals0;
  q.out = vals;
  q.nnz = c->nnz * c->nbatch;
  q.ctrl = c->ctrl;
  q.m_failed = batch ? c->bm_flags : c->m_flags;
  q.m_row = q.m_failed + c->nbatch;
  q.m_pivot = batch ? c->bm_pivot : c->m_pivot;
  q.nbatch = c->nbatch;
  tcbdev::FlowParams P{};
  P.peers = c->peers;
  P.npeers = c->npeers;
  P.rec = c->flow_rec;
  P.item = c->flow_item;
  P.slot = c->flow_slot;
  P.upd = c->flow_upd;
  P.nupd = c->nflow_upd;
  P.a = q.a;
  if (from_copy) q.a = const_cast<double*>(q.vals);  // tells the prelude not to copy
  P.vals = vals;
  P.ctrl = c->ctrl;
  P.trace = c->opt.trace ? c->trace + 2 * c->ntab : nullptr;

  P.m_failed = q.m_failed;
  P.m_row = q.m_row;
  P.m_pivot = q.m_pivot;
  P.nnz = c->nnz;
  P.nbatch = c->nbatch;
  P.nrows = static_cast<int>(c->nflow);
  P.row_ctas = drain ? grid - drain_ctas : grid;
  const long long drain_words = (c->nnz * c->nbatch + 2047) / 2048;
  if (drain) {
    if (drain_words > c->drain_len) {
      TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (c->drain_done) TCG_CUDA_TRY(c, cudaFree(c->drain_done));
      c->drain_done = nullptr;
      TCG_CUDA_TRY(c, cudaMalloc(&c->drain_done, sizeof(unsigned) * drain_words));
      c->drain_len = drain_words;
    }
    P.drain_out = drain_out;
    P.drain_done = c->drain_done;
  }
  if (chunks) {
    P.chunk_left = c->chunk_left;
    P.chunk_flag = c->chunk_flag_d;
    P.nchunks = c->nchunks;
    P.chunk_seq = ++c->chunk_seq;
  }
  const double tmo = c->opt.timeout_s > 0 ? c->opt.timeout_s : 30.0;
  P.timeout_ns = static_cast<unsigned long long>(tmo * 1e9);
  const size_t vbytes = sizeof(double) * static_cast<size_t>(c->nnz) * c->nbatch;
  if (phase == 1) {  // sharded runs: every part resets its U before any part's kernel starts
    TCG_CUDA_TRY(c, tcbdev::launch_flow_prepare(q, c->sm_count, c->stream));
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return TCG_OK;
  }
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
  // host buffers: the upload goes first on the same stream. (Overlapping it
  // with the kernel, which then polled its inputs, saved ~5% but relied on
  // the copy running concurrently with the kernel, which CUDA does not
  // promise -- under a profiler it serialised and the launch stalled.)
  if (host_in) TCG_CUDA_TRY(c, cudaMemcpyAsync(vals, host_in, vbytes, cudaMemcpyHostToDevice, c->stream));
  if (host_a) {  // PᵀAP's values in, init_factor_values on the device (factorize.hpp:71-89)
    // A pinned, mapped input with long rows is gathered in place:
    // init_factor_values reads only the entries U starts from (A's upper
    // triangle, the tail of every row: half of a symmetric A), so the device
    // pulls those over PCIe instead of the copy engine moving all of A. With
    // short rows the halves share their 32-byte sectors and nothing is saved.
    // B200, end to end: C4 (81 entries per row) 3.97 -> 3.31 ms, C3 (27) 3.29 ->
    // 3.26; C2 / C6 (7) 0.96 -> 0.98 / 5.34 -> 5.70, hence the threshold.
    const double* a_src = c->a_stage;
    bool zero_copy = false;
    if (c->nnz_a > 0) {
      int want = c->nnz_a >= 16 * c->n ? 1 : 0;
      if (const char* e = std::getenv("TCG_A_ZEROCOPY")) want = std::atoi(e);
      cudaPointerAttributes attr{};
      if (want && cudaPointerGetAttributes(&attr, host_a) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
          attr.devicePointer) {
        a_src = static_cast<const double*>(attr.devicePointer);
        zero_copy = true;
      } else {
        cudaGetLastError();
      }
    }
    if (c->nnz_a > 0 && !zero_copy)
      TCG_CUDA_TRY(c, cudaMemcpyAsync(c->a_stage, host_a, sizeof(double) * c->nnz_a * c->nbatch,
                                      cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, tcbdev::launch_init_values(a_src, c->a_map, vals, batch ? c->bvals0 : c->vals0, c->nnz,
                                               c->nnz_a, c->nbatch, c->sm_count, c->stream));
  }
  if (phase == 0) TCG_CUDA_TRY(c, tcbdev::launch_flow_prepare(q, c->sm_count, c->stream));
  if (drain) TCG_CUDA_TRY(c, cudaMemsetAsync(c->drain_done, 0, sizeof(unsigned) * drain_words, c->stream));
  if (chunks)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->chunk_left, c->chunk_units, sizeof(int) * c->nchunks, cudaMemcpyDeviceToDevice,
                                    c->stream));
  P.ub = c->flow_ub;
  // the per-lane kernel's Chol pivot through shared memory, the waiting lanes
  // sleeping P.decouple ns between looks (flow_row; TCG_FLOW_DECOUPLE): it let
  // the lanes of a medium-program unit publish independently (C4 1.38 -> 1.30
  // ms at 100 ns) until the last batch was settled warp-wide, which brings the
  // lanes in together anyway (C4 now 1.23 ms without, 1.24 with): off.
  P.decouple = 0;
  if (const char* e = std::getenv("TCG_FLOW_DECOUPLE")) P.decouple = std::atoi(e);
  if (c->nflow > 0) {
    if (pp)
      TCG_CUDA_TRY(c, tcbdev::launch_flow_pp(P, grid, pp_w, pp_k, pp_n, pp_m, extras, dmode, pp_b, pp_d,
                                             c->stream));
    else
      TCG_CUDA_TRY(c, tcbdev::launch_flow_pipe(P, grid, threads, kb, minb, remote, extras, c->stream,
                                               dmode, backoff));
  }
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
  c->pristine = false;  // the working values now hold the factor
  if (host_out && !drain && !chunks)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(host_out, vals, vbytes, cudaMemcpyDeviceToHost, c->stream));
  if (chunks) {
    // the host issues each chunk's copy (adjacent chunks together) on the copy
    // stream as soon as the launch has flagged it; if the launch ends without
    // every flag (a watchdog stop), the rest is copied after it
    std::vector<char> sent(static_cast<size_t>(c->nchunks), 0);
    const volatile int* flag = c->chunk_flag;
    int left = c->nchunks;
    auto copy = [&](int k0, int k1) {  // chunks [k0, k1)
      const std::int64_t b = c->chunk_start[static_cast<size_t>(k0)], e = c->chunk_start[static_cast<size_t>(k1)];
      return cudaMemcpyAsync(host_out + b, vals + b, sizeof(double) * static_cast<size_t>(e - b),
                             cudaMemcpyDeviceToHost, c->d2h_stream);
    };
    unsigned idle = 0;
    while (left > 0) {
      bool any = false;
      for (int k = 0; k < c->nchunks; ++k) {
        if (sent[static_cast<size_t>(k)] || flag[k] != c->chunk_seq) continue;
        int k1 = k + 1;
        while (k1 < c->nchunks && !sent[static_cast<size_t>(k1)] && flag[k1] == c->chunk_seq) ++k1;
        TCG_CUDA_TRY(c, copy(k, k1));
        for (int x = k; x < k1; ++x) sent[static_cast<size_t>(x)] = 1;
        left -= k1 - k;
        any = true;
        k = k1 - 1;
      }
      if (any) {
        idle = 0;
      } else if (++idle >= 256) {
        idle = 0;
        const cudaError_t qe = cudaStreamQuery(c->stream);
        if (qe == cudaErrorNotReady) continue;
        TCG_CUDA_TRY(c, qe);
        bool all = true;  // the launch is over: its flags are all there, unless it was stopped
        for (int k = 0; k < c->nchunks; ++k) all = all && (sent[static_cast<size_t>(k)] || flag[k] == c->chunk_seq);
        if (all) continue;
        for (int k = 0; k < c->nchunks; ++k)
          if (!sent[static_cast<size_t>(k)]) TCG_CUDA_TRY(c, copy(k, k + 1));
        left = 0;
      }
    }
    TCG_CUDA_TRY(c, cudaEventRecord(c->ev3, c->d2h_stream));
    TCG_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev3, 0));
  }
  if (calibrating) TCG_CUDA_TRY(c, cudaEventRecord(c->ev2, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->host_ctrl, c->ctrl, sizeof(tcbdev::Ctrl),
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  TCG_CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (calibrating) {
    float whole = 0.f;
    TCG_CUDA_TRY(c, cudaEventElapsedTime(&whole, c->ev0, c->ev2));
    float& best = c->drain_ms[dmode];
    if (best < 0.f || whole < best) best = whole;
    ++c->drain_calls;
  }
  const tcbdev::Ctrl& h = *c->host_ctrl;
  S.device_ms = ms;
  S.grid_ctas = grid;
  S.threads_per_cta = threads;
  S.staging_cap = kb;  // reported: gather batch
  S.kernel_launches = (c->nflow > 0 ? 1 : 0) + (phase == 0 ? 1 : 0) + (host_a ? 1 : 0);
  S.mode = 5;
  S.drain_ctas = drain ? drain_ctas : chunks ? -c->nchunks : 0;  // (negative: chunked copies, their count)
  if (host_a) c->pristine = false;
  S.lanes_per_row = pp ? 32 * pp_w : 32;
  S.row_kernel = pp ? 2 : 1;
  S.flow_depth = c->flow_depth;
  S.flow_depth = c->flow_depth;
  if (pp) S.threads_per_cta = 256;
  if (pp) S.staging_cap = pp_k;
  const int64_t rows = c->nflow * c->nbatch;
  S.tasks_completed = (h.done.v == rows) ? c->ntasks * c->nbatch : 0;
  S.tasks_executed = h.executed.v;
  S.batch = c->nbatch;
  if (h.error.v) {
    c->err = "device watchdog expired: the value-flow schedule stalled";
    return TCG_TIMEOUT;
  }
  if (h.done.v != rows) {
    c->err = "value-flow schedule finished " + std::to_string(h.done.v) + " of " +
             std::to_string(rows) + " rows";
    return TCG_TIMEOUT;
  }
  if (h.failed.v) {
    S.breakdown_row = h.fail_row;
    S.breakdown_pivot = h.fail_pivot;
    S.breakdown_member = h.fail_member;
    c->err = "factorization breakdown at row " + std::to_string(h.fail_row) + ": pivot " +
             std::to_string(h.fail_pivot) + " is not positive" +
             (batch ? " (member " + std::to_string(h.fail_member) + ")" : std::string());
    return TCG_BREAKDOWN;
  }
  return TCG_OK;
}

tcg_status tcg_factor(tcg_ctx* c, tcg_stats* st) {
  if (!c || !c->uploaded) return TCG_INVALID;
  tcg_stats local{};
  tcg_stats& S = st ? *st : local;
  S = tcg_stats{};
  S.breakdown_row = -1;
  S.breakdown_member = -1;
  S.batch = 1;
  if (c->ntasks == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));

  const int threads = c->opt.threads_per_cta ? c->opt.threads_per_cta : 256;
  int mode = c->opt.mode;
  if (mode == 0)  // value flow wherever the problem has its tables (the default); else the task DAG
    mode = c->has_flow ? 5 : (c->has_programs ? 2 : 1);
  if (((mode == 1 || mode == 2) && c->ntab == 0) || (mode == 2 && !c->has_programs) ||
      (mode == 5 && !c->has_flow) || (mode != 1 && mode != 2 && mode != 5)) {
    c->err = "requested execution mode is not available for the uploaded problem (1, 2: task DAG, "
             "needs tcg_plan_expand; 5: value flow)";
    return TCG_INVALID;
  }
  if (mode != 5 && c->nbatch > 1) {
    c->err = "a batch of value sets needs mode 5 (value flow)";
    return TCG_INVALID;
  }
  if (mode != 5 && (threads == 384 || threads == 768)) {
    c->err = "threads_per_cta 384 and 768 are for mode 5 only";
    return TCG_INVALID;
  }
  if (mode != 5) c->pristine = false;  // the task executors factor the working values in place
  if (mode == 5) return run_flow(c, S, threads);
  int flag_words = (c->max_flag_rows + 31) / 32;
  flag_words = (flag_words + 3) & ~3;
  int cap = c->opt.staging_cap;
  if (cap <= 0) cap = std::min(256, std::max(32, (c->max_target_len + 31) / 32 * 32));
  cap = (cap + 3) & ~3;
  // task metadata staged per single-CTA task (items x 32 B, sources x 16 B)
  int icap = 256, scap = 1024;
  if (const char* e = std::getenv("TCG_ICAP")) icap = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("TCG_SCAP")) scap = std::max(0, std::atoi(e));
  size_t smem = tcbdev::factor_smem_bytes(threads, cap, flag_words, icap, scap);
  const size_t kMaxSmem = 227 * 1024;
  while (smem > kMaxSmem && (cap > 32 || scap > 0)) {
    if (scap > 0) {
      scap /= 2;
      icap /= 2;
    } else {
      cap = std::max(32, cap / 2);
    }
    smem = tcbdev::factor_smem_bytes(threads, cap, flag_words, icap, scap);
  }
  if (smem > kMaxSmem) {
    c->err = "diagonal range too large for the shared-memory row flags (" +
             std::to_string(c->max_flag_rows) + " rows)";
    return TCG_INVALID;
  }
  int occ = 0;
  TCG_CUDA_TRY(c, tcbdev::factor_occupancy(threads, smem, &occ));
  if (occ < 1) {
    c->err = "persistent kernel does not fit on an SM";
    return TCG_INVALID;
  }
  if (c->opt.ctas_per_sm > 0) occ = std::min(occ, c->opt.ctas_per_sm);
  const int grid = std::max(1, occ * c->sm_count);

  tcbdev::PrepParams q{};
  q.indeg0 = c->indeg0;
  q.roots = c->roots;
  q.indeg = c->indeg;
  q.queue = c->queue;
  q.queue2 = nullptr;
  q.claim = c->claim;
  q.fin = c->fin;
  q.ctrl = c->ctrl;
  q.qcap = static_cast<int>(c->qcap);
  q.ntasks = static_cast<int>(c->ntab);
  q.nroots = static_cast<int>(c->nroots);
  TCG_CUDA_TRY(c, tcbdev::launch_prepare(q, c->stream));

  tcbdev::Params P{};
  P.tasks = c->tasks;
  P.items = c->items;
  P.srcs = c->srcs;
  P.succ = c->succ;
  P.cols = c->cols;
  P.vals = c->vals;
  P.indeg = c->indeg;
  P.queue = c->queue;
  P.claim = c->claim;
  P.fin = c->fin;
  P.iflag = c->iflag;
  P.ctrl = c->ctrl;
  P.qcap = static_cast<int>(c->qcap);
  P.epoch = ++c->epoch;
  P.trace = c->opt.trace ? c->trace : nullptr;
  P.itrace = c->opt.trace ? c->trace + 2 * c->ntab : nullptr;
  P.ntasks = static_cast<int>(c->ntab);
  P.cap = cap;
  P.flag_words = flag_words;
  P.icap = icap;
  P.slot_rec = c->slot_rec;
  P.upd = c->upd;
  P.mode = mode;
  P.scap = scap;
  const double tmo = c->opt.timeout_s > 0 ? c->opt.timeout_s : 30.0;
  P.timeout_ns = static_cast<unsigned long long>(tmo * 1e9);
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
  TCG_CUDA_TRY(c, tcbdev::launch_factor(P, grid, threads, smem, c->stream));
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->host_ctrl, c->ctrl, sizeof(tcbdev::Ctrl),
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  TCG_CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  const tcbdev::Ctrl& h = *c->host_ctrl;
  S.device_ms = ms;
  S.tasks_completed = h.done.v;
  S.tasks_executed = h.executed.v;
  S.grid_ctas = grid;
  S.threads_per_cta = threads;
  S.staging_cap = cap;
  S.smem_bytes = static_cast<int64_t>(smem);
  S.kernel_launches = 2;
  S.helpers_run = h.helpers_run.v;
  S.mode = mode;
  if (h.error.v) {
    c->err = h.error.v == 1 ? "device watchdog expired: the task DAG stalled" : "device capacity error";
    return TCG_TIMEOUT;
  }
  if (h.done.v != c->ntab) {
    c->err = "scheduler finished with " + std::to_string(h.done.v) + " of " +
             std::to_string(c->ntab) + " tasks";
    return TCG_TIMEOUT;
  }
  if (h.failed.v) {
    S.breakdown_row = h.fail_row;
    S.breakdown_pivot = h.fail_pivot;
    c->err = "factorization breakdown at row " + std::to_string(h.fail_row) + ": pivot " +
             std::to_string(h.fail_pivot) + " is not positive";
    return TCG_BREAKDOWN;
  }
  return TCG_OK;
}

tcg_status tcg_download(tcg_ctx* c, double* values) {
  if (!c || !c->uploaded || (!values && c->nnz > 0)) return TCG_INVALID;
  if (c->nnz == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(values, c->vals, sizeof(double) * c->nnz,
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TCG_OK;
}

tcg_status tcg_factor_phase(tcg_ctx* c, int32_t phase, tcg_stats* st) {
  if (!c || !c->uploaded || phase < 0 || phase > 2) return TCG_INVALID;
  if (phase == 0) return tcg_factor(c, st);
  if (!c->has_flow || (c->opt.mode != 0 && c->opt.mode != 5)) {
    c->err = "tcg_factor_phase: split phases exist in mode 5 only";
    return TCG_INVALID;
  }
  tcg_stats local{};
  tcg_stats& S = st ? *st : local;
  S = tcg_stats{};
  S.breakdown_row = -1;
  S.breakdown_member = -1;
  S.batch = 1;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  const int threads = c->opt.threads_per_cta ? c->opt.threads_per_cta : 256;
  return run_flow(c, S, threads, nullptr, nullptr, phase);
}

tcg_status tcg_factor_host(tcg_ctx* c, const double* values_in, double* values_out, tcg_stats* st) {
  if (!c || !c->uploaded || ((!values_in || !values_out) && c->nnz > 0)) return TCG_INVALID;
  int mode = c->opt.mode;
  const bool flow = c->has_flow && c->nnz > 0 && c->ntasks > 0 && (mode == 0 || mode == 5);
  if (!flow) {  // other modes: the same three steps, one after the other
    tcg_status r = c->nbatch > 1 ? tcg_set_batch_values(c, values_in) : tcg_set_values(c, values_in);
    if (r != TCG_OK) return r;
    const tcg_status f = tcg_factor(c, st);
    r = c->nbatch > 1 ? tcg_download_batch(c, values_out) : tcg_download(c, values_out);
    return f != TCG_OK ? f : r;
  }
  tcg_stats local{};
  tcg_stats& S = st ? *st : local;
  S = tcg_stats{};
  S.breakdown_row = -1;
  S.breakdown_member = -1;
  S.batch = 1;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  const int threads = c->opt.threads_per_cta ? c->opt.threads_per_cta : 256;
  return run_flow(c, S, threads, values_in, values_out);
}

// C5-style batches end to end, pipelined: the members in chunks, one launch
// per chunk; the upload of chunk i+1 (copy stream) and the download of chunk
// i-1 (another copy stream) run beside the factorization of chunk i (events
// order them; if the copies do not overlap, the result is the same, later).
// Same kernels and arithmetic as one launch over the whole batch.
static tcg_status run_flow_chunked(tcg_ctx* c, tcg_stats& S, int threads, const double* host_a,
                                   double* host_out, int chunks) {
  const double mean = c->nnz > 0 ? static_cast<double>(c->nflow_upd) / static_cast<double>(c->nnz) : 0.0;
  // 4 CTAs per SM: a fifth made the batch kernel slower (C5 x 64: 1.81 -> 1.95 ms)
  const int kb = mean <= 4.0 ? 2 : 3, minb = 3;
  int backoff = kb >= 3 ? 200 : 0;
  if (const char* e = std::getenv("TCG_FLOW_BACKOFF")) backoff = std::atoi(e);
  int occ = 0;
  int pp_w = 0, pp_k = 0, pp_n = 0, pp_m = 0, pp_d = 0, pp_b = -1;
  bool pp = !c->opt.trace && pick_pp(c, mean, &pp_w, &pp_k, &pp_n, &pp_m, &pp_d, &pp_b);
  if (pp) {
    if (pp_b < 0) pp_b = backoff;
    size_t smem = 0;
    if (tcbdev::pp_occupancy(pp_w, pp_k, pp_n, pp_m, 1, 0, pp_b, pp_d, &occ, &smem) != cudaSuccess) {
      cudaGetLastError();
      pp = false;
    }
  }
  if (!pp) TCG_CUDA_TRY(c, tcbdev::pipe_occupancy(threads, kb, minb, 0, 1, &occ, 0, backoff));
  if (occ < 1) {
    c->err = "value-flow kernel does not fit on an SM";
    return TCG_INVALID;
  }
  if (c->opt.ctas_per_sm > 0) occ = std::min(occ, c->opt.ctas_per_sm);
  const int grid = std::max(1, occ * c->sm_count);
  const int nb = c->nbatch;
  if (!c->h2d_stream) TCG_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
  if (!c->d2h_stream) TCG_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
  while (static_cast<int>(c->chunk_ev.size()) < 2 * chunks + 1) {
    cudaEvent_t e = nullptr;
    TCG_CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->chunk_ev.push_back(e);
  }
  if (c->host_ctrls_len < chunks) {
    if (c->host_ctrls) TCG_CUDA_TRY(c, cudaFreeHost(c->host_ctrls));
    c->host_ctrls = nullptr;
    TCG_CUDA_TRY(c, cudaMallocHost(reinterpret_cast<void**>(&c->host_ctrls), sizeof(tcbdev::Ctrl) * chunks));
    c->host_ctrls_len = chunks;
  }
  const double tmo = c->opt.timeout_s > 0 ? c->opt.timeout_s : 30.0;
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev0, c->stream));
  TCG_CUDA_TRY(c, cudaStreamWaitEvent(c->h2d_stream, c->ev0, 0));
  for (int k = 0; k < chunks; ++k) {
    const int m0 = static_cast<int>(static_cast<long long>(nb) * k / chunks);
    const int m1 = static_cast<int>(static_cast<long long>(nb) * (k + 1) / chunks);
    const int nk = m1 - m0;
    cudaEvent_t up = c->chunk_ev[2 * k], done = c->chunk_ev[2 * k + 1];
    double* vals = c->bvals + static_cast<long long>(m0) * c->nnz;
    double* vals0 = c->bvals0 + static_cast<long long>(m0) * c->nnz;
    const double* stage = c->a_stage + static_cast<long long>(m0) * c->nnz_a;
    if (c->nnz_a > 0)
      TCG_CUDA_TRY(c, cudaMemcpyAsync(const_cast<double*>(stage), host_a + static_cast<long long>(m0) * c->nnz_a,
                                      sizeof(double) * c->nnz_a * nk, cudaMemcpyHostToDevice, c->h2d_stream));
    TCG_CUDA_TRY(c, cudaEventRecord(up, c->h2d_stream));
    TCG_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, up, 0));
    TCG_CUDA_TRY(c, tcbdev::launch_init_values(stage, c->a_map, vals, vals0, c->nnz, c->nnz_a, nk, c->sm_count,
                                               c->stream));
    tcbdev::FlowPrepParams q{};
    q.vals = vals;
    q.a = vals;  // the input is the restore copy the init wrote: no snapshot
    q.out = vals;
    q.nnz = c->nnz * nk;
    q.ctrl = c->ctrl;
    q.m_failed = c->bm_flags + m0;
    q.m_row = c->bm_flags + nb + m0;
    q.m_pivot = c->bm_pivot + m0;
    q.nbatch = nk;
    TCG_CUDA_TRY(c, tcbdev::launch_flow_prepare(q, c->sm_count, c->stream));
    tcbdev::FlowParams P{};
    P.rec = c->flow_rec;
    P.item = c->flow_item;
    P.slot = c->flow_slot;
    P.upd = c->flow_upd;
    P.nupd = c->nflow_upd;
    P.a = vals0;
    P.vals = vals;
    P.ctrl = c->ctrl;
    P.m_failed = q.m_failed;
    P.m_row = q.m_row;
    P.m_pivot = q.m_pivot;
    P.nnz = c->nnz;
    P.nbatch = nk;
    P.nrows = static_cast<int>(c->nflow);
    P.timeout_ns = static_cast<unsigned long long>(tmo * 1e9);
    P.row_ctas = grid;
    P.ub = c->flow_ub;
    if (pp)
      TCG_CUDA_TRY(c, tcbdev::launch_flow_pp(P, grid, pp_w, pp_k, pp_n, pp_m, 1, 0, pp_b, pp_d, c->stream));
    else
      TCG_CUDA_TRY(c, tcbdev::launch_flow_pipe(P, grid, threads, kb, minb, 0, 1, c->stream, 0, backoff));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->host_ctrls + k, c->ctrl, sizeof(tcbdev::Ctrl), cudaMemcpyDeviceToHost,
                                    c->stream));
    TCG_CUDA_TRY(c, cudaEventRecord(done, c->stream));
    TCG_CUDA_TRY(c, cudaStreamWaitEvent(c->d2h_stream, done, 0));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(host_out + static_cast<long long>(m0) * c->nnz, vals,
                                    sizeof(double) * c->nnz * nk, cudaMemcpyDeviceToHost, c->d2h_stream));
  }
  TCG_CUDA_TRY(c, cudaEventRecord(c->ev1, c->stream));
  TCG_CUDA_TRY(c, cudaEventRecord(c->chunk_ev[2 * chunks], c->d2h_stream));
  TCG_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->chunk_ev[2 * chunks], 0));  // later work sees the copies done
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->d2h_stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  TCG_CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->pristine = false;
  S.device_ms = ms;
  S.grid_ctas = grid;
  S.threads_per_cta = threads;
  S.staging_cap = pp ? pp_k : kb;
  S.kernel_launches = 3 * chunks;
  S.mode = 5;
  S.lanes_per_row = pp ? 32 * pp_w : 32;
  S.row_kernel = pp ? 2 : 1;
  S.flow_depth = c->flow_depth;
  S.batch = nb;
  S.chunks = chunks;
  bool error = false;
  int64_t rows = 0, executed = 0;
  for (int k = 0; k < chunks; ++k) {
    const tcbdev::Ctrl& h = c->host_ctrls[k];
    const int m0 = static_cast<int>(static_cast<long long>(nb) * k / chunks);
    error = error || h.error.v;
    rows += h.done.v;
    executed += h.executed.v;
    if (h.failed.v && S.breakdown_row < 0) {
      S.breakdown_row = h.fail_row;
      S.breakdown_pivot = h.fail_pivot;
      S.breakdown_member = h.fail_member + m0;
    }
  }
  S.tasks_completed = rows == c->nflow * nb ? c->ntasks * nb : 0;
  S.tasks_executed = executed;
  if (error) {
    c->err = "device watchdog expired: the value-flow schedule stalled";
    return TCG_TIMEOUT;
  }
  if (rows != c->nflow * nb) {
    c->err = "value-flow schedule finished " + std::to_string(rows) + " of " + std::to_string(c->nflow * nb) +
             " rows";
    return TCG_TIMEOUT;
  }
  if (S.breakdown_row >= 0) {
    c->err = "factorization breakdown at row " + std::to_string(S.breakdown_row) + ": pivot " +
             std::to_string(S.breakdown_pivot) + " is not positive (member " +
             std::to_string(S.breakdown_member) + ")";
    return TCG_BREAKDOWN;
  }
  return TCG_OK;
}

tcg_status tcg_factor_host_a(tcg_ctx* c, const double* a_values, double* values_out, tcg_stats* st) {
  if (!c || !c->uploaded || ((!a_values && c->nnz_a > 0) || (!values_out && c->nnz > 0))) return TCG_INVALID;
  if (!c->a_map) {
    c->err = "tcg_factor_host_a: the problem has no A -> U map (duplicate entries in A?)";
    return TCG_INVALID;
  }
  const bool flow = c->has_flow && c->nnz > 0 && c->ntasks > 0 && (c->opt.mode == 0 || c->opt.mode == 5);
  if (!flow) {  // other modes: the same steps, one after the other
    tcg_status r = tcg_set_a_values(c, c->nbatch, a_values);
    if (r != TCG_OK) return r;
    const tcg_status f = tcg_factor(c, st);
    r = c->nbatch > 1 ? tcg_download_batch(c, values_out) : tcg_download(c, values_out);
    return f != TCG_OK ? f : r;
  }
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  const int64_t need = c->nnz_a * c->nbatch;  // staging for A (outside the timed region)
  if (need > c->a_stage_len) {
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->a_stage) TCG_CUDA_TRY(c, cudaFree(c->a_stage));
    c->a_stage = nullptr;
    TCG_CUDA_TRY(c, cudaMalloc(&c->a_stage, sizeof(double) * std::max<int64_t>(need, 1)));
    c->a_stage_len = need;
  }
  tcg_stats local{};
  tcg_stats& S = st ? *st : local;
  S = tcg_stats{};
  S.breakdown_row = -1;
  S.breakdown_member = -1;
  S.batch = c->nbatch;
  const int threads = c->opt.threads_per_cta ? c->opt.threads_per_cta : 256;
  // batches of 8 or more: pipelined over 4 member chunks, 8 from 32 members on (TCG_CHUNKS
  // overrides; 1 = one launch). B200, 64 C5 matrices end to end: 5.37 / 4.19 / 3.49 / 3.37 /
  // 4.35 ms at 1 / 2 / 4 / 8 / 16 chunks.
  int chunks = c->nbatch >= 32 ? 8 : c->nbatch >= 8 ? 4 : 1;
  if (const char* e = std::getenv("TCG_CHUNKS")) chunks = std::max(1, std::atoi(e));
  chunks = std::min(chunks, c->nbatch);
  if (chunks > 1 && threads == 256 && !c->opt.trace && c->npeers <= 1)
    return run_flow_chunked(c, S, threads, a_values, values_out, chunks);
  return run_flow(c, S, threads, nullptr, values_out, 0, a_values);
}

tcg_status tcg_set_batch(tcg_ctx* c, int32_t nbatch, const double* values) {
  if (!c || !c->uploaded || nbatch < 1 || (!values && c->nnz > 0)) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->batch_arena) {
    TCG_CUDA_TRY(c, cudaFree(c->batch_arena));
    c->batch_arena = nullptr;
  }
  c->nbatch = 1;
  c->drain_ms[0] = c->drain_ms[1] = c->drain_ms[2] = -1.f;
  c->drain_calls = 0;
  if (nbatch == 1) return tcg_set_values(c, values);
  if (!c->has_flow) {
    c->err = "tcg_set_batch: the plan has no value-flow tables (mode 5)";
    return TCG_INVALID;
  }
  const size_t vb = sizeof(double) * static_cast<size_t>(c->nnz) * nbatch;
  const size_t fb = align_up(sizeof(int) * 2 * nbatch, 256);
  const size_t bytes = 3 * align_up(vb, 256) + fb + sizeof(double) * nbatch;
  TCG_CUDA_TRY(c, cudaMalloc(&c->batch_arena, bytes));
  char* base = static_cast<char*>(c->batch_arena);
  c->bvals = reinterpret_cast<double*>(base);
  c->bvals0 = reinterpret_cast<double*>(base + align_up(vb, 256));
  c->ba = reinterpret_cast<double*>(base + 2 * align_up(vb, 256));
  c->bm_flags = reinterpret_cast<int*>(base + 3 * align_up(vb, 256));
  c->bm_pivot = reinterpret_cast<double*>(base + 3 * align_up(vb, 256) + fb);
  c->nbatch = nbatch;
  c->drain_ms[0] = c->drain_ms[1] = c->drain_ms[2] = -1.f;
  c->drain_calls = 0;
  if (vb) {
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->bvals0, values, vb, cudaMemcpyHostToDevice, c->stream));
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->bvals, c->bvals0, vb, cudaMemcpyDeviceToDevice, c->stream));
  }
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->pristine = true;
  return TCG_OK;
}

tcg_status tcg_set_a_values(tcg_ctx* c, int32_t nbatch, const double* a_values) {
  if (!c || !c->uploaded || nbatch < 1 || (!a_values && c->nnz_a > 0)) return TCG_INVALID;
  if (!c->a_map) {
    c->err = "tcg_set_a_values: the problem has no A -> U map (duplicate entries in A?)";
    return TCG_INVALID;
  }
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (nbatch != c->nbatch) {  // resize the batch (values are overwritten below)
    if (nbatch > 1) {
      std::vector<double> zeros;  // tcg_set_batch needs host values; use a cheap device path instead
      TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (c->batch_arena) {
        TCG_CUDA_TRY(c, cudaFree(c->batch_arena));
        c->batch_arena = nullptr;
      }
      const size_t vb = sizeof(double) * static_cast<size_t>(c->nnz) * nbatch;
      const size_t fb = align_up(sizeof(int) * 2 * nbatch, 256);
      TCG_CUDA_TRY(c, cudaMalloc(&c->batch_arena, 3 * align_up(vb, 256) + fb + sizeof(double) * nbatch));
      char* base = static_cast<char*>(c->batch_arena);
      c->bvals = reinterpret_cast<double*>(base);
      c->bvals0 = reinterpret_cast<double*>(base + align_up(vb, 256));
      c->ba = reinterpret_cast<double*>(base + 2 * align_up(vb, 256));
      c->bm_flags = reinterpret_cast<int*>(base + 3 * align_up(vb, 256));
      c->bm_pivot = reinterpret_cast<double*>(base + 3 * align_up(vb, 256) + fb);
    } else if (c->batch_arena) {
      TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      TCG_CUDA_TRY(c, cudaFree(c->batch_arena));
      c->batch_arena = nullptr;
    }
    c->nbatch = nbatch;
    c->drain_ms[0] = c->drain_ms[1] = c->drain_ms[2] = -1.f;
    c->drain_calls = 0;
  }
  const int64_t need = c->nnz_a * nbatch;
  if (need > c->a_stage_len) {
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->a_stage) TCG_CUDA_TRY(c, cudaFree(c->a_stage));
    c->a_stage = nullptr;
    TCG_CUDA_TRY(c, cudaMalloc(&c->a_stage, sizeof(double) * std::max<int64_t>(need, 1)));
    c->a_stage_len = need;
  }
  if (need > 0)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(c->a_stage, a_values, sizeof(double) * need, cudaMemcpyHostToDevice,
                                    c->stream));
  double* v = nbatch > 1 ? c->bvals : c->vals;
  double* v0 = nbatch > 1 ? c->bvals0 : c->vals0;
  TCG_CUDA_TRY(c, tcbdev::launch_init_values(c->a_stage, c->a_map, v, v0, c->nnz, c->nnz_a, nbatch,
                                             c->sm_count, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->pristine = true;
  return TCG_OK;
}

tcg_status tcg_set_batch_values(tcg_ctx* c, const double* values) {
  if (!c || !c->uploaded || (!values && c->nnz > 0)) return TCG_INVALID;
  if (c->nbatch == 1) return tcg_set_values(c, values);
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t vb = sizeof(double) * static_cast<size_t>(c->nnz) * c->nbatch;
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->bvals0, values, vb, cudaMemcpyHostToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(c->bvals, c->bvals0, vb, cudaMemcpyDeviceToDevice, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->pristine = true;
  return TCG_OK;
}

int32_t tcg_batch_size(const tcg_ctx* c) { return c ? c->nbatch : 0; }

tcg_status tcg_download_batch(tcg_ctx* c, double* values) {
  if (!c || !c->uploaded || (!values && c->nnz > 0)) return TCG_INVALID;
  if (c->nbatch == 1) return tcg_download(c, values);
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(values, c->bvals, sizeof(double) * c->nnz * c->nbatch,
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TCG_OK;
}

tcg_status tcg_batch_breakdown(tcg_ctx* c, int32_t* rows, double* pivots) {
  if (!c || !c->uploaded || !rows || !pivots) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  const int* flags = c->nbatch > 1 ? c->bm_flags : c->m_flags;
  const double* piv = c->nbatch > 1 ? c->bm_pivot : c->m_pivot;
  TCG_CUDA_TRY(c, cudaMemcpyAsync(rows, flags + c->nbatch, sizeof(int) * c->nbatch,
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(pivots, piv, sizeof(double) * c->nbatch, cudaMemcpyDeviceToHost,
                                  c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TCG_OK;
}

tcg_status tcg_download_trace(tcg_ctx* c, uint64_t* stamps) {
  if (!c || !c->uploaded || !stamps) return TCG_INVALID;
  if (c->ntasks == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  TCG_CUDA_TRY(c, cudaMemcpyAsync(stamps, c->trace, sizeof(uint64_t) * (2 * c->ntab + 4 * std::max(c->nitems, c->nflow)),
                                  cudaMemcpyDeviceToHost, c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TCG_OK;
}

tcg_status tcg_flow_records(tcg_ctx* c, int32_t* rec, int32_t* item, int32_t* depth) {
  if (!c || !c->uploaded || !c->has_flow) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (rec) TCG_CUDA_TRY(c, cudaMemcpy(rec, c->flow_rec, sizeof(int4) * c->nflow, cudaMemcpyDeviceToHost));
  if (item) TCG_CUDA_TRY(c, cudaMemcpy(item, c->flow_item, sizeof(int) * c->nflow, cudaMemcpyDeviceToHost));
  if (depth) *depth = c->flow_depth;
  return TCG_OK;
}

tcg_status tcg_flow_programs(tcg_ctx* c, int32_t* slot, int32_t* upd, int64_t* nupd, double* build_ms) {
  if (!c || !c->uploaded || !c->has_flow) return TCG_INVALID;
  if (nupd) *nupd = c->nflow_upd;
  if (build_ms) *build_ms = c->prog_build_ms;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (slot && c->nnz > 0)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(slot, c->flow_slot, sizeof(int4) * c->nnz, cudaMemcpyDeviceToHost, c->stream));
  if (upd && c->nflow_upd > 0)
    TCG_CUDA_TRY(c, cudaMemcpyAsync(upd, c->flow_upd, sizeof(int2) * c->nflow_upd, cudaMemcpyDeviceToHost,
                                    c->stream));
  TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TCG_OK;
}

tcg_status tcg_device_values(tcg_ctx* c, double** dptr, int64_t* nnz) {
  if (!c || !c->uploaded) return TCG_INVALID;
  c->pristine = false;  // the caller may write the working values
  if (dptr) *dptr = c->vals;
  if (nnz) *nnz = c->nnz;
  return TCG_OK;
}

int64_t tcg_arena_bytes(const tcg_ctx* c) { return c ? static_cast<int64_t>(c->arena_bytes) : 0; }

tcg_status tcg_set_peers(tcg_ctx* c, int32_t nparts, const uint64_t* values_ptrs) {
  if (!c || nparts < 0 || nparts > 64 || (nparts > 0 && !values_ptrs)) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->peers) {
    TCG_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    TCG_CUDA_TRY(c, cudaFree(c->peers));
    c->peers = nullptr;
  }
  c->npeers = nparts;
  if (nparts == 0) return TCG_OK;
  TCG_CUDA_TRY(c, cudaMalloc(&c->peers, sizeof(double*) * nparts));
  TCG_CUDA_TRY(c, cudaMemcpy(c->peers, values_ptrs, sizeof(double*) * nparts, cudaMemcpyHostToDevice));
  return TCG_OK;
}

tcg_status tcg_ipc_values_handle(tcg_ctx* c, void* handle, int64_t* offset) {
  if (!c || !c->uploaded || !handle || !offset) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  TCG_CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->arena));
  std::memcpy(handle, &h, sizeof(h));
  *offset = static_cast<int64_t>(reinterpret_cast<char*>(c->vals) - static_cast<char*>(c->arena));
  return TCG_OK;
}

tcg_status tcg_ipc_open(tcg_ctx* c, const void* handle, int64_t offset, uint64_t* values_ptr) {
  if (!c || !handle || !values_ptr || offset < 0) return TCG_INVALID;
  TCG_CUDA_TRY(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  TCG_CUDA_TRY(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->ipc_opened.push_back(p);
  *values_ptr = reinterpret_cast<uint64_t>(static_cast<char*>(p) + offset);
  return TCG_OK;
}

// ------------------------------------------------------------ analysis ----

struct tch_matrix {
  tcb::CsrMatrix m;
};
struct tch_analysis {
  tcb::Analysis an;
  std::vector<int32_t> bounds;
};

tch_matrix* tch_generate(const char* kind, int64_t p0, int64_t p1, uint64_t seed) {
  try {
    if (!kind) throw std::invalid_argument("null kind");
    const std::string k(kind);
    auto out = std::make_unique<tch_matrix>();
    const auto i0 = static_cast<tcb::index_t>(p0);
    if (p0 < 0 || p0 > (1LL << 24)) throw std::invalid_argument("size out of range");
    if (k == "grid2d") out->m = tcb::grid_laplacian_2d(i0, static_cast<tcb::index_t>(p1));
    else if (k == "lap7") out->m = tcb::laplacian_7pt(i0);
    else if (k == "stencil27") out->m = tcb::stencil27_variable(i0, seed);
    else if (k == "elasticity") out->m = tcb::elasticity27(i0, seed);
    else if (k == "diffusion") out->m = tcb::diffusion_7pt_lognormal(i0, seed, static_cast<double>(p1) / 1000.0);
    else if (k == "path") out->m = tcb::path_matrix(i0, 2.0);
    else if (k == "random_spd")
      out->m = tcb::random_spd(i0, static_cast<double>(p1) / 1e6, static_cast<std::uint32_t>(seed));
    else throw std::invalid_argument("unknown generator '" + k + "'");
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

tch_matrix* tch_matrix_from_csr(const tcg_csr_view* view) {
  try {
    auto out = std::make_unique<tch_matrix>();
    out->m = csr_from_view(view, true);
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

void tch_matrix_free(tch_matrix* m) { delete m; }
void tch_matrix_view(const tch_matrix* m, tcg_csr_view* out) {
  if (m && out) view_of(m->m, out);
}

tch_analysis* tch_analyze(const tch_matrix* a, int32_t level, int32_t treecut, int32_t leaf_size,
                          int32_t max_depth, int32_t threads) {
  try {
    if (!a) throw std::invalid_argument("null matrix");
    tcb::AnalyzeOptions opt;
    opt.level = level;
    opt.treecut = treecut;
    opt.leaf_size = leaf_size;
    opt.max_depth = max_depth;
    auto out = std::make_unique<tch_analysis>();
    out->an = tcb::analyze(a->m, opt, threads);
    out->bounds.clear();
    for (const tcb::Range& r : out->an.ranges.ranges) {
      if (out->bounds.empty()) out->bounds.push_back(r.begin);
      out->bounds.push_back(r.end);
    }
    if (out->bounds.empty()) out->bounds.push_back(0);
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

tch_matrix* tch_load_matrix_market(const char* path) {
  try {
    if (!path) throw std::invalid_argument("null path");
    auto out = std::make_unique<tch_matrix>();
    out->m = tcb::load_matrix_market(path);
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

tcg_status tch_write_matrix_market(const tcg_csr_view* m, const char* path) {
  try {
    if (!path) throw std::invalid_argument("null path");
    tcb::write_matrix_market(csr_from_view(m, true), path);
    return TCG_OK;
  } catch (const std::invalid_argument& e) {
    g_tch_error = e.what();
    return TCG_INVALID;
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return TCG_INVALID;
  }
}

int32_t tch_load_ordering(const char* path, int32_t n, int32_t* perm, int32_t cap, int32_t* bounds) {
  try {
    if (!path) throw std::invalid_argument("null path");
    auto [p, rl] = tcb::load_ordering(path, n);
    if (perm) std::copy(p.perm.begin(), p.perm.end(), perm);
    const int32_t count = rl.count();
    if (bounds && cap >= count) {
      bounds[0] = count ? rl.ranges[0].begin : 0;
      for (int32_t k = 0; k < count; ++k) bounds[k + 1] = rl.ranges[static_cast<size_t>(k)].end;
    }
    return count;
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return -1;
  }
}

tch_analysis* tch_analyze_with_ordering(const tch_matrix* a, const int32_t* perm, int32_t nranges,
                                        const int32_t* bounds, int32_t level, int32_t threads) {
  try {
    if (!a || (!perm && a->m.nrows > 0) || nranges < 0 || !bounds) throw std::invalid_argument("null input");
    const tcb::index_t n = a->m.nrows;
    tcb::Permutation p;
    p.perm.assign(perm, perm + n);
    p.iperm.assign(static_cast<size_t>(n), -1);
    for (tcb::index_t i = 0; i < n; ++i) {
      const tcb::index_t q = p.perm[static_cast<size_t>(i)];
      if (q < 0 || q >= n || p.iperm[static_cast<size_t>(q)] >= 0)
        throw std::invalid_argument("permutation: not a bijection");
      p.iperm[static_cast<size_t>(q)] = i;
    }
    tcb::RangeList rl;
    for (int32_t k = 0; k < nranges; ++k) rl.ranges.push_back({bounds[k], bounds[k + 1]});
    tcb::validate_ranges(rl, n);
    auto out = std::make_unique<tch_analysis>();
    out->an = tcb::analyze_with_ordering(a->m, std::move(p), std::move(rl), level, threads);
    out->bounds.assign(bounds, bounds + nranges + 1);
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

void tch_analysis_free(tch_analysis* an) { delete an; }
const char* tch_error(void) { return g_tch_error.c_str(); }

void tch_analysis_perm(const tch_analysis* an, const int32_t** perm, const int32_t** iperm) {
  if (!an) return;
  if (perm) *perm = an->an.perm.perm.data();
  if (iperm) *iperm = an->an.perm.iperm.data();
}

int32_t tch_analysis_subtrees(const tch_analysis* an, int32_t depth, int32_t cap, int32_t* lo, int32_t* hi) {
  if (!an || depth < 0 || depth > 20) return -1;
  const tcb::NdTree& T = an->an.tree;
  if (T.root < 0) return 0;
  std::vector<tcb::index_t> level{T.root};
  for (int32_t d = 0; d < depth; ++d) {  // a leaf above `depth` stands for itself
    std::vector<tcb::index_t> next;
    for (tcb::index_t id : level) {
      const auto& ch = T.nodes[id].children;
      if (ch.empty()) next.push_back(id);
      else next.insert(next.end(), ch.begin(), ch.end());
    }
    level.swap(next);
  }
  for (size_t i = 0; i < level.size() && static_cast<int32_t>(i) < cap; ++i) {
    if (lo) lo[i] = T.span_begin(level[i]);
    if (hi) hi[i] = T.span_end(level[i]);
  }
  return static_cast<int32_t>(level.size());
}

int32_t tch_analysis_ranges(const tch_analysis* an, const int32_t** bounds) {
  if (!an) return -1;
  if (bounds) *bounds = an->bounds.data();
  return an->an.ranges.count();
}

void tch_analysis_permuted(const tch_analysis* an, tcg_csr_view* out) {
  if (an && out) view_of(an->an.a_permuted, out);
}
void tch_analysis_pattern(const tch_analysis* an, tcg_csr_view* out) {
  if (an && out) view_of(an->an.pattern.pattern, out);
}
void tch_analysis_times(const tch_analysis* an, double* ordering_s, double* symbolic_s) {
  if (!an) return;
  if (ordering_s) *ordering_s = an->an.ordering_seconds;
  if (symbolic_s) *symbolic_s = an->an.symbolic_seconds;
}

tch_matrix* tch_levelk_pattern(const tch_matrix* a, int32_t level, int32_t threads) {
  try {
    if (!a) throw std::invalid_argument("null matrix");
    auto out = std::make_unique<tch_matrix>();
    out->m = tcb::levelk_pattern(a->m, level, threads).pattern;
    return out.release();
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return nullptr;
  }
}

tcg_status tch_init_values(const tcg_csr_view* a_permuted, const tcg_csr_view* pattern, double* out) {
  try {
    const tcb::CsrMatrix a = csr_from_view(a_permuted, true);
    const tcb::CsrMatrix u = csr_from_view(pattern, false);
    const std::vector<double> v = tcb::init_factor_values(a, u);
    std::copy(v.begin(), v.end(), out);
    return TCG_OK;
  } catch (const std::exception& e) {
    g_tch_error = e.what();
    return TCG_INVALID;
  }
}

}  // extern "C"

// Internal accessor for the other C-ABI units (solve_capi.cpp): the device,
// stream and factor values of a context, without touching its state.
namespace tcb_internal {
bool ctx_factor(tcg_ctx* c, int member, int* device, cudaStream_t* stream, const double** vals,
                std::int64_t* n, std::int64_t* nnz) {
  if (!c || !c->uploaded || member < 0 || member >= c->nbatch) return false;
  *device = c->device;
  *stream = c->stream;
  *vals = c->nbatch == 1 ? c->vals : c->bvals + static_cast<std::int64_t>(member) * c->nnz;
  *n = c->n;
  *nnz = c->nnz;
  return true;
}
}  // namespace tcb_internal
