// Device-side types shared by the persistent IC(k) factorization kernel and
// its host launcher.
#pragma once

#include <cstdint>

namespace tcbdev {

constexpr int kChol = 0, kTrsm = 1, kHerk = 2, kGemm = 3;
// Queue entries with this bit set are helper tickets of a multi-CTA task.
constexpr int kHelperBit = 0x40000000;
// Row successor entries with this bit set go to the priority queue (plan.hpp kRowHot).
constexpr int kRowHotBit = 0x40000000;
// Task records are three int4 (plan.hpp kTaskWords = 12).
constexpr int kTaskInt4 = 3;

// Scheduler / status words, one per factorization (reset before each run).
// Every word that is polled or updated by many warps sits on its own
// 128-byte line: idle pollers of one counter must not slow down the
// atomics on another.
struct alignas(128) Line {
  int v;
  int pad[31];
};
struct Ctrl {
  Line q_head;       // next ticket handed to a polling CTA / warp
  Line q_tail;       // next free ready-queue slot
  Line hi_head;      // row mode: priority queue tickets
  Line hi_tail;
  Line done;         // tasks (rows) completed
  Line failed;       // breakdown latch (reference factorize.hpp:146-167), plus error below
  Line error;        // 1 = watchdog expired
  Line executed;     // task (row) bodies actually run (skipped after a breakdown)
  Line helpers_run;  // helper tickets that joined a multi-CTA task
  int fail_row;
  int fail_member;   // mode 5 batch: member of the first breakdown
  double fail_pivot;
  // trace mode, row kernel: per-phase SM cycles summed over warps
  // {pop wait, row body, publish fence, release, rows, pops, pushes, 0}
  unsigned long long prof[8];
};

struct Params {
  const int4* tasks;   // 3 x int4 per task
  const int4* items;   // 2 x int4 per item (kItemWords)
  const int4* srcs;    // 1 x int4 per source (kSrcWords)
  const int4* succ;    // 4 x int4 per edge: {successor, 0, 0, 0} + its task record
  const int* cols;
  double* vals;
  int* indeg;
  int* queue;
  int* claim;          // per task: next item of a multi-CTA task
  int* fin;            // per task: items finished of a multi-CTA task
  int* iflag;          // per item: epoch stamp when the row is final (multi-CTA Chol/Trsm)
  Ctrl* ctrl;
  unsigned long long* trace;  // optional: {start, end} globaltimer per task
  unsigned long long* itrace; // optional: {claimed, sources ready, merged, published} per item
  int ntasks;
  int qcap;            // ready-queue capacity (tasks + helper tickets)
  int cap;             // per-warp staging capacity (target row entries), multiple of 4
  int flag_words;      // 32-bit words of the per-CTA row-done bitmask, multiple of 4
  int icap;            // items staged in shared memory per single-CTA task
  int scap;            // sources staged in shared memory per single-CTA task
  int epoch;           // factorization counter (iflag stamps)
  int mode;            // 1 = device merge of sorted indices, 2 = update programs
  const int4* slot_rec;  // update programs (mode 2): {u_b, u_e, m0, o0} per target slot
  const int2* upd;
  unsigned long long timeout_ns;
};


// Value-flow schedule (mode 5, flow_kernel.cu): the finalising rows only,
// readers polling the values they gather until they are no longer kUnset.
// kUnset is a signalling NaN: arithmetic never produces one.
constexpr unsigned long long kUnset = 0x7FF40000DEADBEEFull;

struct FlowParams {
  const int4* rec;       // per position {tb, L | kind << 30, dpos, t} (plan.hpp kFlowWords)
  const int* item;       // per position: its item (trace only)
  const int4* slot;      // per coordinate of U: {u_b, u_e, m0, o0}
  const int2* upd;       // (m, o) pairs
  const int* ub;         // per coordinate of U: its first product in upd (nnz + 1; product-parallel rows)
  const double* a;       // input values (snapshot taken by the prelude), nbatch x nnz
  double* vals;          // output; kUnset until the owning row writes it; nbatch x nnz
  Ctrl* ctrl;
  unsigned long long* trace;  // optional: {start, end} per item (member 0)
  int* m_failed;         // per member: breakdown latch, row, pivot
  int* m_row;
  double* m_pivot;
  long long nnz;         // values per member
  long long nupd;        // (m, o) pairs in upd (bounds checks)
  int nrows;             // schedule rows (per member)
  int nbatch;            // members sharing the pattern
  double* const* peers;  // sharded (C6): every part's U, indexed by part; operands of other parts
  int npeers;            //   arrive as kRemoteBit | part << 25 | position (flow_plan.hpp build_flow_part)
  unsigned long long timeout_ns;
  // drain (end to end, factor_flow_pipe DRAIN = 1): CTAs [row_ctas, grid) copy
  // final values to the host while the rows run
  double* drain_out;     // device-accessible pinned host buffer (nnz values)
  unsigned* drain_done;  // per batch of 32 groups of 64 values: groups copied (zeroed per launch)
  int row_ctas;          // CTAs that run rows
  int decouple;          // per-lane kernel: Chol pivot through shared memory (lanes publish independently)
  // chunked download (end to end, DRAIN = 2): U in nchunks position ranges cut at unit starts (a unit at
  // tb lies in chunk tb * nchunks / nnz); the unit that completes a chunk tells the host, whose copy
  // engine then takes the chunk to the host while the rest of the rows run
  int* chunk_left;       // per chunk: units still to run (reset per launch)
  int* chunk_flag;       // per chunk, host-mapped: chunk_seq once the chunk is final
  int nchunks;
  int chunk_seq;
};

// Device-built update programs (flow_program.cu): U's pattern and its
// transposed index in, the value-flow slot records and (m, o) pairs out.
struct ProgParams {
  int n;
  const int* row_ptr;   // n + 1 positions
  const int* cols;      // U column indices
  const int* col_ptr;   // n + 1: sources of row t
  const int* col_src;   //   source row r, ascending
  const int* col_pos;   //   position of U(r, t)
  int* count;           // pass 1 out: products per coordinate
  const int* ub;        // pass 2 in: first product of each coordinate
  int4* slot;           // pass 2 out: {u_b, u_e, m0, o0} per coordinate
  int2* upd;            // pass 2 out: (m, o) pairs
  int* next_row;        // two work counters (zeroed before pass 1)
};


// The value-flow schedule built on the device (flow_schedule.cu).
struct SchedParams {
  int n;
  int slack_pct;     // placement between a unit's earliest and latest level, in percent (flow_order_keys)
  long long nnz;     // entries of U (the grid of the frontier kernel is sized by the mean row length)
  int nunits;
  const int* row_ptr;   // n + 1
  const int* cols;
  const int* col_ptr;   // transposed index: sources of row t
  const int* col_src;   //   their rows
  const int* col_pos;   //   positions of U(r, t)
  const int* ufirst;    // n + 1
  const int* u_tb;
  const int* u_len;
  int* uc0;             // per unit: first and last column (scratch, filled by flow_schedule)
  int* uc1;
  int* level;           // 0 until known
  int* height;
  int* acc;             // per unit: largest dependence level seen (rows of more than 8 units; zeroed)
  int* acc2;            // per unit: largest dependent height seen (the same)
  int* depth;           // out: largest level
  int* error;           // watchdog
  unsigned long long timeout_ns;
};

struct FlowPrepParams {
  const double* vals;    // working values (input of the factorization)
  double* a;             // snapshot of them; == vals: no copy (the input already lives in `a`)
  double* out;           // = vals in place: set to kUnset
  long long nnz;         // all members
  int* m_failed;         // reset per member
  int* m_row;
  double* m_pivot;
  int nbatch;

  Ctrl* ctrl;
};

struct PrepParams {
  const int* indeg0;
  const int* roots;
  int* indeg;
  int* queue;
  int* claim;
  int* fin;
  int* queue2;     // optional second queue (row mode priority queue), set to -1
  Ctrl* ctrl;
  int ntasks;
  int qcap;
  int nroots;
};

}  // namespace tcbdev
