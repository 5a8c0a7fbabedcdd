// Device-side types shared by the persistent IC(k) factorization kernel and
// its host launcher.
#pragma once

#include <cstdint>

namespace tcbdev {

constexpr int kChol = 0, kTrsm = 1, kHerk = 2, kGemm = 3;

// Scheduler / status words, one per factorization (reset before each run).
struct Ctrl {
  int q_head;        // next ticket handed to a polling CTA
  int q_tail;        // next free ready-queue slot
  int done;          // tasks completed (released)
  int failed;        // breakdown latch (reference factorize.hpp:146-167)
  int fail_row;
  int error;         // 1 = watchdog expired, 2 = staging/flag capacity exceeded
  int executed;      // task bodies actually run (skipped after a breakdown)
  int pad0;
  double fail_pivot;
  unsigned long long pad1;
};

struct Params {
  const int4* tasks;   // 2 x int4 per task (plan.hpp kTaskWords)
  const int4* items;   // 2 x int4 per item (kItemWords)
  const int4* srcs;    // 1 x int4 per source (kSrcWords)
  const int* succ;
  const int* cols;
  double* vals;
  int* indeg;
  int* queue;
  Ctrl* ctrl;
  unsigned long long* trace;  // optional: {start, end} globaltimer per task
  int ntasks;
  int cap;             // per-warp staging capacity (target row entries)
  int flag_words;      // 32-bit words of the per-CTA row-done bitmask
  unsigned long long timeout_ns;
};

struct PrepParams {
  const int* indeg0;
  const int* roots;
  int* indeg;
  int* queue;
  Ctrl* ctrl;
  int ntasks;
  int nroots;
};

}  // namespace tcbdev
