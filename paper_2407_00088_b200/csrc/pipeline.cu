// Op-list executors over per-op launches (pipeline.py): the planner that
// gives each op its launch flags (PDL waits, INDEPENDENT launches, grouped
// table builds and lookups, fused table ops) and the stream-ordered
// launchers -- programmatic dependent launch (bitlut_pipeline_launch_ops) or
// per-launch completion counters (bitlut_pipeline_launch_ops_counted).
// Per-op arithmetic is the per-call kernels', so results are bitwise
// identical to bitlut_build_lut + bitlut_mpgemm.
#include "gemv_core.cuh"
#include "lut_core.cuh"

#include <cstdlib>

using namespace blk;

// ---------------------------------------------------------------------------
// Per-op executor: the same op list as stream-ordered launches of the
// per-call kernels (bitlut_build_lut / bitlut_mpgemm / bitlut_mpgemv_fused),
// chained with programmatic dependent launch; meant to be captured once into
// a CUDA graph (pipeline.py) so a replay costs one graph launch.
//
// Table-build fusion (opt-in: BITLUT_FLAG_FUSED_TABLES on the table op): a
// batch-1 fp16 table op whose every consumer is a fast-epilogue lookup on a
// 32-stream tile is not launched; each consumer
// runs as bitlut_mpgemv_fused from the table op's activations instead (one
// launch per GEMV, tables built in-kernel by the CTA cluster).  A fused
// lookup's inputs are the table op's inputs, so its dependencies are the
// table op's.
//
// Which lookups may skip the start-of-kernel wait (BITLUT_FLAG_INDEPENDENT)
// follows from when each kernel releases its successor:
//   * a table build triggers first, then waits              -> releases early
//   * an INDEPENDENT lookup triggers first, waits at exit   -> releases early
//   * a dependent lookup waits for its predecessor, then triggers.
// So when kernel i starts, every op before the most recent dependent lookup
// d < i (ops 0..d-1) has completed -- waits are transitive, since every
// kernel waits for its predecessor before exiting.  Lookup i runs
// INDEPENDENT iff all its (effective) deps are in that completed prefix (q
// after its table build waits; k and v, which read the same inputs, do
// not); the same holds for table builds (which never advance the prefix:
// they release before waiting).  Inputs made before the op list count as
// complete once any kernel of the list has waited.
// ---------------------------------------------------------------------------
bool bl_gemv_b1_fused_fits(const bl::LayoutV2& L, bool zeros, int scale_dtype);   // gemv_b1.cu

static bool fusable_lookup(const bitlut_pipe_op& s, const bitlut_pipe_op& t) {
  if (s.type != BITLUT_OP_LOOKUP || t.type != BITLUT_OP_TABLES) return false;
  if (!(s.flags & BITLUT_FLAG_FAST_EPILOGUE) || s.n != 1 || t.n != 1 || t.a_dtype != BITLUT_DT_F16) return false;
  if (s.flags & BITLUT_FLAG_LAYER_SET) return false;    // the fused kernel reads layout v2
  if (s.k != t.k || s.group_size != t.group_size) return false;
  bl::LayoutV2 L;
  if (bl::make_layout(s.m, s.k, s.bits, s.group_size, &L) || L.n_sg != 1) return false;
  return bl_gemv_b1_fused_fits(L, s.zeros != nullptr, s.scale_dtype);
}

static bool groupable_tables(const bitlut_pipe_op& a, const bitlut_pipe_op& b) {
  return a.type == BITLUT_OP_TABLES && b.type == BITLUT_OP_TABLES && a.a_dtype == b.a_dtype;
}

// Lookups that read the same table op (single dep) and can share one batch-1
// launch (bitlut_mpgemv_multi): q/k/v, gate/up.
bool bl_mixed_tables_ok(const bl::LayoutV2& L);   // gemv_b1.cu

// Two lookups can share a launch when they read the same tables (any
// epilogue), or -- fast epilogue, lean-kernel shapes -- different tables
// (bitlut_mpgemv_multi_tab: one launch for e.g. q,k,v,o,gate,up of a layer).
static bool groupable_lookups(const bitlut_pipe_op& a, const bitlut_pipe_op& b, const bitlut_pipe_op* specs) {
  if (a.type != BITLUT_OP_LOOKUP || b.type != BITLUT_OP_LOOKUP) return false;
  if (a.dep[0] < 0 || a.dep[1] >= 0 || a.dep[2] >= 0 || b.dep[0] < 0 || b.dep[1] >= 0 || b.dep[2] >= 0)
    return false;
  if (specs[b.dep[0]].type != BITLUT_OP_TABLES) return false;
  if (b.dep[0] != a.dep[0]) {
    if (!(a.flags & BITLUT_FLAG_FAST_EPILOGUE) || !(b.flags & BITLUT_FLAG_FAST_EPILOGUE)) return false;
    bl::LayoutV2 La;
    if (bl::make_layout(a.m, a.k, a.bits, a.group_size, &La) || !bl_mixed_tables_ok(La)) return false;
    if (specs[a.dep[0]].n != 1 || specs[b.dep[0]].n != 1) return false;
  }
  if ((a.flags & BITLUT_FLAG_FAST_EPILOGUE) != (b.flags & BITLUT_FLAG_FAST_EPILOGUE)) return false;
  if ((a.flags & BITLUT_FLAG_LAYER_SET) != (b.flags & BITLUT_FLAG_LAYER_SET)) return false;
  if (a.n != 1 || b.n != 1 || a.k != b.k || a.bits != b.bits || a.group_size != b.group_size) return false;
  if (a.scale_dtype != b.scale_dtype || (a.zeros != nullptr) != (b.zeros != nullptr)) return false;
  if (specs[a.dep[0]].type != BITLUT_OP_TABLES) return false;
  bl::LayoutV2 L;
  if (bl::make_layout(a.m, a.k, a.bits, a.group_size, &L) || L.n_sg != 1) return false;
  if (bl::make_layout(b.m, b.k, b.bits, b.group_size, &L) || L.n_sg != 1) return false;
  return true;
}

static bool grouping_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BITLUT_PLAN_NOGROUP");      // diagnostic: 1 disables launch grouping
    on = (e && atoi(e)) ? 0 : 1;
  }
  return on != 0;
}

constexpr int kMaxGroupTables = 8, kMaxGroupLookups = 8;

extern "C" int bitlut_pipeline_plan_flags(const bitlut_pipe_op* specs, int n_ops, int* flags_out) {
  if (n_ops <= 0 || !specs || !flags_out) return BITLUT_EPARAM;
  for (int i = 0; i < n_ops; i++) {
    if (specs[i].type != BITLUT_OP_TABLES && specs[i].type != BITLUT_OP_LOOKUP) return BITLUT_EPARAM;
    for (int d = 0; d < 3; d++)
      if (specs[i].dep[d] >= i || specs[i].dep[d] < -1) return BITLUT_EPARAM;
    flags_out[i] = 0;
  }
  // 1. which table ops can be folded into all of their consumers
  for (int t = 0; t < n_ops; t++) {
    if (specs[t].type != BITLUT_OP_TABLES || !(specs[t].flags & BITLUT_FLAG_FUSED_TABLES)) continue;
    bool all = true, any = false;
    for (int i = t + 1; i < n_ops && all; i++) {
      const bitlut_pipe_op& s = specs[i];
      bool uses = false;
      for (int d = 0; d < 3; d++) uses = uses || s.dep[d] == t;
      if (!uses) continue;
      any = true;
      // a fused consumer must depend on the table op alone
      const bool only = s.dep[0] == t && s.dep[1] < 0 && s.dep[2] < 0;
      all = only && fusable_lookup(s, specs[t]);
    }
    if (any && all) {
      flags_out[t] = BITLUT_PLAN_SKIP;
      for (int i = t + 1; i < n_ops; i++)
        if (specs[i].dep[0] == t) flags_out[i] = BITLUT_FLAG_FUSED_TABLES;
    }
  }
  // 2. launch groups: consecutive table builds; consecutive lookups over the same tables
  if (grouping_enabled()) {
    int lead = -1, size = 0;
    for (int i = 0; i < n_ops; i++) {
      if (flags_out[i] == BITLUT_PLAN_SKIP) continue;
      const bool plain = !(flags_out[i] & BITLUT_FLAG_FUSED_TABLES);
      bool join = false;
      if (lead >= 0 && plain && !(flags_out[lead] & BITLUT_FLAG_FUSED_TABLES)) {
        if (groupable_tables(specs[lead], specs[i])) join = size < kMaxGroupTables;
        else if (groupable_lookups(specs[lead], specs[i], specs)) join = size < kMaxGroupLookups;
      }
      if (join) {
        flags_out[i] |= BITLUT_PLAN_JOINED;
        size++;
      } else {
        lead = i;
        size = 1;
      }
    }
  }
  // 3. launch flags per launch unit (a group runs as one kernel)
  int done_below = 0;            // ops [0, done_below) complete when the next kernel starts
  for (int i = 0; i < n_ops;) {
    if (flags_out[i] == BITLUT_PLAN_SKIP) { i++; continue; }
    int j = i + 1;
    while (j < n_ops && flags_out[j] != BITLUT_PLAN_SKIP && (flags_out[j] & BITLUT_PLAN_JOINED)) j++;
    // inputs from before the op list are complete once any kernel of the
    // list has waited (done_below >= 1)
    bool ok = done_below >= 1;
    for (int u = i; u < j; u++) {
      const bitlut_pipe_op& s = specs[u];
      const int* deps = (flags_out[u] & BITLUT_FLAG_FUSED_TABLES) ? specs[s.dep[0]].dep : s.dep;
      for (int d = 0; d < 3; d++)
        if (deps[d] >= 0) ok = ok && deps[d] < done_below;
    }
    const bool lookup = specs[i].type == BITLUT_OP_LOOKUP;
    for (int u = i; u < j; u++) {
      int fl = BITLUT_FLAG_PDL | flags_out[u];
      if (ok) fl |= BITLUT_FLAG_INDEPENDENT;
      if (lookup) fl |= specs[u].flags & (BITLUT_FLAG_FAST_EPILOGUE | BITLUT_FLAG_LAYER_SET);
      flags_out[u] = fl;
    }
    if (lookup && !ok) done_below = i;   // waits for its predecessor (hence all earlier), then releases
    i = j;
  }
  return BITLUT_OK;
}

extern "C" int bitlut_pipeline_launch_ops(const bitlut_pipe_op* specs, int n_ops, void* stream) {
  if (n_ops <= 0 || !specs) return BITLUT_EPARAM;
  int stack_flags[256];
  int* flags = n_ops <= 256 ? stack_flags : static_cast<int*>(malloc(sizeof(int) * n_ops));
  if (!flags) return BITLUT_EINTERNAL;
  int rc = bitlut_pipeline_plan_flags(specs, n_ops, flags);
  for (int i = 0; rc == BITLUT_OK && i < n_ops;) {
    const bitlut_pipe_op& s = specs[i];
    const int fl = flags[i];
    if (fl == BITLUT_PLAN_SKIP) { i++; continue; }
    int j = i + 1;
    while (j < n_ops && flags[j] != BITLUT_PLAN_SKIP && (flags[j] & BITLUT_PLAN_JOINED)) j++;
    const int lf = fl & (BITLUT_FLAG_PDL | BITLUT_FLAG_INDEPENDENT | BITLUT_FLAG_FAST_EPILOGUE |
                         (s.type == BITLUT_OP_LOOKUP ? BITLUT_FLAG_LAYER_SET : 0));
    if (s.type == BITLUT_OP_TABLES) {
      if (j - i == 1) {
        rc = bitlut_build_lut(s.a, s.a_dtype, s.n, s.k, s.group_size, BITLUT_TABLE_Q8, s.tables,
                              s.tscales, s.rowsums, lf, stream);
      } else {
        bitlut_lut_job jobs[kMaxGroupTables];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          jobs[u - i] = {t.a, t.a_dtype, t.n, t.k, t.group_size, t.tables, t.tscales, t.rowsums};
        }
        rc = bitlut_build_lut_multi(jobs, j - i, BITLUT_TABLE_Q8, lf, stream);
      }
    } else if (fl & BITLUT_FLAG_FUSED_TABLES) {
      const bitlut_pipe_op& t = specs[s.dep[0]];
      rc = bitlut_mpgemv_fused(t.a, t.a_dtype, s.wgpu, s.m, s.k, s.bits, s.group_size, s.wscales, s.zeros,
                               s.scale_dtype, s.out, lf, stream);
    } else if (j - i == 1) {
      rc = bitlut_mpgemm(s.wgpu, s.m, s.k, s.bits, s.group_size, s.wscales, s.zeros, s.scale_dtype,
                         s.tables, s.tscales, s.rowsums, BITLUT_TABLE_Q8, s.n, s.out, nullptr, lf, stream);
    } else {
      bool same = true;
      for (int u = i + 1; u < j; u++) same = same && specs[u].dep[0] == s.dep[0];
      if (same) {
        bitlut_mat mats[kMaxGroupLookups];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          mats[u - i] = {t.wgpu, t.wscales, t.zeros, t.m, t.out};
        }
        rc = bitlut_mpgemv_multi(mats, j - i, s.k, s.bits, s.group_size, s.scale_dtype, s.tables, s.tscales,
                                 s.rowsums, lf, stream);
      } else {
        bitlut_mat_tab mats[kMaxGroupLookups];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          mats[u - i] = {t.wgpu, t.wscales, t.zeros, t.m, t.out, t.tables, t.tscales, t.rowsums};
        }
        rc = bitlut_mpgemv_multi_tab(mats, j - i, s.k, s.bits, s.group_size, s.scale_dtype, lf, stream);
        if (rc == BITLUT_ELAYOUT) {                     // shape outside the lean kernel: one launch each
          rc = BITLUT_OK;
          for (int u = i; rc == BITLUT_OK && u < j; u++) {
            const bitlut_pipe_op& t = specs[u];
            rc = bitlut_mpgemm(t.wgpu, t.m, t.k, t.bits, t.group_size, t.wscales, t.zeros, t.scale_dtype,
                               t.tables, t.tscales, t.rowsums, BITLUT_TABLE_Q8, t.n, t.out, nullptr, lf, stream);
          }
        }
      }
    }
    i = j;
  }
  if (flags != stack_flags) free(flags);
  return rc;
}

// ---------------------------------------------------------------------------
// Counted variant: every launch unit starts without griddepcontrol.wait and
// instead waits (one thread, ld.acquire) on the completion counters of the
// units that produce its inputs; each CTA counts itself into its unit's
// counter after its last global write (common.cuh DepSync).  No kernel
// drains the stream: a consumer's CTAs are resident, with their weights
// already streaming in, when the producer finishes.  Counters are zeroed by
// a memset at the head of the list (ordered after all earlier stream work,
// which also makes inputs from before the list complete).  Counted kernels
// never wait for their stream predecessor; a final join kernel waits until
// every CTA of the list has counted itself, so the list's stream completion
// still means "all done".  At most 8 producer launches per launch (else
// EPARAM: use the PDL variant).  Bitwise identical to the plain launches.
// ---------------------------------------------------------------------------
int bl_build_lut_launch(const void* a, int a_dtype, int n, int k, int group_size, int mode, void* tables,
                        float* tscales, float* rowsums, cudaStream_t stream, bool pdl, bool independent,
                        const bl::DepSync& dep, int* grid_out);
int bl_build_lut_multi_launch(const bitlut_lut_job* jobs, int n_jobs, int mode, int flags, void* stream,
                              const bl::DepSync& dep, int* grid_out);
int bl_mpgemm_launch(const uint8_t* wgpu, int m, int k, int bits, int group_size, const void* wscales,
                     const void* zeros, int scale_dtype, const void* tables, const float* tscales,
                     const float* rowsums, int mode, int n, float* out, int32_t* partials, int flags,
                     unsigned long long* trace, void* stream, const bl::DepSync& dep, int* grid_out);
int bl_mpgemv_multi_tab_launch(const bitlut_mat_tab* mats, int n_mats, int k, int bits, int group_size,
                               int scale_dtype, int flags, void* stream, const bl::DepSync& dep, int* grid_out);
int bl_mpgemv_multi_launch(const bitlut_mat* mats, int n_mats, int k, int bits, int group_size,
                           int scale_dtype, const void* tables, const float* tscales, const float* rowsums,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out);
int bl_mpgemv_fused_launch(const void* a, int a_dtype, const uint8_t* wgpu, int m, int k, int bits,
                           int group_size, const void* wscales, const void* zeros, int scale_dtype, float* out,
                           int flags, void* stream, const bl::DepSync& dep, int* grid_out);

constexpr int kMaxJoinUnits = 1024;
struct JoinArgs {
  const unsigned* counters;
  int n_units;
  unsigned unit[kMaxJoinUnits];     // counter index of each launch unit
  unsigned target[kMaxJoinUnits];   // its CTA count
};

// The list's last launch: completes once every launch unit has counted all
// of its CTAs (one lane per unit, strided).
__global__ void join_kernel(const __grid_constant__ JoinArgs J) {
  for (int i = threadIdx.x; i < J.n_units; i += blockDim.x)
    while (bl::ld_acquire_u32(J.counters + J.unit[i]) < J.target[i]) __nanosleep(64);
}

extern "C" int bitlut_pipeline_launch_ops_counted(const bitlut_pipe_op* specs, int n_ops, unsigned* counters,
                                                  void* stream) {
  if (n_ops <= 0 || !specs || !counters) return BITLUT_EPARAM;
  int* flags = static_cast<int*>(malloc(sizeof(int) * n_ops * 3));
  if (!flags) return BITLUT_EINTERNAL;
  int* leader = flags + n_ops;        // launch unit (leader op index) of each op, -1 for skipped
  int* grid = flags + 2 * n_ops;      // CTAs of each unit (at its leader)
  int rc = bitlut_pipeline_plan_flags(specs, n_ops, flags);
  if (rc == BITLUT_OK &&
      cudaMemsetAsync(counters, 0, sizeof(unsigned) * (n_ops + 1), (cudaStream_t)stream) != cudaSuccess)
    rc = BITLUT_EINTERNAL;
  JoinArgs* join = static_cast<JoinArgs*>(malloc(sizeof(JoinArgs)));
  if (!join) rc = BITLUT_EINTERNAL;
  else { join->counters = counters; join->n_units = 0; }
  for (int i = 0; i < n_ops; i++) { leader[i] = -1; grid[i] = 0; }
  for (int i = 0; rc == BITLUT_OK && i < n_ops;) {
    const bitlut_pipe_op& s = specs[i];
    const int fl = flags[i];
    if (fl == BITLUT_PLAN_SKIP) { i++; continue; }
    int j = i + 1;
    while (j < n_ops && flags[j] != BITLUT_PLAN_SKIP && (flags[j] & BITLUT_PLAN_JOINED)) j++;
    for (int u = i; u < j; u++) leader[u] = i;
    // producer units of every member's (effective) inputs
    bl::DepSync dep = {};
    bool overflow = false;
    for (int u = i; u < j; u++) {
      const bitlut_pipe_op& m = specs[u];
      const int* deps = (flags[u] & BITLUT_FLAG_FUSED_TABLES) ? specs[m.dep[0]].dep : m.dep;
      for (int d = 0; d < 3; d++) {
        if (deps[d] < 0) continue;
        const int pu = leader[deps[d]];
        if (pu < 0) { overflow = true; continue; }
        bool seen = false;
        for (int w = 0; w < dep.n_wait; w++) seen = seen || dep.wait_cnt[w] == counters + pu;
        if (seen) continue;
        if (dep.n_wait == bl::kMaxDepWaits) { overflow = true; continue; }
        dep.wait_cnt[dep.n_wait] = counters + pu;
        dep.wait_target[dep.n_wait] = (unsigned)grid[pu];
        dep.n_wait++;
      }
    }
    if (overflow) { rc = BITLUT_EPARAM; break; }   // > 8 producer launches: use sync="pdl"
    const int lf = BITLUT_FLAG_PDL | (fl & BITLUT_FLAG_FAST_EPILOGUE) |
                   (s.type == BITLUT_OP_LOOKUP ? (fl & BITLUT_FLAG_LAYER_SET) : 0);
    dep.counted = 1;
    dep.done = counters + i;
    dep.total = nullptr;
    int g = 0;
    if (s.type == BITLUT_OP_TABLES) {
      if (j - i == 1) {
        rc = bl_build_lut_launch(s.a, s.a_dtype, s.n, s.k, s.group_size, BITLUT_TABLE_Q8, s.tables, s.tscales,
                                 s.rowsums, (cudaStream_t)stream, true, false, dep, &g);
      } else {
        bitlut_lut_job jobs[kMaxGroupTables];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          jobs[u - i] = {t.a, t.a_dtype, t.n, t.k, t.group_size, t.tables, t.tscales, t.rowsums};
        }
        rc = bl_build_lut_multi_launch(jobs, j - i, BITLUT_TABLE_Q8, lf, stream, dep, &g);
      }
    } else if (fl & BITLUT_FLAG_FUSED_TABLES) {
      const bitlut_pipe_op& t = specs[s.dep[0]];
      rc = bl_mpgemv_fused_launch(t.a, t.a_dtype, s.wgpu, s.m, s.k, s.bits, s.group_size, s.wscales, s.zeros,
                                  s.scale_dtype, s.out, lf, stream, dep, &g);
    } else if (j - i == 1) {
      rc = bl_mpgemm_launch(s.wgpu, s.m, s.k, s.bits, s.group_size, s.wscales, s.zeros, s.scale_dtype, s.tables,
                            s.tscales, s.rowsums, BITLUT_TABLE_Q8, s.n, s.out, nullptr, lf, nullptr, stream, dep,
                            &g);
    } else {
      bool same = true;
      for (int u = i + 1; u < j; u++) same = same && specs[u].dep[0] == s.dep[0];
      if (same) {
        bitlut_mat mats[kMaxGroupLookups];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          mats[u - i] = {t.wgpu, t.wscales, t.zeros, t.m, t.out};
        }
        rc = bl_mpgemv_multi_launch(mats, j - i, s.k, s.bits, s.group_size, s.scale_dtype, s.tables, s.tscales,
                                    s.rowsums, lf, stream, dep, &g);
      } else {
        bitlut_mat_tab mats[kMaxGroupLookups];
        for (int u = i; u < j; u++) {
          const bitlut_pipe_op& t = specs[u];
          mats[u - i] = {t.wgpu, t.wscales, t.zeros, t.m, t.out, t.tables, t.tscales, t.rowsums};
        }
        rc = bl_mpgemv_multi_tab_launch(mats, j - i, s.k, s.bits, s.group_size, s.scale_dtype, lf, stream, dep,
                                        &g);
      }
    }
    grid[i] = g;
    if (rc == BITLUT_OK && g <= 0) rc = BITLUT_EINTERNAL;
    if (rc == BITLUT_OK) {
      if (join->n_units == kMaxJoinUnits) { rc = BITLUT_EPARAM; break; }
      join->unit[join->n_units] = (unsigned)i;
      join->target[join->n_units] = (unsigned)g;
      join->n_units++;
    }
    i = j;
  }
  if (rc == BITLUT_OK) {     // the list completes when its last CTA has counted itself
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, join_kernel, *join) != cudaSuccess) rc = BITLUT_EINTERNAL;
  }
  free(join);
  free(flags);
  return rc;
}
