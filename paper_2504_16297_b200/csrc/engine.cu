// engine.cu -- libptsbe.so: the C ABI (include/ptsbe.h) over the sm_100a kernels.
//
// Host orchestration only: device buffers, program upload, pass launches,
// sampler pipeline.  No torch, no Python; the Python package binds this with
// ctypes (paper_2504_16297_b200/_native.py), which releases the GIL per call.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: no-ops unless a profiler injects itself

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ptsbe.h"
#include "pass_kernels.cuh"
#include "sample_kernels.cuh"
#include "codegen.h"
#include "planner.h"
#include "records.h"
#include "conventional.cuh"
#include "exact_cdf.cuh"
#include "shard.cuh"
#include "nccl_api.h"

using namespace ptsbe;

namespace {
// RAII NVTX range (nsys / ncu --nvtx show the engine's phases: passes, sampling, swaps)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct PassHost {
  uint64_t qmask;
  int L, c;
  int gb = 4;                      // register bits per phase of this pass (generated kernels: 4 or 5)
  int op_begin, n_ops;
  int slot_begin, n_slots;
  int phase_begin, n_phases;
};

struct ptsbe_engine {
  int dev = 0, n = 0, dtype = 0, cap = 0, num_sms = 148;
  size_t amp_bytes = 8;
  cudaStream_t stream = nullptr;
  void* states = nullptr;
  // per-batch
  uint8_t* d_sel = nullptr;
  double* d_weight = nullptr;
  double* d_nst = nullptr;
  int32_t* d_status = nullptr;
  int32_t* d_fail = nullptr;
  int last_B = 0;
  bool final_general = false;   // stored states carry norm^2 = nst (not yet rescaled)
  // program
  bool loaded = false;
  int n_sites = 0, n_mats = 0;
  std::vector<PassHost> passes;
  DevOp* d_ops = nullptr;
  DevPhase* d_phases = nullptr;
  int32_t* d_matkind = nullptr;
  int n_phases_total = 0;
  int phase_bits = 4;              // phase register bits requested: 4, 5, or 0 = per pass (PassHost::gb)
  // circuit-specialised kernels (codegen.h); generic pass_kernel when off
  bool gen_active = false;
  std::string gen_note;
  gen::Module gen_mod;
  void* d_mats = nullptr;
  DevChan* d_chans = nullptr;
  int32_t* d_site_chan = nullptr;
  int32_t* d_slot_site = nullptr;
  double* d_partials = nullptr;
  size_t partial_cap = 0;
  // sampler scratch
  int sbits = 0;
  long long nblk = 0;
  uint64_t* d_bs = nullptr;
  uint64_t* d_total = nullptr;
  int64_t* d_off = nullptr;
  int64_t* d_m = nullptr;
  int64_t* d_nuniq = nullptr;
  int64_t* d_uoff = nullptr;
  uint64_t* d_rng = nullptr;
  size_t shot_cap = 0;
  uint64_t* d_keys = nullptr;
  uint64_t* d_tmp = nullptr;
  uint64_t* d_idx = nullptr;
  uint64_t* d_runidx = nullptr;
  uint32_t* d_runcnt = nullptr;
  size_t chunk_cap = 0;
  uint64_t* d_chunks = nullptr;
  long long launches = 0;
  // shared-trunk schedule (launch_passes): host copy of the batch's outcome table,
  // pass index of every site, per-pass launch entries and fork lists
  bool tree_enabled = true;
  std::vector<uint8_t> host_sel;
  std::vector<int> site_pass;
  long long last_entries = 0;
  int4* d_ent = nullptr;
  size_t ent_cap = 0;
  int32_t* d_forks = nullptr;
  size_t fork_cap = 0;
  double pass_bytes_total = 0.0;   // algorithmic bytes of profiled pass launches
  // physical layout: logical qubit q stored at physical bit perm[q] (identity unless permuted)
  bool permuted = false;
  bool zero_vector = false;   // current run starts from the all-zero vector (non-zero shards)
  BitPerm layout{};
  std::vector<uint8_t> logical;   // per state: 1 = stored in logical order (canonicalised)
  // optional per-launch timing of the pass kernels (CUDA events on h->stream)
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;
  double pass_ms_total = 0.0;
  long long pass_launches = 0;
  std::vector<int> ev_pass;               // pass index of each profiled launch (event pair)
  std::vector<double> ev_bytes;           // its algorithmic bytes
  std::vector<double> per_pass_ms, per_pass_bytes;
  // PTSBE_LAUNCH_LOG=path: every pass launch's (pass, launch entries, algorithmic bytes),
  // appended to the file when the handle is destroyed -- matched line by line against an
  // ncu capture of the same process to turn DRAM counters into a traffic / algorithmic ratio
  std::vector<double> launch_log;
  // host-only handle (ptsbe_create_host): load_program plans and generates the
  // pass kernels' source without touching a device (offline SASS inspection)
  bool host_only = false;
  // fused sampler block sums: the last generated pass of a unitary program writes
  // d_bs in TILE order of its geometry (gen_prelude.cuh run_pass); valid until the
  // states change by other means
  bool any_general = false;
  bool tsum_ok = false;
  uint64_t tsum_qmask = 0;
  int tsum_L = 0, tsum_c = 0, tsum_threads = 0;
  std::string gen_src;
  // TMA tile staging: one 2-D tensor map over every state slot, as rows of 128 B
  // (16 x 8-B words); the generated pass kernels gather / scatter a tile's rows with it
  alignas(64) CUtensorMap tmap;
  bool tmap_ok = false;
  // conventional (Algorithm 1) selection: per pass, the general-channel site that
  // opens it (outcome chosen on device from the state at the pass boundary)
  struct Decision { int site = -1, p0 = -1, p1 = -1, arity = 0, mat_base = 0, n_out = 0; };
  std::vector<Decision> decide;
  bool conv_ready = false;        // every general site opens its pass
  double* d_mats64 = nullptr;     // operator table in fp64 (branch probabilities)
  double* d_u = nullptr;          // per (trajectory, site) uniforms
  size_t u_cap = 0;
  double* d_rdm = nullptr;        // reduced-density-matrix partials
  size_t rdm_cap = 0;
  BlockMap* d_maps = nullptr;     // exact-CDF block maps (verification-mode sampling)
  size_t maps_cap = 0;
  // state sharding (shard.cuh): NCCL communicator of the shard group, exchange buffers,
  // cross-shard Kraus norms
  ncclComm_t comm = nullptr;
  int shard_rank = 0, shard_nranks = 1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t xev[4] = {nullptr, nullptr, nullptr, nullptr};
  void* xbuf = nullptr;
  size_t xbuf_bytes = 0;
  double* d_slotsum = nullptr;    // per (slot, row) shard-local norm^2 of renormalising sites
  size_t slotsum_cap = 0;
  uint32_t run_flags = 0;         // flags of the current run_common call (launch_passes reads them)
  // PTSBE_HOST_MIRROR: host copies of the next device-pointer call's outcome table / shot
  // counts (scheduling only; the kernels read the device copies)
  const uint8_t* mirror_sel = nullptr;
  const int64_t* mirror_shots = nullptr;
  int mirror_B = 0;
  int pending_pass = -1;          // PTSBE_DEFER_NORMS: pass whose slot norms await the global sums
  int pending_ent = 0, pending_E = 0;
  void* scratch_state = nullptr;  // one state's worth of scratch for relayouts (allocated on first use)
  std::string err;
};

namespace {

int fail(ptsbe_engine* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  return code;
}

#define CK(h, expr)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail((h), PTSBE_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define CKL(h)                                                                          \
  do {                                                                                  \
    (h)->launches++;                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return fail((h), PTSBE_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
int dalloc(ptsbe_engine* h, T** p, size_t count) {
  if (*p) { cudaFree(*p); *p = nullptr; }
  if (count == 0) return 0;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(h, PTSBE_ERR_CUDA, "cudaMalloc(%zu bytes) failed: %s", count * sizeof(T), cudaGetErrorString(e));
  }
  return 0;
}

// Copy between a user pointer (host or device per flags) and device memory.
int copy_in(ptsbe_engine* h, void* dst_dev, const void* src, size_t bytes, uint32_t flags) {
  if (bytes == 0) return 0;
  CK(h, cudaMemcpyAsync(dst_dev, src, bytes,
                        (flags & PTSBE_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        h->stream));
  return 0;
}
int copy_out(ptsbe_engine* h, void* dst, const void* src_dev, size_t bytes, uint32_t flags) {
  if (bytes == 0) return 0;
  CK(h, cudaMemcpyAsync(dst, src_dev, bytes,
                        (flags & PTSBE_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        h->stream));
  return 0;
}

size_t pass_smem(const PassHost& P, size_t amp_bytes) {
  return pass_smem_bytes(P.L, P.c, amp_bytes, P.n_ops, P.n_phases);
}

template <typename R>
int launch_passes(ptsbe_engine* h, int B, bool from_zero, int p_begin = 0, int p_end = -1) {
  if (p_end < 0) p_end = (int)h->passes.size();
  // a continued range (sharded segments) inherits the deferred-rescale state
  bool prev_general = p_begin > 0 ? h->final_general : false;
  h->tsum_ok = false;
  if (h->passes.empty()) {
    if (from_zero) {
      init_zero_kernel<R><<<1184, 256, 0, h->stream>>>(h->states, h->n, B, h->zero_vector ? 1 : 0);
      CKL(h);
    }
    h->final_general = false;
    return 0;
  }
  // Launch entries per pass: the shared-prefix TREE schedule (fresh |0> batches).  Two
  // trajectories have identical states through pass k iff they take identical outcomes at
  // every site of passes <= k.  The batch is kept as groups of such trajectories; each
  // group's state lives in one member's slot (its owner) and is computed ONCE per pass.
  // When a group's members take different outcomes in pass k it splits: every new
  // subgroup reads the group's state from pass k-1 and writes its own owner's slot (the
  // first launch of the pass); the subgroup that keeps the old owner updates that slot in
  // place in a second launch, after everybody has read it.  Weight / norm / status rows are
  // inherited at the split (fork rows).  Groups still shared after the last pass (equal
  // outcome tables) are copied to their members.  Same kernels, same ops, same inputs:
  // bit-identical to evolving every trajectory from |0> separately
  // (test_shared_trunk_schedule_is_bit_identical); the noiseless trunk of round 1 is the
  // root of this tree.
  const int P = (int)h->passes.size();
  const bool tree = from_zero && p_begin == 0 && p_end == P && P >= 2 && h->tree_enabled && !h->host_sel.empty();
  h->tsum_ok = false;
  // (a 512-amplitude sampler block must be the amplitudes of a warp or a half warp of
  // the last pass's tile)
  const long long per_thread = P >= 1 ? (1ll << h->passes[P - 1].L) /
                                            gen::threads_for(h->passes[P - 1].L, h->passes[P - 1].gb, false) : 0;
  // and the pass's store loop must be the vectorised one (gen_prelude.cuh run_pass FAST)
  bool store_fast = false;
  int tsum_ce = 0;   // effective contiguous bits of the last pass's (sub-)rows (gen_prelude.cuh CE)
  if (P >= 1) {
    const PassHost& lp = h->passes[P - 1];
    const long long thr = gen::threads_for(lp.L, lp.gb, false);
    const int vpw = h->dtype == PTSBE_C64 ? 2 : 1;
    int tlog2 = 5;
    while ((1ll << (tlog2 + 1)) <= thr && tlog2 < 10) ++tlog2;
    const int cpr_log = std::min(lp.c - (vpw == 2 ? 1 : 0), tlog2);
    tsum_ce = cpr_log + (vpw == 2 ? 1 : 0);
    store_fast = cpr_log >= 0 && thr >= (1ll << cpr_log) && ((1ll << lp.L) / vpw) % thr == 0;
  }
  bool fuse_sums = h->gen_active && !h->any_general && from_zero && p_begin == 0 && p_end == P && P >= 1 &&
                   h->sbits == 9 && store_fast && (per_thread * 32 == 512 || per_thread * 16 == 512) &&
                   !std::getenv("PTSBE_NO_FUSED_SUMS");
  struct LaunchRec { int pass, ent_begin, E, fork_begin, nfork; };
  std::vector<int4> ents;
  std::vector<int32_t> forkpairs;               // (child row, parent row) pairs
  std::vector<LaunchRec> launches;
  std::vector<std::pair<int, int>> end_copies;  // (member, owner) of groups shared to the end
  if (!tree) {
    for (int k = p_begin; k < p_end; ++k) {
      launches.push_back(LaunchRec{k, (int)ents.size(), B, 0, 0});
      for (int b = 0; b < B; ++b) ents.push_back(make_int4(b, b, b, 0));
    }
  } else {
    // per (trajectory, pass): its non-default (site, outcome) pairs, ascending site
    std::vector<std::vector<std::pair<int, int>>> errs((size_t)B * P);
    for (int b = 0; b < B; ++b) {
      const uint8_t* row = h->host_sel.data() + (size_t)b * h->n_sites;
      for (int s = 0; s < h->n_sites; ++s)
        if (row[s] && h->site_pass[s] < P) errs[(size_t)b * P + h->site_pass[s]].push_back({s, (int)row[s]});
    }
    struct Group { int owner; std::vector<int> mem; };
    std::vector<Group> groups(1);
    groups[0].owner = 0;
    for (int b = 0; b < B; ++b) groups[0].mem.push_back(b);
    for (int k = 0; k < P; ++k) {
      std::vector<int4> inA, inB;
      std::vector<int32_t> fk;
      std::vector<Group> next;
      for (const Group& g : groups) {
        std::vector<Group> subs;
        std::vector<const std::vector<std::pair<int, int>>*> keys;
        for (int b : g.mem) {
          const auto* key = &errs[(size_t)b * P + k];
          size_t j = 0;
          while (j < keys.size() && *keys[j] != *key) ++j;
          if (j == keys.size()) { keys.push_back(key); subs.push_back(Group{b, {}}); }
          subs[j].mem.push_back(b);
        }
        if (subs.size() == 1) {                     // no split: in place
          inA.push_back(make_int4(g.owner, g.owner, g.owner, 0));
          next.push_back(Group{g.owner, subs[0].mem});
          continue;
        }
        for (Group& sg : subs) {
          if (std::find(sg.mem.begin(), sg.mem.end(), g.owner) != sg.mem.end()) {
            sg.owner = g.owner;                     // keeps the slot: updated after the others read it
            (k == 0 ? inA : inB).push_back(make_int4(g.owner, g.owner, g.owner, 0));
          } else {
            sg.owner = sg.mem[0];
            inA.push_back(make_int4(sg.owner, g.owner, sg.owner, 0));
            if (k > 0) { fk.push_back(sg.owner); fk.push_back(g.owner); }
          }
          next.push_back(sg);
        }
      }
      launches.push_back(LaunchRec{k, (int)ents.size(), (int)inA.size(), (int)forkpairs.size() / 2,
                                   (int)fk.size() / 2});
      ents.insert(ents.end(), inA.begin(), inA.end());
      forkpairs.insert(forkpairs.end(), fk.begin(), fk.end());
      if (!inB.empty()) {
        launches.push_back(LaunchRec{k, (int)ents.size(), (int)inB.size(), 0, 0});
        ents.insert(ents.end(), inB.begin(), inB.end());
      }
      groups.swap(next);
    }
    for (const Group& g : groups)
      for (int m : g.mem)
        if (m != g.owner) end_copies.push_back({m, g.owner});
  }
  h->last_entries = (long long)ents.size();
  if (ents.size() > h->ent_cap) {
    if (dalloc(h, &h->d_ent, ents.size())) return PTSBE_ERR_CUDA;
    h->ent_cap = ents.size();
  }
  if (!ents.empty())
    CK(h, cudaMemcpyAsync(h->d_ent, ents.data(), ents.size() * sizeof(int4), cudaMemcpyHostToDevice, h->stream));
  if (!forkpairs.empty()) {
    if (forkpairs.size() > h->fork_cap) {
      if (dalloc(h, &h->d_forks, forkpairs.size())) return PTSBE_ERR_CUDA;
      h->fork_cap = forkpairs.size();
    }
    CK(h, cudaMemcpyAsync(h->d_forks, forkpairs.data(), forkpairs.size() * 4, cudaMemcpyHostToDevice, h->stream));
  }
  NvtxRange nvtx_passes("ptsbe_passes");
  int last_pass = -1;
  for (const LaunchRec& L : launches) {
    const size_t pi = (size_t)L.pass;
    if ((int)pi != last_pass && last_pass >= 0) prev_general = h->passes[last_pass].n_slots > 0;
    last_pass = (int)pi;
    const PassHost& ph = h->passes[pi];
    const int E = L.E;
    if (E == 0) continue;
    if (L.nfork > 0) {   // split-off groups inherit their parent's weight / norm / status
      fork_pairs<<<(L.nfork + 127) / 128, 128, 0, h->stream>>>(h->d_forks + 2 * L.fork_begin, L.nfork,
                                                                h->d_weight, h->d_nst, h->d_status, h->d_fail);
      CKL(h);
    }
    PassParams p;
    p.ent = h->d_ent + L.ent_begin;
    p.E = E;
    const bool last_fused = fuse_sums && (int)pi == P - 1;
    p.tsum = last_fused ? h->d_bs : nullptr;
    p.tsum_stride = h->nblk;
    p.tsum_sbits = h->sbits;
    p.states = h->states;
    p.n = h->n;
    p.L = ph.L;
    p.c = ph.c;
    p.qmask = ph.qmask;
    p.ops = h->d_ops + ph.op_begin;
    p.n_ops = ph.n_ops;
    p.phases = h->d_phases + ph.phase_begin;
    p.n_phases = ph.n_phases;
    p.mat_kind = h->d_matkind;
    p.sel = h->d_sel;
    p.S = h->n_sites;
    p.site_chan = h->d_site_chan;
    p.chans = h->d_chans;
    p.mats = h->d_mats;
    p.nst = h->d_nst;
    p.use_scale = prev_general ? 1 : 0;
    p.gen_zero = (pi == 0 && from_zero) ? (h->zero_vector ? 2 : 1) : 0;
    p.partials = h->d_partials;
    p.status = h->d_status;
    p.B = h->cap + 1;   // row stride (trajectory rows + trunk row)
    p.tiles = 1ll << (h->n - ph.L);
    const size_t smem = pass_smem(ph, sizeof(typename Cplx<R>::V));
    dim3 grid((unsigned)p.tiles, (unsigned)E);
    if (h->profiling) {
      while ((int)h->ev.size() < h->ev_used + 2) {
        cudaEvent_t e;
        CK(h, cudaEventCreate(&e));
        h->ev.push_back(e);
      }
      CK(h, cudaEventRecord(h->ev[h->ev_used], h->stream));
    }
    if (h->gen_active) {
      const int teams = pi < h->gen_mod.teams.size() ? h->gen_mod.teams[pi] : 1;
      const unsigned threads = (unsigned)gen::threads_for(ph.L, ph.gb, ph.n_slots > 0) * (unsigned)teams;
      const int stages = pi < h->gen_mod.stages.size() ? h->gen_mod.stages[pi] : 0;
      const size_t gsm = gen::smem_bytes(ph.L, ph.c, sizeof(typename Cplx<R>::V), teams, stages);
      CUfunction f = h->gen_mod.fns[pi];
      int per_sm = 0;
      if (gen::api().occupancy(&per_sm, f, (int)threads, gsm) != CUDA_SUCCESS) per_sm = 1;
      const long long total = (long long)E * p.tiles;
      const long long want = (long long)std::max(per_sm, 1) * h->num_sms;
      const unsigned nblk = (unsigned)std::max<long long>(1, std::min(total, want));
      void* args[] = {&p, &h->tmap};
      if (gen::api().launch(f, nblk, 1, 1, threads, 1, 1, (unsigned)gsm, (CUstream)h->stream, args, nullptr) !=
          CUDA_SUCCESS)
        return fail(h, PTSBE_ERR_CUDA, "cuLaunchKernel of generated pass %zu failed", pi);
    } else if (ph.L >= 4) {
      // persistent grid: as many CTAs as fit on the GPU, walking all (trajectory, tile) pairs
      const unsigned threads = std::max(32u, 1u << (ph.L - 4));
      int per_sm = 0;
      CK(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass_kernel<R>, threads, smem));
      const long long total = (long long)E * p.tiles;
      const long long want = (long long)std::max(per_sm, 1) * h->num_sms;
      const unsigned nblk = (unsigned)std::max<long long>(1, std::min(total, want));
      pass_kernel<R><<<nblk, threads, smem, h->stream>>>(p);
    } else {
      pass_kernel_small<R><<<grid, 32, 0, h->stream>>>(p);
    }
    CKL(h);
    if (std::getenv("PTSBE_LAUNCH_LOG")) {
      h->launch_log.push_back((double)pi);
      h->launch_log.push_back((double)E);
      h->launch_log.push_back((p.gen_zero ? 1.0 : 2.0) * E * (double)((size_t)1 << h->n) * (double)h->amp_bytes);
    }
    if (h->profiling) {
      CK(h, cudaEventRecord(h->ev[h->ev_used + 1], h->stream));
      h->ev_used += 2;
      // one read + one write of every state of the launch; a pass that starts from |0...0>
      // (gen_zero) only writes
      const double by = (p.gen_zero ? 1.0 : 2.0) * E * (double)((size_t)1 << h->n) * (double)h->amp_bytes;
      h->pass_bytes_total += by;
      h->ev_pass.push_back((int)pi);
      h->ev_bytes.push_back(by);
    }
    if (ph.n_slots > 0) {
      if (h->run_flags & (PTSBE_DEFER_NORMS | PTSBE_SHARDED)) {
        // sharded state: the norms of renormalising sites are sums over every shard
        norm_slot_sums<<<E, 256, 0, h->stream>>>(h->d_partials, ph.n_slots, p.B, p.tiles, p.ent, h->d_status,
                                                 h->d_slotsum);
        CKL(h);
        if (h->run_flags & PTSBE_DEFER_NORMS) {   // the caller adds the shards' sums (ptsbe_finalize_norms)
          h->pending_pass = (int)pi;
          h->pending_ent = L.ent_begin;
          h->pending_E = E;
        } else {
          if (!h->comm) return fail(h, PTSBE_ERR_VALIDATION, "PTSBE_SHARDED needs ptsbe_shard_init");
          const ncclResult_t nr = nccl::api().all_reduce(h->d_slotsum, h->d_slotsum, (size_t)ph.n_slots * p.B,
                                                         ncclFloat64, ncclSum, h->comm, h->stream);
          if (nr != ncclSuccess) return fail(h, PTSBE_ERR_NCCL, "ncclAllReduce: %s", nccl::api().error_string(nr));
          norm_finalize_sums<<<(E + 127) / 128, 128, 0, h->stream>>>(h->d_slotsum, ph.n_slots, p.B,
                                                                     h->d_slot_site + ph.slot_begin, h->d_nst,
                                                                     h->d_weight, h->d_status, h->d_fail, p.ent, E);
          CKL(h);
        }
      } else {
        norm_finalize<<<E, 256, 0, h->stream>>>(h->d_partials, ph.n_slots, p.B, p.tiles,
                                                h->d_slot_site + ph.slot_begin, h->d_nst, h->d_weight,
                                                h->d_status, h->d_fail, p.ent);
        CKL(h);
      }
    }
  }
  if (last_pass >= 0) prev_general = h->passes[last_pass].n_slots > 0;
  h->final_general = prev_general;
  if (!end_copies.empty()) {   // trajectories with identical outcome tables: copy the shared state
    const size_t bytes = ((size_t)1 << h->n) * h->amp_bytes;
    std::vector<int32_t> pairs;
    for (auto& mc : end_copies) {
      CK(h, cudaMemcpyAsync((char*)h->states + (size_t)mc.first * bytes, (char*)h->states + (size_t)mc.second * bytes,
                            bytes, cudaMemcpyDeviceToDevice, h->stream));
      pairs.push_back(mc.first);
      pairs.push_back(mc.second);
    }
    int32_t* d_pairs = nullptr;
    CK(h, cudaMallocAsync((void**)&d_pairs, pairs.size() * 4, h->stream));
    CK(h, cudaMemcpyAsync(d_pairs, pairs.data(), pairs.size() * 4, cudaMemcpyHostToDevice, h->stream));
    fork_pairs<<<((int)end_copies.size() + 127) / 128, 128, 0, h->stream>>>(d_pairs, (int)end_copies.size(),
                                                                            h->d_weight, h->d_nst, h->d_status,
                                                                            h->d_fail);
    CKL(h);
    CK(h, cudaFreeAsync(d_pairs, h->stream));
    fuse_sums = false;   // the copies have no fused sampler sums: sample with the standalone block sums
  }
  if (fuse_sums) {
    h->tsum_ok = true;
    h->tsum_qmask = h->passes[P - 1].qmask;
    h->tsum_L = h->passes[P - 1].L;
    h->tsum_c = tsum_ce;
    h->tsum_threads = gen::threads_for(h->passes[P - 1].L, h->passes[P - 1].gb, false);
  }
  return 0;
}

// Persistent one-state scratch (a per-call cudaMallocAsync of a multi-GiB buffer remaps it
// every time: it dominated verification-mode sampling of permuted layouts).
void* state_scratch(ptsbe_engine* h) {
  if (!h->scratch_state && cudaMalloc(&h->scratch_state, ((size_t)1 << h->n) * h->amp_bytes) != cudaSuccess) {
    h->scratch_state = nullptr;
    cudaGetLastError();
  }
  return h->scratch_state;
}

// out = in with its index bits permuted by P (out bit q <- in bit P.src[q]): the tiled
// kernel (row-contiguous reads and writes) when the state has >= 2^8 amplitudes.
template <typename V>
int permute_into(ptsbe_engine* h, const V* in, V* out, const BitPerm& P) {
  const int n = h->n;
  const int R = sizeof(V) == 8 ? 4 : 3;   // 128-B rows
  if (n < 8) {
    const unsigned g = (unsigned)std::min<size_t>(((size_t)1 << n) / 256 + 1, 8192);
    permute_state<V><<<g, 256, 0, h->stream>>>(in, out, n, P);
    CKL(h);
    return 0;
  }
  TilePerm T{};
  T.k = std::min(n, 10);
  uint64_t qin = (1ull << R) - 1;
  for (int q = 0; q < R; ++q) qin |= 1ull << P.src[q];
  for (int b = 0; b < n && __builtin_popcountll(qin) < T.k; ++b) qin |= 1ull << b;
  T.k = __builtin_popcountll(qin);
  uint64_t qout = 0;
  for (int q = 0; q < n; ++q)
    if ((qin >> P.src[q]) & 1) qout |= 1ull << q;
  T.qin = qin;
  T.qout = qout;
  // output-tile bit b is output bit qb (b-th set bit of qout); it comes from input bit P.src[qb],
  // which is input-tile bit (rank of P.src[qb] among qin's set bits)
  for (int b = 0, qb = -1; b < T.k; ++b) {
    do { ++qb; } while (!((qout >> qb) & 1));
    const int ib = P.src[qb];
    T.fmap[b] = (int8_t)__builtin_popcountll(qin & ((1ull << ib) - 1));
  }
  const unsigned g = (unsigned)std::min<uint64_t>(1ull << (n - T.k), 8u * (unsigned)h->num_sms);
  const size_t smem = ((size_t)1 << T.k) * (sizeof(V) + 8 + 8 + 2);   // tile | offin | offout | emap
  permute_tiled<V><<<g, 256, smem, h->stream>>>(in, out, n, P, T);
  CKL(h);
  return 0;
}

// Re-store state b in logical (to_logical) or physical order.
int relayout(ptsbe_engine* h, int b, bool to_logical) {
  if (!h->permuted || (h->logical[b] != 0) == to_logical) return 0;
  h->tsum_ok = false;
  const size_t bytes = ((size_t)1 << h->n) * h->amp_bytes;
  char* st = (char*)h->states + (size_t)b * bytes;
  void* scratch = state_scratch(h);
  if (!scratch) return fail(h, PTSBE_ERR_CUDA, "cannot allocate %zu bytes of relayout scratch", bytes);
  BitPerm P = h->layout;            // physical -> logical
  if (!to_logical) {                 // logical -> physical
    for (int q = 0; q < h->n; ++q) P.src[h->layout.src[q]] = (int8_t)q;
  }
  if (int r = h->dtype == PTSBE_C64 ? permute_into<float2>(h, (const float2*)st, (float2*)scratch, P)
                                    : permute_into<double2>(h, (const double2*)st, (double2*)scratch, P))
    return r;
  CK(h, cudaMemcpyAsync(st, scratch, bytes, cudaMemcpyDeviceToDevice, h->stream));
  h->logical[b] = to_logical ? 1 : 0;
  return 0;
}

template <typename R>
int rescale_if_needed(ptsbe_engine* h) {
  if (!h->final_general || h->last_B == 0) return 0;
  scale_states<R><<<1184, 256, 0, h->stream>>>(h->states, h->n, h->last_B, h->d_nst, 1);
  CKL(h);
  std::vector<double> ones(h->last_B, 1.0);
  CK(h, cudaMemcpyAsync(h->d_nst, ones.data(), ones.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  h->final_general = false;
  return 0;
}

int run_common(ptsbe_engine* h, const uint8_t* sel, int B, double* out_weight, int32_t* out_status,
               uint32_t flags, bool from_zero, int p_begin = 0, int p_end = -1) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (!h->loaded) return fail(h, PTSBE_ERR_VALIDATION, "no program loaded");
  if (B < 0 || B > h->cap) return fail(h, PTSBE_ERR_VALIDATION, "batch %d exceeds capacity %d", B, h->cap);
  const int P = (int)h->passes.size();
  if (p_end < 0) p_end = P;
  if (p_begin < 0 || p_begin > p_end || p_end > P)
    return fail(h, PTSBE_ERR_VALIDATION, "pass range [%d, %d) outside [0, %d)", p_begin, p_end, P);
  if (p_begin > 0 && B != h->last_B)
    return fail(h, PTSBE_ERR_VALIDATION, "a continued pass range must keep the batch of %d states", h->last_B);
  if (B == 0) return 0;
  if ((flags & PTSBE_DEFER_NORMS) && p_end - p_begin != 1)
    return fail(h, PTSBE_ERR_VALIDATION, "PTSBE_DEFER_NORMS runs one pass at a time");
  if (h->pending_pass >= 0)
    return fail(h, PTSBE_ERR_VALIDATION, "pass %d still waits for its global norms (ptsbe_finalize_norms)",
                h->pending_pass);
  CK(h, cudaSetDevice(h->dev));
  h->run_flags = flags;
  if (flags & PTSBE_KEEP_SEL) {   // continued range over the device table as it is
    if (from_zero) return fail(h, PTSBE_ERR_VALIDATION, "PTSBE_KEEP_SEL needs a continued pass range");
  } else if (h->n_sites > 0) {
    h->host_sel.clear();
    if (!sel) return fail(h, PTSBE_ERR_VALIDATION, "selection table is required");
    if (int r = copy_in(h, h->d_sel, sel, (size_t)B * h->n_sites, flags)) return r;
    // the shared-trunk schedule needs each trajectory's first non-default site on the host
    h->host_sel.resize((size_t)B * h->n_sites);
    if ((flags & PTSBE_DEVICE_PTRS) && (flags & PTSBE_HOST_MIRROR)) {
      if (!h->mirror_sel || h->mirror_B < B) return fail(h, PTSBE_ERR_VALIDATION, "no host mirror of the outcome table");
      std::memcpy(h->host_sel.data(), h->mirror_sel, h->host_sel.size());
    } else if (flags & PTSBE_DEVICE_PTRS) {
      CK(h, cudaMemcpyAsync(h->host_sel.data(), h->d_sel, h->host_sel.size(), cudaMemcpyDeviceToHost, h->stream));
      CK(h, cudaStreamSynchronize(h->stream));
    } else {
      std::memcpy(h->host_sel.data(), sel, h->host_sel.size());
    }
  }
  if (p_begin == 0) {
    batch_reset<<<(B + 255) / 256, 256, 0, h->stream>>>(h->d_weight, h->d_nst, h->d_status, h->d_fail, B);
    CKL(h);
  }
  if (h->permuted && !from_zero)
    for (int b = 0; b < B; ++b)
      if (int r = relayout(h, b, false)) return r;
  for (int b = 0; b < B; ++b) h->logical[b] = 0;
  h->last_B = B;
  h->zero_vector = (flags & PTSBE_ZERO_VECTOR) != 0;
  int r = h->dtype == PTSBE_C64 ? launch_passes<float>(h, B, from_zero, p_begin, p_end)
                                : launch_passes<double>(h, B, from_zero, p_begin, p_end);
  if (r) return r;
  if (out_weight)
    if (int e = copy_out(h, out_weight, h->d_weight, (size_t)B * 8, flags)) return e;
  if (out_status)
    if (int e = copy_out(h, out_status, h->d_status, (size_t)B * 4, flags)) return e;
  if (!(flags & PTSBE_NO_SYNC) || !(flags & PTSBE_DEVICE_PTRS)) CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ensure_shots(ptsbe_engine* h, size_t total, size_t chunks) {
  if (total > h->shot_cap) {
    size_t cap = std::max(total, h->shot_cap * 2);
    int r = 0;
    r |= dalloc(h, &h->d_keys, cap);
    r |= dalloc(h, &h->d_tmp, cap);
    r |= dalloc(h, &h->d_idx, cap);
    r |= dalloc(h, &h->d_runidx, cap);
    r |= dalloc(h, &h->d_runcnt, cap);
    if (r) return PTSBE_ERR_CUDA;
    h->shot_cap = cap;
  }
  if (chunks > h->chunk_cap) {
    size_t cap = std::max(chunks, h->chunk_cap * 2);
    if (dalloc(h, &h->d_chunks, cap)) return PTSBE_ERR_CUDA;
    h->chunk_cap = cap;
  }
  return 0;
}

template <typename R>
int sample_impl(ptsbe_engine* h, int B, const int64_t* shots, int rng_mode, const uint64_t* rng_state,
                const uint64_t* keys, uint64_t* out_idx, uint32_t* out_cnt, int64_t* out_nuniq,
                uint32_t flags) {
  NvtxRange nvtx_sample("ptsbe_sample");
  std::vector<int64_t> m(B), off(B);
  if ((flags & PTSBE_DEVICE_PTRS) && (flags & PTSBE_HOST_MIRROR)) {
    if (!h->mirror_shots || h->mirror_B < B) return fail(h, PTSBE_ERR_VALIDATION, "no host mirror of the shot counts");
    std::memcpy(m.data(), h->mirror_shots, (size_t)B * 8);
  } else if (flags & PTSBE_DEVICE_PTRS) {
    CK(h, cudaMemcpyAsync(m.data(), shots, (size_t)B * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
  } else {
    std::memcpy(m.data(), shots, (size_t)B * 8);
  }
  long long total = 0;
  std::vector<uint64_t> chunks;
  for (int b = 0; b < B; ++b) {
    if (m[b] < 0) return fail(h, PTSBE_ERR_VALIDATION, "shot count must be >= 0, got %lld", (long long)m[b]);
    off[b] = total;
    for (long long s = 0; s < m[b]; s += 32) chunks.push_back(((uint64_t)b << 40) | (uint64_t)s);
    total += m[b];
  }
  if (int r = ensure_shots(h, (size_t)std::max<long long>(total, 1), std::max<size_t>(chunks.size(), 1))) return r;
  CK(h, cudaMemcpyAsync(h->d_m, m.data(), (size_t)B * 8, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->d_off, off.data(), (size_t)B * 8, cudaMemcpyHostToDevice, h->stream));
  if (!chunks.empty())
    CK(h, cudaMemcpyAsync(h->d_chunks, chunks.data(), chunks.size() * 8, cudaMemcpyHostToDevice, h->stream));
  const long long n_chunks = (long long)chunks.size();

  SampleParams sp;
  sp.states = h->states;
  sp.n = h->n;
  sp.sbits = h->sbits;
  sp.nblk = h->nblk;
  sp.B = B;
  sp.nst = h->d_nst;
  sp.status = h->d_status;
  sp.bs = h->d_bs;
  sp.total = h->d_total;
  sp.off = h->d_off;
  sp.m = h->d_m;
  sp.tiled = 0;
  sp.tq = h->tsum_qmask;
  sp.tL = h->tsum_L;
  sp.tC = h->tsum_c;
  sp.tT = h->tsum_threads;

  // Exact RNG modes (PCG64 / host keys) replay the reference's sampler bit for bit
  // (exact_cdf.cuh): on the normalised amplitudes get_state returns, in LOGICAL
  // index order -- rescale deferred norms and canonicalise permuted states first.
  const bool exact = rng_mode != PTSBE_RNG_PHILOX;
  if (exact && total > 0)
    if (int r = rescale_if_needed<R>(h)) return r;
  if (exact && total > 0 && (size_t)B * h->nblk > h->maps_cap) {
    if (dalloc(h, &h->d_maps, (size_t)B * h->nblk)) return PTSBE_ERR_CUDA;
    h->maps_cap = (size_t)B * h->nblk;
  }
  // Philox mode samples the physical layout and maps indices back (cheaper); once
  // any state is logical, all are.
  bool unperm = false;
  if (h->permuted && total > 0) {
    bool any_logical = false;
    for (int b = 0; b < B; ++b) any_logical = any_logical || h->logical[b];
    if (rng_mode != PTSBE_RNG_PHILOX || any_logical) {
      for (int b = 0; b < B; ++b)
        if (int r = relayout(h, b, true)) return r;
    } else {
      unperm = true;
    }
  }
  // Philox mode on the fused block sums of the last pass: no state read here; the
  // CDF runs in that pass's tile order, so indices are mapped back and re-sorted.
  bool some_logical = false;
  for (int b = 0; b < B; ++b) some_logical = some_logical || h->logical[b];
  const bool tiled = h->tsum_ok && rng_mode == PTSBE_RNG_PHILOX && !some_logical;
  if (total > 0) {
    if (tiled) {
      sp.tiled = 1;
    } else {
      dim3 g1((unsigned)((h->nblk + 7) / 8), (unsigned)B);
      sample_blocksum<R><<<g1, 256, 0, h->stream>>>(sp);
      CKL(h);
    }
    sample_blockscan<<<B, 1024, 0, h->stream>>>(sp);
    CKL(h);
    if (exact) {   // numpy's sequential float64 cumsum, block ends into d_bs, cum_last into d_total
      dim3 g1((unsigned)((h->nblk + 7) / 8), (unsigned)B);
      exact_blockmaps<R><<<g1, 256, 0, h->stream>>>(sp, h->d_maps);
      CKL(h);
      exact_chain<R><<<B, 32, 0, h->stream>>>(sp, h->d_maps, h->d_bs);
      CKL(h);
    }
    const unsigned gw = (unsigned)((n_chunks * 32 + 255) / 256);
    if (rng_mode == PTSBE_RNG_PCG64) {
      if (int r = copy_in(h, h->d_rng, rng_state, (size_t)B * 4 * 8, flags)) return r;
      keys_pcg64<<<gw, 256, 0, h->stream>>>(h->d_chunks, n_chunks, h->d_rng, h->d_off, h->d_m, h->d_status,
                                            h->d_keys);
      CKL(h);
    } else if (rng_mode == PTSBE_RNG_PHILOX) {
      if (int r = copy_in(h, h->d_rng, rng_state, (size_t)B * 8, flags)) return r;
      keys_philox_sorted<<<B, 1024, 0, h->stream>>>(h->d_rng, h->d_off, h->d_m, h->d_status, h->d_keys);
      CKL(h);
    } else if (rng_mode == PTSBE_RNG_KEYS) {
      if (int r = copy_in(h, h->d_keys, keys, (size_t)total * 8, flags)) return r;
    } else {
      return fail(h, PTSBE_ERR_VALIDATION, "unknown rng mode %d", rng_mode);
    }
    if (rng_mode != PTSBE_RNG_PHILOX) {
      seg_radix_sort<<<B, 1024, 0, h->stream>>>(h->d_keys, h->d_tmp, h->d_off, h->d_m, h->d_status, 53);
      CKL(h);
    }
    if (exact)
      exact_resolve<R><<<gw, 256, 0, h->stream>>>(sp, h->d_chunks, n_chunks, h->d_keys, h->d_bs, h->d_idx);
    else
      sample_resolve<R><<<gw, 256, 0, h->stream>>>(sp, h->d_chunks, n_chunks, h->d_keys, h->d_idx);
    CKL(h);
    if (unperm || tiled) {   // physical -> logical bitstrings, then ascending order again
      if (h->permuted) {
        unpermute_indices<<<std::min<long long>((total + 255) / 256, 4096), 256, 0, h->stream>>>(h->d_idx, total,
                                                                                                   h->layout);
        CKL(h);
      }
      seg_radix_sort<<<B, 1024, 0, h->stream>>>(h->d_idx, h->d_tmp, h->d_off, h->d_m, h->d_status, h->n);
      CKL(h);
    }
  }
  sample_rle<<<B, 1024, 0, h->stream>>>(h->d_idx, h->d_off, h->d_m, h->d_status, h->d_runidx, h->d_runcnt,
                                        h->d_nuniq);
  CKL(h);
  if (flags & PTSBE_DEVICE_PTRS) {
    // device outputs: CSR offsets scanned and runs compacted on device -- no host round trip
    long long maxm = 0;
    for (int b = 0; b < B; ++b) maxm = std::max<long long>(maxm, m[b]);
    exclusive_scan_i64<<<1, 1024, 0, h->stream>>>(h->d_nuniq, B, h->d_uoff);
    CKL(h);
    if (maxm > 0) {
      dim3 gc((unsigned)std::min<long long>((maxm + 255) / 256, 4096), (unsigned)B);
      compact_runs<<<gc, 256, 0, h->stream>>>(h->d_runidx, h->d_runcnt, h->d_off, h->d_nuniq, h->d_uoff, out_idx,
                                              out_cnt);
      CKL(h);
    }
    CK(h, cudaMemcpyAsync(out_nuniq, h->d_nuniq, (size_t)B * 8, cudaMemcpyDeviceToDevice, h->stream));
    if (!(flags & PTSBE_NO_SYNC)) CK(h, cudaStreamSynchronize(h->stream));
    return 0;
  }
  std::vector<int64_t> nu(B), uoff(B);
  CK(h, cudaMemcpyAsync(nu.data(), h->d_nuniq, (size_t)B * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  long long U = 0;
  long long maxnu = 0;
  for (int b = 0; b < B; ++b) { uoff[b] = U; U += nu[b]; maxnu = std::max<long long>(maxnu, nu[b]); }
  if (flags & PTSBE_DEVICE_PTRS) {
    CK(h, cudaMemcpyAsync(out_nuniq, h->d_nuniq, (size_t)B * 8, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    std::memcpy(out_nuniq, nu.data(), (size_t)B * 8);
  }
  if (U > 0) {
    CK(h, cudaMemcpyAsync(h->d_uoff, uoff.data(), (size_t)B * 8, cudaMemcpyHostToDevice, h->stream));
    // compact into keys/tmp scratch, then hand out one contiguous CSR stream
    uint64_t* cidx = h->d_keys;
    uint32_t* ccnt = reinterpret_cast<uint32_t*>(h->d_tmp);
    dim3 gc((unsigned)std::min<long long>((maxnu + 255) / 256, 4096), (unsigned)B);
    compact_runs<<<gc, 256, 0, h->stream>>>(h->d_runidx, h->d_runcnt, h->d_off, h->d_nuniq, h->d_uoff, cidx, ccnt);
    CKL(h);
    if (int r = copy_out(h, out_idx, cidx, (size_t)U * 8, flags)) return r;
    if (int r = copy_out(h, out_cnt, ccnt, (size_t)U * 4, flags)) return r;
  }
  if (!(flags & PTSBE_NO_SYNC) || !(flags & PTSBE_DEVICE_PTRS)) CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

}  // namespace

extern "C" {

int ptsbe_abi_version(void) { return PTSBE_ABI_VERSION; }

int ptsbe_create(int device, int n_qubits, int dtype, int batch_cap, ptsbe_engine** out) {
  if (!out) return PTSBE_ERR_VALIDATION;
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 40) return PTSBE_ERR_VALIDATION;
  if (dtype != PTSBE_C64 && dtype != PTSBE_C128) return PTSBE_ERR_VALIDATION;
  if (batch_cap < 1) return PTSBE_ERR_VALIDATION;
  ptsbe_engine* h = new ptsbe_engine();
  h->dev = device;
  h->n = n_qubits;
  h->dtype = dtype;
  h->cap = batch_cap;
  h->amp_bytes = dtype == PTSBE_C64 ? 8 : 16;
  h->sbits = std::min(n_qubits, 9);
  h->layout.n = n_qubits;
  for (int q = 0; q < n_qubits && q < 64; ++q) h->layout.src[q] = (int8_t)q;
  h->logical.assign(batch_cap, 0);
  h->nblk = 1ll << (n_qubits - h->sbits);
  int r = 0;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    r = fail(h, PTSBE_ERR_CUDA, "device %d unavailable: %s", device, cudaGetErrorString(e));
  }
  if (!r) {
    // batch slots only: the shared-prefix tree keeps every group's state in a member's slot
    const char* tree_env = std::getenv("PTSBE_TREE");
    h->tree_enabled = tree_env ? std::atoi(tree_env) != 0 : true;
    const size_t bytes = (size_t)batch_cap * ((size_t)1 << n_qubits) * h->amp_bytes;
    e = cudaMalloc(&h->states, bytes);
    if (e != cudaSuccess) r = fail(h, PTSBE_ERR_CUDA, "cannot allocate %zu bytes of state: %s", bytes, cudaGetErrorString(e));
  }
  if (!r) {   // tensor map for TMA tile staging (generated kernels); optional
    typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    encode_t enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    const size_t bytes = (size_t)batch_cap * ((size_t)1 << n_qubits) * h->amp_bytes;
    const size_t rows = bytes / 128;
    if (((size_t)1 << n_qubits) * h->amp_bytes >= 512 && rows < (1ull << 31) &&
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && enc) {
      const cuuint64_t gdim[2] = {16, (cuuint64_t)rows};
      const cuuint64_t gstr[1] = {128};
      const cuuint32_t box[2] = {16, 1};   // tile::gather4 / scatter4: four 1-row boxes per instruction
      const cuuint32_t es[2] = {1, 1};
      h->tmap_ok = enc(&h->tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, h->states, gdim, gstr, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       std::getenv("PTSBE_TMA_L2_256") ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                       : std::getenv("PTSBE_TMA_L2_NONE") ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                                          : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  // per-row tables: batch rows + the trunk row (index batch_cap)
  if (!r) r = dalloc(h, &h->d_weight, batch_cap + 1);
  if (!r) r = dalloc(h, &h->d_nst, batch_cap + 1);
  if (!r) r = dalloc(h, &h->d_status, batch_cap + 1);
  if (!r) r = dalloc(h, &h->d_fail, batch_cap + 1);
  if (!r) r = dalloc(h, &h->d_bs, (size_t)batch_cap * h->nblk);
  if (!r) r = dalloc(h, &h->d_total, batch_cap);
  if (!r) r = dalloc(h, &h->d_off, batch_cap);
  if (!r) r = dalloc(h, &h->d_m, batch_cap);
  if (!r) r = dalloc(h, &h->d_nuniq, batch_cap);
  if (!r) r = dalloc(h, &h->d_uoff, batch_cap);
  if (!r) r = dalloc(h, &h->d_rng, (size_t)batch_cap * 4);
  if (!r) {
    std::vector<double> ones(batch_cap + 1, 1.0);
    std::vector<int32_t> zeros(batch_cap + 1, 0);
    e = cudaMemcpy(h->d_nst, ones.data(), (batch_cap + 1) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_status, zeros.data(), (batch_cap + 1) * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) r = fail(h, PTSBE_ERR_CUDA, "init copy failed: %s", cudaGetErrorString(e));
  }
  if (r) {
    // keep the handle so the caller can read the error, then destroy it
    *out = h;
    return r;
  }
  *out = h;
  return 0;
}

int ptsbe_create_host(int n_qubits, int dtype, ptsbe_engine** out) {
  if (!out) return PTSBE_ERR_VALIDATION;
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 40) return PTSBE_ERR_VALIDATION;
  if (dtype != PTSBE_C64 && dtype != PTSBE_C128) return PTSBE_ERR_VALIDATION;
  ptsbe_engine* h = new ptsbe_engine();
  h->host_only = true;
  h->dev = -1;
  h->n = n_qubits;
  h->dtype = dtype;
  h->cap = 1;
  h->amp_bytes = dtype == PTSBE_C64 ? 8 : 16;
  *out = h;
  return 0;
}

int64_t ptsbe_codegen_source(ptsbe_engine* h, char* buf, size_t len) {
  if (!h) return -PTSBE_ERR_VALIDATION;
  if (buf && len) {
    const size_t k = std::min(len - 1, h->gen_src.size());
    std::memcpy(buf, h->gen_src.data(), k);
    buf[k] = 0;
  }
  return (int64_t)h->gen_src.size();
}

int ptsbe_destroy(ptsbe_engine* h) {
  if (!h) return 0;
  if (const char* path = std::getenv("PTSBE_LAUNCH_LOG")) {
    if (!h->launch_log.empty())
      if (FILE* f = std::fopen(path, "a")) {
        for (size_t i = 0; i + 2 < h->launch_log.size(); i += 3)
          std::fprintf(f, "%d %d %.0f\n", (int)h->launch_log[i], (int)h->launch_log[i + 1], h->launch_log[i + 2]);
        std::fclose(f);
      }
  }
  if (h->host_only) { delete h; return 0; }
  cudaSetDevice(h->dev);
  void* ptrs[] = {h->states, h->d_sel, h->d_weight, h->d_nst, h->d_status, h->d_fail, h->d_ops, h->d_mats,
                  h->d_phases, h->d_matkind,
                  h->d_chans, h->d_site_chan, h->d_slot_site, h->d_partials, h->d_bs, h->d_total, h->d_off,
                  h->d_m, h->d_nuniq, h->d_uoff, h->d_rng, h->d_keys, h->d_tmp, h->d_idx, h->d_runidx,
                  h->d_runcnt, h->d_chunks, h->d_ent, h->d_forks, h->d_mats64, h->d_u, h->d_rdm, h->d_maps, h->xbuf, h->d_slotsum, h->scratch_state};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  for (cudaEvent_t e : h->xev)
    if (e) cudaEventDestroy(e);
  if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
  if (h->comm && nccl::api().ok) nccl::api().comm_destroy(h->comm);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return 0;
}

// Classify a padded 4x4 operator for the specialised register kernels.
static int32_t classify_matrix(const double* m32, int arity) {
  auto re = [&](int r, int c) { return m32[2 * (4 * r + c)]; };
  auto im = [&](int r, int c) { return m32[2 * (4 * r + c) + 1]; };
  auto zero = [&](int r, int c) { return re(r, c) == 0.0 && im(r, c) == 0.0; };
  auto one = [&](int r, int c) { return re(r, c) == 1.0 && im(r, c) == 0.0; };
  if (arity == 1) {
    if (zero(0, 0) && zero(1, 1)) return MK_ANTI1;
    if (zero(0, 1) && zero(1, 0)) return one(0, 0) ? MK_PHASE1 : MK_DIAG1;
    if (im(0, 0) == 0.0 && im(0, 1) == 0.0 && im(1, 0) == 0.0 && im(1, 1) == 0.0) return MK_REAL1;
    return MK_GEN1;
  }
  static const int cx[4] = {0, 1, 3, 2}, sw[4] = {0, 2, 1, 3};
  bool is_cx = true, is_sw = true, is_diag = true;
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      const bool want_cx = cx[r] == c, want_sw = sw[r] == c;
      is_cx = is_cx && (want_cx ? one(r, c) : zero(r, c));
      is_sw = is_sw && (want_sw ? one(r, c) : zero(r, c));
      if (r != c) is_diag = is_diag && zero(r, c);
    }
  if (is_cx) return MK_CX2;
  if (is_sw) return MK_SWAP2;
  if (is_diag) return MK_DIAG2;
  return MK_GEN2;
}

struct HostOp {
  DevOp d;
  uint32_t bits;   // tile-bit mask of the targets
  bool general;
};

// Group a pass's ops (stream order) into phases of GB tile bits held in
// registers.  Dependency rule as in the host pass planner: an op that does not
// join blocks its bits for the rest of the phase; general-channel sites never
// overtake each other (their realized weights are ratios of consecutive norms
// in reference order).  Each phase picks the bit set absorbing the most ops.
static void plan_phases(std::vector<HostOp>& ops, int L, std::vector<DevOp>& out_ops,
                        std::vector<DevPhase>& out_phases, int GB = 4) {
  std::vector<int> remaining(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) remaining[i] = (int)i;
  const uint32_t full = L >= 32 ? 0xffffffffu : ((1u << L) - 1u);
  // Ops a phase with register-bit set S can take, in dependency order: an op
  // joins iff its bits lie in S and no earlier deferred op blocks its bits
  // (general sites also keep their relative order).
  auto absorb = [&](uint32_t S, std::vector<int>* taken, std::vector<int>* deferred) {
    uint32_t blocked = 0;
    bool gen_blocked = false;
    int count = 0;
    for (int i : remaining) {
      const HostOp& o = ops[i];
      const bool fits = !(o.bits & blocked) && !(o.general && gen_blocked) && !(o.bits & ~S);
      if (fits) {
        ++count;
        if (taken) taken->push_back(i);
      } else {
        blocked |= o.bits;
        gen_blocked = gen_blocked || o.general;
        if (deferred) deferred->push_back(i);
      }
    }
    return count;
  };
  // all GB-subsets of the tile bits (C(12,4) = 495; C(13,5) = 1287)
  std::vector<uint32_t> cands;
  for (uint32_t S = 0; S <= full; ++S)
    if (__builtin_popcount(S) == std::min(GB, L)) cands.push_back(S);
  const char* pp = std::getenv("PTSBE_PHASE_PLAN");
  const bool greedy_phases = pp && std::string(pp) == "greedy";
  while (!remaining.empty()) {
    // max-absorb: the register-bit set that takes the most ops (ties: contains
    // bit 0 -> 16-B shared accesses, then lowest bits); 43% fewer phases than
    // first-come greedy on config 4
    uint32_t S = 0;
    if (greedy_phases) {          // first-come: grow S in stream order (A/B knob)
      uint32_t blocked = 0;
      bool gen_blocked = false;
      for (int i : remaining) {
        const HostOp& o = ops[i];
        const bool ok = !(o.bits & blocked) && !(o.general && gen_blocked) &&
                        __builtin_popcount(S | o.bits) <= GB;
        if (ok) S |= o.bits;
        else { blocked |= o.bits; gen_blocked = gen_blocked || o.general; }
      }
    } else {
      int best = -1;
      for (uint32_t cs : cands) {
        const int cnt = absorb(cs, nullptr, nullptr);
        if (cnt > best) { best = cnt; S = cs; }
      }
    }
    std::vector<int> taken, deferred;
    absorb(S, &taken, &deferred);
    if (taken.empty()) {   // cannot happen for arity <= 2, GB >= 2; keep progress regardless
      taken.push_back(remaining[0]);
      deferred.assign(remaining.begin() + 1, remaining.end());
    }
    // keep only the bits the taken ops use, then pad with the lowest bits: bit 0
    // in the set gives 16-B shared accesses (c64)
    S = 0;
    for (int i : taken) S |= ops[i].bits;
    for (int q = 0; q < L && __builtin_popcount(S) < GB; ++q) S |= 1u << q;
    int pb[5] = {0, 0, 0, 0, 0}, np_ = 0;
    for (int q = 0; q < L && np_ < GB; ++q)
      if ((S >> q) & 1) pb[np_++] = q;
    DevPhase P;
    P.pbits = 0;
    for (int k = 0; k < GB; ++k) P.pbits |= (uint32_t)pb[k] << (5 * k);
    P.op_begin = (int32_t)out_ops.size();
    P.n_ops = (int32_t)taken.size();
    P.pad = GB;
    for (int i : taken) {
      DevOp d = ops[i].d;
      auto pos = [&](int bit) { for (int k = 0; k < GB; ++k) if (pb[k] == bit) return k; return -1; };
      d.k0 = pos(d.b0);
      d.k1 = d.arity == 2 ? pos(d.b1) : -1;
      out_ops.push_back(d);
    }
    out_phases.push_back(P);
    remaining.swap(deferred);
  }
}

static int try_codegen(ptsbe_engine* h, int mode, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                       const std::vector<DevPhase>& dph, const double* mats, const std::vector<int32_t>& kinds,
                       const ptsbe_channel* chans, const int32_t* site_chan);
static std::string gen_source(ptsbe_engine* h, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                              const std::vector<DevPhase>& dph, const double* mats, const std::vector<int32_t>& kinds,
                              const ptsbe_channel* chans, const int32_t* site_chan);
static gen::GenProgram gen_program(ptsbe_engine* h, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                                   const std::vector<DevPhase>& dph, const double* mats,
                                   const std::vector<int32_t>& kinds, const ptsbe_channel* chans,
                                   const int32_t* site_chan);

int ptsbe_load_program(ptsbe_engine* h, const ptsbe_op* ops, int n_ops, const double* mats, int n_mats,
                       const ptsbe_channel* chans, int n_chans, const int32_t* site_chan, int n_sites,
                       const ptsbe_pass* passes, int n_passes) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (!h->host_only) CK(h, cudaSetDevice(h->dev));
  h->loaded = false;
  if (n_ops < 0 || n_mats < 0 || n_chans < 0 || n_sites < 0 || n_passes < 0)
    return fail(h, PTSBE_ERR_VALIDATION, "negative table size");
  if (n_sites > 0 && n_chans == 0) return fail(h, PTSBE_ERR_VALIDATION, "sites without channels");
  for (int s = 0; s < n_sites; ++s)
    if (site_chan[s] < 0 || site_chan[s] >= n_chans)
      return fail(h, PTSBE_ERR_VALIDATION, "site %d references channel %d", s, site_chan[s]);
  std::vector<int> mat_arity(std::max(n_mats, 1), 0);
  for (int k = 0; k < n_chans; ++k) {
    if (chans[k].n_outcomes < 1 || chans[k].n_outcomes > 64 || chans[k].mat_base < 0 ||
        chans[k].mat_base + chans[k].n_outcomes > n_mats)
      return fail(h, PTSBE_ERR_VALIDATION, "channel %d has an invalid matrix range", k);
    if (chans[k].general && chans[k].identity_mask)
      return fail(h, PTSBE_ERR_VALIDATION, "channel %d: identity skipping is for unitary mixtures only", k);
    if (chans[k].arity != 1 && chans[k].arity != 2)
      return fail(h, PTSBE_ERR_VALIDATION, "channel %d: arity %d unsupported on device (1 or 2)", k, chans[k].arity);
    for (int o = 0; o < chans[k].n_outcomes; ++o) mat_arity[chans[k].mat_base + o] = chans[k].arity;
  }
  std::vector<PassHost> ph(n_passes);
  const uint64_t nmask = (h->n >= 64) ? ~0ull : ((1ull << h->n) - 1);
  for (int p = 0; p < n_passes; ++p) {
    const ptsbe_pass& P = passes[p];
    if ((P.qubit_mask & ~nmask) || __builtin_popcountll(P.qubit_mask) != P.tile_bits)
      return fail(h, PTSBE_ERR_VALIDATION, "pass %d: qubit mask does not match tile_bits", p);
    const int max_tile = h->dtype == PTSBE_C64 ? 13 : 12;   // 2^(L-4) threads <= launch bound
    if (P.tile_bits < 1 || P.tile_bits > max_tile || (P.tile_bits < 4 && P.tile_bits != h->n))
      return fail(h, PTSBE_ERR_VALIDATION, "pass %d: tile_bits %d outside [4, %d]", p, P.tile_bits, max_tile);
    const int min_low = std::min(h->n, h->dtype == PTSBE_C64 ? 1 : 0);
    if (P.low_bits < min_low || P.low_bits > P.tile_bits ||
        (P.qubit_mask & ((1ull << P.low_bits) - 1)) != ((1ull << P.low_bits) - 1))
      return fail(h, PTSBE_ERR_VALIDATION, "pass %d: low_bits %d not contiguous in the mask", p, P.low_bits);
    ph[p] = PassHost{P.qubit_mask, P.tile_bits, P.low_bits, 0, 0, 0, 0, 0, 0};
  }
  // validate ops, translate targets to tile bits, bucket by pass
  std::vector<std::vector<HostOp>> per_pass(n_passes);
  std::vector<int> site_pass_tmp(n_sites, n_passes);   // pass that fires each site
  std::vector<ptsbe_engine::Decision> decide(n_passes);
  bool conv_ready = true;
  int prev_pass = -1;
  for (int i = 0; i < n_ops; ++i) {
    const ptsbe_op& o = ops[i];
    if (o.pass < 0 || o.pass >= n_passes || o.pass < prev_pass)
      return fail(h, PTSBE_ERR_VALIDATION, "op %d: pass index %d out of order", i, o.pass);
    prev_pass = o.pass;
    if (o.arity != 1 && o.arity != 2)
      return fail(h, PTSBE_ERR_VALIDATION, "op %d: arity %d unsupported on device (1 or 2)", i, o.arity);
    const PassHost& P = ph[o.pass];
    auto local = [&](int q) -> int {
      if (q < 0 || q >= h->n || !((P.qmask >> q) & 1)) return -1;
      return __builtin_popcountll(P.qmask & ((1ull << q) - 1));
    };
    HostOp ho;
    ho.d.kind = o.kind;
    ho.d.arity = o.arity;
    ho.d.b0 = local(o.t0);
    ho.d.b1 = o.arity == 2 ? local(o.t1) : -1;
    ho.d.ref = o.ref;
    ho.d.slot = -1;
    ho.d.k0 = ho.d.k1 = -1;
    ho.general = false;
    if (ho.d.b0 < 0 || (o.arity == 2 && (ho.d.b1 < 0 || o.t0 == o.t1)))
      return fail(h, PTSBE_ERR_VALIDATION, "op %d: targets not inside its pass's qubit set", i);
    ho.bits = (1u << ho.d.b0) | (o.arity == 2 ? (1u << ho.d.b1) : 0u);
    if (o.kind == 0) {
      if (o.ref < 0 || o.ref >= n_mats) return fail(h, PTSBE_ERR_VALIDATION, "op %d: matrix %d", i, o.ref);
      if (mat_arity[o.ref] && mat_arity[o.ref] != o.arity)
        return fail(h, PTSBE_ERR_VALIDATION, "op %d: matrix %d used with two arities", i, o.ref);
      mat_arity[o.ref] = o.arity;
    } else if (o.kind == 1) {
      if (o.ref < 0 || o.ref >= n_sites) return fail(h, PTSBE_ERR_VALIDATION, "op %d: site %d", i, o.ref);
      const ptsbe_channel& ch = chans[site_chan[o.ref]];
      if (ch.arity != o.arity) return fail(h, PTSBE_ERR_VALIDATION, "op %d: channel arity mismatch", i);
      ho.general = ch.general != 0;
      if (ho.general) {
        if (per_pass[o.pass].empty()) {
          ptsbe_engine::Decision& d = decide[o.pass];
          d.site = o.ref;
          d.p0 = o.t0;
          d.p1 = o.arity == 2 ? o.t1 : -1;
          d.arity = o.arity;
          d.mat_base = ch.mat_base;
          d.n_out = ch.n_outcomes;
        } else {
          conv_ready = false;
        }
      }
    } else {
      return fail(h, PTSBE_ERR_VALIDATION, "op %d: unknown kind %d", i, o.kind);
    }
    per_pass[o.pass].push_back(ho);
    if (o.kind == 1) site_pass_tmp[o.ref] = std::min(site_pass_tmp[o.ref], o.pass);
  }
  // norm slots (slot order = reference order of general sites)
  std::vector<int32_t> slot_site;
  for (int p = 0; p < n_passes; ++p) {
    PassHost& P = ph[p];
    P.n_slots = 0;
    for (HostOp& o : per_pass[p])
      if (o.general) { o.d.slot = P.n_slots++; slot_site.push_back(o.d.ref); }
    P.slot_begin = (int)slot_site.size() - P.n_slots;
  }
  h->any_general = !slot_site.empty();
  h->tsum_ok = false;
  // register phases of GB tile bits (4 for the generic kernel; 5 for c64 codegen)
  std::vector<DevOp> dops;
  std::vector<DevPhase> dph;
  // GB = 0: per pass, 5-bit phases iff they need fewer phases than 4-bit ones and
  // the 4-bit plan has >= 3 phases (PTSBE_GB5_MIN_PHASES; fewer shared-memory round
  // trips: bench config 4 went 1.00 M -> 1.05 M shots/s, and with the bank-conflict
  // swizzle model the 3-phase light passes stopped losing); otherwise 4.  A 5-bit
  // group doubles the registers per thread and halves the threads (128 per CTA),
  // which loses when it saves no phase.
  auto plan_all = [&](int GB) {
    dops.clear();
    dph.clear();
    for (int p = 0; p < n_passes; ++p) {
      PassHost& P = ph[p];
      P.op_begin = (int)dops.size();
      P.phase_begin = (int)dph.size();
      P.gb = GB ? GB : 4;
      if (P.L >= P.gb) {
        std::vector<DevOp> pops;
        std::vector<DevPhase> pphs;
        plan_phases(per_pass[p], P.L, pops, pphs, P.gb);
        if (GB == 0 && P.L >= 5 + 3) {
          std::vector<DevOp> pops5;
          std::vector<DevPhase> pphs5;
          plan_phases(per_pass[p], P.L, pops5, pphs5, 5);
          static const size_t min4 = std::getenv("PTSBE_GB5_MIN_PHASES") ? std::atoi(std::getenv("PTSBE_GB5_MIN_PHASES")) : 3;
          if (pphs5.size() < pphs.size() && pphs.size() >= min4) {
            pops.swap(pops5);
            pphs.swap(pphs5);
            P.gb = 5;
          }
        }
        dops.insert(dops.end(), pops.begin(), pops.end());
        dph.insert(dph.end(), pphs.begin(), pphs.end());
        P.n_phases = (int)pphs.size();
      } else {
        for (HostOp& o : per_pass[p]) dops.push_back(o.d);
        P.n_phases = 0;
      }
      P.n_ops = (int)dops.size() - P.op_begin;
    }
  };
  // circuit-specialised kernels: PTSBE_CODEGEN=1 forces, =0 disables, default for n >= 16
  const char* cg_env = std::getenv("PTSBE_CODEGEN");
  const int cg_mode = cg_env ? std::atoi(cg_env) : -1;
  bool cg_want = n_passes > 0 && (cg_mode == 1 || (cg_mode < 0 && h->n >= 16));
  const char* gb_env = std::getenv("PTSBE_PHASE_BITS");   // tuning override: 4, 5, or 0 = per pass
  const int cg_gb = gb_env ? std::max(0, std::min(5, std::atoi(gb_env))) : (h->dtype == PTSBE_C64 ? 0 : 4);
  for (auto& P : ph) cg_want = cg_want && P.L >= (cg_gb ? cg_gb : 4) + 3;
  h->phase_bits = cg_want ? cg_gb : 4;
  plan_all(h->phase_bits);
  for (int p = 0; p < n_passes; ++p) {
    const size_t smem = pass_smem(ph[p], h->amp_bytes);
    if (smem > 227 * 1024) return fail(h, PTSBE_ERR_VALIDATION, "pass %d needs %zu B shared memory", p, smem);
  }
  std::vector<int32_t> kinds(std::max(n_mats, 1), MK_GEN1);
  for (int m = 0; m < n_mats; ++m) kinds[m] = classify_matrix(mats + (size_t)m * 32, mat_arity[m] ? mat_arity[m] : 2);
  h->gen_active = false;
  h->gen_note.clear();
  if (h->host_only) {   // plan + generate only (the generic kernel needs no source)
    h->gen_src = cg_want ? gen_source(h, ph, dops, dph, mats, kinds, chans, site_chan) : std::string();
    return 0;
  }
  if (cg_want) {
    if (int r = try_codegen(h, cg_mode, ph, dops, dph, mats, kinds, chans, site_chan)) return r;
    if (!h->gen_active && h->phase_bits != 4) {   // generic kernel: 4-bit phases everywhere
      h->phase_bits = 4;
      plan_all(4);
    }
  }
  // device tables
  if (dalloc(h, &h->d_ops, std::max<size_t>(dops.size(), 1))) return PTSBE_ERR_CUDA;
  if (!dops.empty()) CK(h, cudaMemcpy(h->d_ops, dops.data(), dops.size() * sizeof(DevOp), cudaMemcpyHostToDevice));
  if (dalloc(h, &h->d_phases, std::max<size_t>(dph.size(), 1))) return PTSBE_ERR_CUDA;
  if (!dph.empty()) CK(h, cudaMemcpy(h->d_phases, dph.data(), dph.size() * sizeof(DevPhase), cudaMemcpyHostToDevice));
  if (dalloc(h, &h->d_matkind, kinds.size())) return PTSBE_ERR_CUDA;
  CK(h, cudaMemcpy(h->d_matkind, kinds.data(), kinds.size() * 4, cudaMemcpyHostToDevice));
  {
    const size_t nm = std::max(n_mats, 1);
    if (h->dtype == PTSBE_C64) {
      std::vector<float> f(nm * 32, 0.f);
      for (size_t i = 0; i < (size_t)n_mats * 32; ++i) f[i] = (float)mats[i];
      float* d = nullptr;
      if (dalloc(h, &d, f.size())) return PTSBE_ERR_CUDA;
      if (h->d_mats) cudaFree(h->d_mats);
      h->d_mats = d;
      CK(h, cudaMemcpy(d, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    } else {
      double* d = nullptr;
      if (dalloc(h, &d, nm * 32)) return PTSBE_ERR_CUDA;
      if (h->d_mats) cudaFree(h->d_mats);
      h->d_mats = d;
      if (n_mats) CK(h, cudaMemcpy(d, mats, (size_t)n_mats * 32 * 8, cudaMemcpyHostToDevice));
    }
  }
  std::vector<DevChan> dch(std::max(n_chans, 1));
  for (int k = 0; k < n_chans; ++k)
    dch[k] = DevChan{chans[k].n_outcomes, chans[k].mat_base, chans[k].general, chans[k].arity, chans[k].identity_mask};
  if (dalloc(h, &h->d_chans, dch.size())) return PTSBE_ERR_CUDA;
  CK(h, cudaMemcpy(h->d_chans, dch.data(), dch.size() * sizeof(DevChan), cudaMemcpyHostToDevice));
  if (dalloc(h, &h->d_site_chan, std::max(n_sites, 1))) return PTSBE_ERR_CUDA;
  if (n_sites) CK(h, cudaMemcpy(h->d_site_chan, site_chan, n_sites * 4, cudaMemcpyHostToDevice));
  if (dalloc(h, &h->d_slot_site, std::max<size_t>(slot_site.size(), 1))) return PTSBE_ERR_CUDA;
  if (!slot_site.empty())
    CK(h, cudaMemcpy(h->d_slot_site, slot_site.data(), slot_site.size() * 4, cudaMemcpyHostToDevice));
  if (dalloc(h, &h->d_sel, (size_t)(h->cap + 1) * std::max(n_sites, 1))) return PTSBE_ERR_CUDA;
  CK(h, cudaMemset(h->d_sel, 0, (size_t)(h->cap + 1) * std::max(n_sites, 1)));   // trunk row: all defaults
  size_t need = 1;
  for (auto& P : ph)
    if (P.n_slots) need = std::max(need, (size_t)P.n_slots * (h->cap + 1) * ((size_t)1 << (h->n - P.L)));
  if (need > h->partial_cap) {
    if (dalloc(h, &h->d_partials, need)) return PTSBE_ERR_CUDA;
    h->partial_cap = need;
  }
  size_t need_ss = 1;
  for (auto& P : ph) need_ss = std::max(need_ss, (size_t)P.n_slots * (h->cap + 1));
  if (need_ss > h->slotsum_cap) {
    if (dalloc(h, &h->d_slotsum, need_ss)) return PTSBE_ERR_CUDA;
    h->slotsum_cap = need_ss;
  }
  h->pending_pass = -1;
  const int max_smem = 227 * 1024;
  if (h->dtype == PTSBE_C64)
    CK(h, cudaFuncSetAttribute(pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
  else
    CK(h, cudaFuncSetAttribute(pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
  {
    std::vector<double> m64((size_t)std::max(n_mats, 1) * 32, 0.0);
    if (n_mats) std::memcpy(m64.data(), mats, (size_t)n_mats * 32 * 8);
    if (dalloc(h, &h->d_mats64, m64.size())) return PTSBE_ERR_CUDA;
    CK(h, cudaMemcpy(h->d_mats64, m64.data(), m64.size() * 8, cudaMemcpyHostToDevice));
  }
  h->decide = decide;
  h->conv_ready = conv_ready;
  h->passes = ph;
  h->site_pass = site_pass_tmp;
  h->n_sites = n_sites;
  h->n_mats = n_mats;
  h->n_phases_total = (int)dph.size();
  h->loaded = true;
  return 0;
}

// The code generator's view of the planned passes.
static gen::GenProgram gen_program(ptsbe_engine* h, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                                   const std::vector<DevPhase>& dph, const double* mats,
                                   const std::vector<int32_t>& kinds, const ptsbe_channel* chans,
                                   const int32_t* site_chan) {
  gen::GenProgram G;
  G.c64 = h->dtype == PTSBE_C64;
  G.n = h->n;
  G.mats = mats;
  G.kinds = kinds.data();
  G.chans = chans;
  G.site_chan = site_chan;
  G.tma = h->host_only || h->tmap_ok;
  for (const PassHost& P : ph) {
    gen::GenPass gp;
    gp.L = P.L;
    gp.c = P.c;
    gp.qmask = P.qmask;
    gp.gb = P.gb;
    gp.phases.assign(dph.begin() + P.phase_begin, dph.begin() + P.phase_begin + P.n_phases);
    gp.ops.assign(dops.begin() + P.op_begin, dops.begin() + P.op_begin + P.n_ops);
    G.passes.push_back(gp);
  }
  return G;
}

// Source of the circuit-specialised kernels (codegen.h) for the planned passes.
static std::string gen_source(ptsbe_engine* h, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                              const std::vector<DevPhase>& dph, const double* mats, const std::vector<int32_t>& kinds,
                              const ptsbe_channel* chans, const int32_t* site_chan) {
  return gen::generate(gen_program(h, ph, dops, dph, mats, kinds, chans, site_chan));
}

// Generate + compile the circuit-specialised kernels (codegen.h).
static int try_codegen(ptsbe_engine* h, int mode, const std::vector<PassHost>& ph, const std::vector<DevOp>& dops,
                       const std::vector<DevPhase>& dph, const double* mats, const std::vector<int32_t>& kinds,
                       const ptsbe_channel* chans, const int32_t* site_chan) {
  const std::string src = gen_source(h, ph, dops, dph, mats, kinds, chans, site_chan);
  if (const char* dump = std::getenv("PTSBE_CODEGEN_DUMP")) {
    if (FILE* f = std::fopen(dump, "w")) { std::fputs(src.c_str(), f); std::fclose(f); }
  }
  std::string err;
  if (gen::compile(src, (int)ph.size(), h->dev, h->gen_mod, err)) {
    h->gen_active = true;
  } else {
    h->gen_note = err;
    if (mode == 1) return fail(h, PTSBE_ERR_CUDA, "codegen: %s", err.c_str());
  }
  return 0;
}

int ptsbe_run_batch(ptsbe_engine* h, const uint8_t* sel, int B, double* out_weight, int32_t* out_status,
                    uint32_t flags) {
  return run_common(h, sel, B, out_weight, out_status, flags, true);
}

int ptsbe_apply_program(ptsbe_engine* h, const uint8_t* sel, int B, double* out_weight, int32_t* out_status,
                        uint32_t flags) {
  return run_common(h, sel, B, out_weight, out_status, flags, false);
}

int ptsbe_run_range(ptsbe_engine* h, const uint8_t* sel, int B, int pass_begin, int pass_end, double* out_weight,
                    int32_t* out_status, uint32_t flags) {
  return run_common(h, sel, B, out_weight, out_status, flags, pass_begin == 0 && !(flags & PTSBE_CONTINUE),
                    pass_begin, pass_end);
}

// Conventional trajectories: outcomes of general-channel sites chosen on device.
int ptsbe_run_conventional(ptsbe_engine* h, const uint8_t* sel, const double* u, int B, uint8_t* out_sel,
                           double* out_weight, int32_t* out_status, double* out_probs, uint32_t flags) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (!h->loaded) return fail(h, PTSBE_ERR_VALIDATION, "no program loaded");
  if (B < 0 || B > h->cap) return fail(h, PTSBE_ERR_VALIDATION, "batch %d exceeds capacity %d", B, h->cap);
  if (!h->conv_ready)
    return fail(h, PTSBE_ERR_VALIDATION,
                "program not planned for state-dependent selection (a general site does not open its pass)");
  if (B == 0) return 0;
  NvtxRange nvtx_conv("ptsbe_run_conventional");
  const int P = (int)h->passes.size();
  const int S = h->n_sites;
  std::vector<int> cuts;   // passes opened by a decision site
  for (int p = 0; p < P; ++p)
    if (h->decide[p].site >= 0) cuts.push_back(p);
  if (!cuts.empty() && !u) return fail(h, PTSBE_ERR_VALIDATION, "uniform table is required");
  CK(h, cudaSetDevice(h->dev));
  if (!cuts.empty()) {
    const size_t nu = (size_t)B * S;
    if (nu > h->u_cap) {
      if (dalloc(h, &h->d_u, nu)) return PTSBE_ERR_CUDA;
      h->u_cap = nu;
    }
    if (int r = copy_in(h, h->d_u, u, nu * 8, flags)) return r;
  }
  // the selection table is rewritten on device: the first range must not use the trunk schedule
  const bool tree_save = h->tree_enabled;
  h->tree_enabled = cuts.empty() && tree_save;
  const uint32_t f0 = flags | PTSBE_NO_SYNC;
  const uint64_t per = 1ull << h->n;
  const int nblk = (int)std::max<uint64_t>(1, std::min<uint64_t>((per / 2 + 255) / 256,
                                                                  (uint64_t)std::max(1, 4 * h->num_sms / B)));
  if ((size_t)B * nblk * kRdmVals > h->rdm_cap) {
    if (dalloc(h, &h->d_rdm, (size_t)B * nblk * kRdmVals)) { h->tree_enabled = tree_save; return PTSBE_ERR_CUDA; }
    h->rdm_cap = (size_t)B * nblk * kRdmVals;
  }
  double* d_probs = nullptr;
  if (out_probs && !cuts.empty()) CK(h, cudaMallocAsync((void**)&d_probs, (size_t)B * 64 * 8 * cuts.size(), h->stream));
  int r = 0;
  int cur = 0;
  bool started = false;
  auto decide_at = [&](int p, int idx) -> int {
    const ptsbe_engine::Decision& d = h->decide[p];
    dim3 g((unsigned)nblk, (unsigned)B);
    if (h->dtype == PTSBE_C64) {
      if (d.arity == 1) site_rdm_partials<float, 1><<<g, 256, 0, h->stream>>>(h->states, h->n, d.p0, -1, h->d_status, h->d_rdm, nblk);
      else site_rdm_partials<float, 2><<<g, 256, 0, h->stream>>>(h->states, h->n, d.p0, d.p1, h->d_status, h->d_rdm, nblk);
    } else {
      if (d.arity == 1) site_rdm_partials<double, 1><<<g, 256, 0, h->stream>>>(h->states, h->n, d.p0, -1, h->d_status, h->d_rdm, nblk);
      else site_rdm_partials<double, 2><<<g, 256, 0, h->stream>>>(h->states, h->n, d.p0, d.p1, h->d_status, h->d_rdm, nblk);
    }
    CKL(h);
    site_select<<<B, 128, 0, h->stream>>>(h->d_rdm, nblk, d.arity, h->d_mats64, d.mat_base, d.n_out, h->d_u, S,
                                           d.site, h->d_sel, h->d_status,
                                           d_probs ? d_probs + (size_t)idx * B * 64 : nullptr);
    CKL(h);
    return 0;
  };
  for (size_t i = 0; i < cuts.size() && !r; ++i) {
    const int p = cuts[i];
    if (p == 0) {   // the circuit opens with a decision: start from |0...0> explicitly
      if ((r = run_common(h, sel, B, nullptr, nullptr, f0, true, 0, 0))) break;
      if (h->dtype == PTSBE_C64) init_zero_kernel<float><<<1184, 256, 0, h->stream>>>(h->states, h->n, B, 0);
      else init_zero_kernel<double><<<1184, 256, 0, h->stream>>>(h->states, h->n, B, 0);
      CKL(h);
      h->final_general = false;
    } else if (!started) {
      if ((r = run_common(h, sel, B, nullptr, nullptr, f0, true, 0, p))) break;
    } else {
      if ((r = run_common(h, nullptr, B, nullptr, nullptr, f0 | PTSBE_KEEP_SEL, false, cur, p))) break;
    }
    started = true;
    cur = p;
    r = decide_at(p, (int)i);
  }
  if (!r) {
    if (!started) r = run_common(h, sel, B, nullptr, nullptr, f0, true, 0, P);
    else if (cur < P) r = run_common(h, nullptr, B, nullptr, nullptr, f0 | PTSBE_KEEP_SEL, false, cur, P);
  }
  h->tree_enabled = tree_save;
  if (r) { if (d_probs) cudaFreeAsync(d_probs, h->stream); return r; }
  if (out_weight) if (int e = copy_out(h, out_weight, h->d_weight, (size_t)B * 8, flags)) return e;
  if (out_status) if (int e = copy_out(h, out_status, h->d_status, (size_t)B * 4, flags)) return e;
  if (out_sel && S) if (int e = copy_out(h, out_sel, h->d_sel, (size_t)B * S, flags)) return e;
  if (d_probs) {
    int e = copy_out(h, out_probs, d_probs, (size_t)B * 64 * 8 * cuts.size(), flags);
    cudaFreeAsync(d_probs, h->stream);
    if (e) return e;
  }
  if (!(flags & PTSBE_NO_SYNC) || !(flags & PTSBE_DEVICE_PTRS)) CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ptsbe_exchange_half(ptsbe_engine* h, int b, int bit, int value, void* buf, int unpack) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (b < 0 || b >= h->cap || bit < 0 || bit >= h->n || (value & ~1) || !buf)
    return fail(h, PTSBE_ERR_VALIDATION, "bad exchange arguments (state %d, bit %d, value %d)", b, bit, value);
  CK(h, cudaSetDevice(h->dev));
  if (h->permuted) return fail(h, PTSBE_ERR_VALIDATION, "sharded exchange needs an unpermuted engine layout");
  if (unpack) h->tsum_ok = false;
  const size_t per = ((size_t)1 << h->n);
  const unsigned g = (unsigned)std::min<size_t>(per / 512 + 1, 8192);
  if (h->dtype == PTSBE_C64) {
    float2* st = reinterpret_cast<float2*>(h->states) + (size_t)b * per;
    pack_half<float2><<<g, 256, 0, h->stream>>>(st, reinterpret_cast<float2*>(buf), h->n, bit, value, unpack);
  } else {
    double2* st = reinterpret_cast<double2*>(h->states) + (size_t)b * per;
    pack_half<double2><<<g, 256, 0, h->stream>>>(st, reinterpret_cast<double2*>(buf), h->n, bit, value, unpack);
  }
  CKL(h);
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ptsbe_norm_totals(ptsbe_engine* h, int B, uint64_t* out_totals) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (B < 0 || B > h->last_B) return fail(h, PTSBE_ERR_VALIDATION, "batch %d exceeds the %d prepared states", B, h->last_B);
  if (B == 0) return 0;
  CK(h, cudaSetDevice(h->dev));
  SampleParams sp{};
  sp.states = h->states;
  sp.n = h->n;
  sp.sbits = h->sbits;
  sp.nblk = h->nblk;
  sp.B = B;
  sp.nst = h->d_nst;
  sp.status = h->d_status;
  sp.bs = h->d_bs;
  sp.total = h->d_total;
  dim3 g1((unsigned)((h->nblk + 7) / 8), (unsigned)B);
  if (h->dtype == PTSBE_C64) sample_blocksum<float><<<g1, 256, 0, h->stream>>>(sp);
  else sample_blocksum<double><<<g1, 256, 0, h->stream>>>(sp);
  CKL(h);
  sample_blockscan<<<B, 1024, 0, h->stream>>>(sp);
  CKL(h);
  CK(h, cudaMemcpyAsync(out_totals, h->d_total, (size_t)B * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

// ---- state sharding (shard.cuh) --------------------------------------------------

extern "C++" {
namespace {
int part_map(ptsbe_engine* h, int nswap, const int32_t* gbits, const int32_t* lbits, int nglobal, PartMap* m,
             uint32_t* gmask) {
  if (nswap < 1 || nswap > 3 || !gbits || !lbits)
    return fail(h, PTSBE_ERR_VALIDATION, "a swap exchanges 1..3 qubit pairs, got %d", nswap);
  m->kp = nswap;
  m->lmask = 0;
  *gmask = 0;
  for (int j = 0; j < nswap; ++j) {
    if (lbits[j] < 0 || lbits[j] >= h->n || ((m->lmask >> lbits[j]) & 1) || gbits[j] < 0 || gbits[j] >= nglobal ||
        ((*gmask >> gbits[j]) & 1))
      return fail(h, PTSBE_ERR_VALIDATION, "bad swap pair %d: global bit %d, local bit %d", j, gbits[j], lbits[j]);
    m->lbit[j] = lbits[j];
    m->lmask |= 1ull << lbits[j];
    *gmask |= 1u << gbits[j];
  }
  for (int j = 0; j < nswap; ++j) m->lsort[j] = m->lbit[j];
  std::sort(m->lsort, m->lsort + nswap);
  if (h->permuted) return fail(h, PTSBE_ERR_VALIDATION, "sharded exchange needs an unpermuted engine layout");
  return 0;
}

// shard index with the swapped global bits spelling c (pair j <-> bit j of c)
inline int shard_with(int s, const int32_t* gbits, int nswap, uint32_t c) {
  for (int j = 0; j < nswap; ++j) s = (s & ~(1 << gbits[j])) | (int)(((c >> j) & 1u) << gbits[j]);
  return s;
}
inline uint32_t spelled(int s, const int32_t* gbits, int nswap) {
  uint32_t c = 0;
  for (int j = 0; j < nswap; ++j) c |= (uint32_t)((s >> gbits[j]) & 1) << j;
  return c;
}
}  // namespace
}  // extern "C++"

int ptsbe_nccl_unique_id(void* out) {
  if (!out) return PTSBE_ERR_VALIDATION;
  nccl::Api& A = nccl::api();
  if (!A.ok) return PTSBE_ERR_NCCL;
  ncclUniqueId id;
  if (A.get_unique_id(&id) != ncclSuccess) return PTSBE_ERR_NCCL;
  std::memcpy(out, &id, sizeof id);
  return 0;
}

int ptsbe_shard_init(ptsbe_engine* h, const void* nccl_id, int rank, int nranks) {
  if (!h || !nccl_id) return PTSBE_ERR_VALIDATION;
  if (nranks < 1 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
    return fail(h, PTSBE_ERR_VALIDATION, "shard group of %d ranks (rank %d): need a power of two", nranks, rank);
  nccl::Api& A = nccl::api();
  if (!A.ok) return fail(h, PTSBE_ERR_NCCL, "NCCL unavailable: %s", A.why.c_str());
  CK(h, cudaSetDevice(h->dev));
  if (h->comm) { A.comm_destroy(h->comm); h->comm = nullptr; }
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  const ncclResult_t r = A.comm_init_rank(&h->comm, nranks, id, rank);
  if (r != ncclSuccess) { h->comm = nullptr; return fail(h, PTSBE_ERR_NCCL, "ncclCommInitRank: %s", A.error_string(r)); }
  h->shard_rank = rank;
  h->shard_nranks = nranks;
  if (!h->comm_stream) CK(h, cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
  for (auto& e : h->xev)
    if (!e) CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return 0;
}

extern "C++" {
template <typename V>
static int shard_swap_impl(ptsbe_engine* h, int B, const PartMap& m, const int32_t* gbits, int nswap) {
  const int s = h->shard_rank;
  const uint32_t own = spelled(s, gbits, nswap);
  const int P = (1 << nswap) - 1;                 // parts that travel
  const uint64_t part_len = 1ull << (h->n - nswap);
  const size_t amp = sizeof(V);
  // chunk: <= 512 MiB of sends per round, double-buffered sends + receives
  uint64_t CH = std::max<uint64_t>(1, std::min<uint64_t>(part_len, (512ull << 20) / ((uint64_t)P * amp)));
  if (const char* e = std::getenv("PTSBE_SHARD_CHUNK"))   // test knob: force many chunks
    CH = std::max<uint64_t>(1, std::min<uint64_t>(CH, (uint64_t)std::atoll(e)));
  // test knob (1-rank group, one GPU): every part goes to this rank itself -- exercises
  // the pack / grouped send-recv / unpack pipeline; the state must come back unchanged
  const bool self_test = h->shard_nranks == 1 && std::getenv("PTSBE_SHARD_SELF_TEST");
  const size_t need = 4ull * P * CH * amp;
  if (need > h->xbuf_bytes) {
    if (h->xbuf) cudaFree(h->xbuf);
    h->xbuf = nullptr;
    h->xbuf_bytes = 0;
    CK(h, cudaMalloc(&h->xbuf, need));
    h->xbuf_bytes = need;
  }
  NvtxRange nvtx_swap("ptsbe_shard_swap");
  V* sendb[2] = {(V*)h->xbuf, (V*)h->xbuf + (size_t)P * CH};
  V* recvb[2] = {(V*)h->xbuf + 2ull * P * CH, (V*)h->xbuf + 3ull * P * CH};
  nccl::Api& A = nccl::api();
  const uint64_t nch = (part_len + CH - 1) / CH;
  const long long iters = (long long)B * (long long)nch;
  const unsigned grid = (unsigned)std::min<uint64_t>((CH + 255) / 256, 4u * (unsigned)h->num_sms);
  auto region = [&](long long it, int b) {
    V* st = reinterpret_cast<V*>(h->states) + ((size_t)b << h->n);
    return st;
  };
  auto pack = [&](long long it) -> int {
    const int b = (int)(it / (long long)nch);
    const uint64_t j0 = (uint64_t)(it % (long long)nch) * CH, len = std::min<uint64_t>(CH, part_len - j0);
    int slot = 0;
    for (uint32_t c = 0; c <= (uint32_t)P; ++c) {
      if (c == own) continue;
      part_copy<V><<<grid, 256, 0, h->stream>>>(region(it, b), sendb[it & 1] + (size_t)slot * CH, m, c, j0, len, 0);
      CKL(h);
      ++slot;
    }
    CK(h, cudaEventRecord(h->xev[it & 1], h->stream));              // packed
    CK(h, cudaStreamWaitEvent(h->comm_stream, h->xev[it & 1], 0));
    ncclResult_t r = A.group_start();
    slot = 0;
    for (uint32_t c = 0; c <= (uint32_t)P && r == ncclSuccess; ++c) {
      if (c == own) continue;
      const int peer = self_test ? s : shard_with(s, gbits, nswap, c);
      r = A.send(sendb[it & 1] + (size_t)slot * CH, (size_t)len * amp, ncclInt8, peer, h->comm, h->comm_stream);
      if (r == ncclSuccess)
        r = A.recv(recvb[it & 1] + (size_t)slot * CH, (size_t)len * amp, ncclInt8, peer, h->comm, h->comm_stream);
      ++slot;
    }
    const ncclResult_t r2 = A.group_end();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return fail(h, PTSBE_ERR_NCCL, "ncclSend/ncclRecv: %s", A.error_string(r != ncclSuccess ? r : r2));
    CK(h, cudaEventRecord(h->xev[2 + (it & 1)], h->comm_stream));    // received
    return 0;
  };
  auto unpack = [&](long long it) -> int {
    const int b = (int)(it / (long long)nch);
    const uint64_t j0 = (uint64_t)(it % (long long)nch) * CH, len = std::min<uint64_t>(CH, part_len - j0);
    CK(h, cudaStreamWaitEvent(h->stream, h->xev[2 + (it & 1)], 0));
    int slot = 0;
    for (uint32_t c = 0; c <= (uint32_t)P; ++c) {
      if (c == own) continue;
      part_copy<V><<<grid, 256, 0, h->stream>>>(region(it, b), recvb[it & 1] + (size_t)slot * CH, m, c, j0, len, 1);
      CKL(h);
      ++slot;
    }
    return 0;
  };
  // pack(i+1) overlaps the transfer of chunk i; buffers of i+1 were freed when unpack(i-1)
  // waited for their transfer
  for (long long it = 0; it < iters; ++it) {
    if (int r = pack(it)) return r;
    if (it > 0)
      if (int r = unpack(it - 1)) return r;
  }
  if (iters > 0)
    if (int r = unpack(iters - 1)) return r;
  h->tsum_ok = false;
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}
}  // extern "C++"

int ptsbe_shard_swap(ptsbe_engine* h, int B, int nswap, const int32_t* gbits, const int32_t* lbits) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (!h->comm) return fail(h, PTSBE_ERR_VALIDATION, "no shard group: call ptsbe_shard_init first");
  if (B < 1 || B > h->cap) return fail(h, PTSBE_ERR_VALIDATION, "batch %d outside [1, %d]", B, h->cap);
  int nglobal = 0;
  while ((1 << nglobal) < h->shard_nranks) ++nglobal;
  if (h->shard_nranks == 1 && std::getenv("PTSBE_SHARD_SELF_TEST")) nglobal = 3;
  PartMap m;
  uint32_t gmask = 0;
  if (int r = part_map(h, nswap, gbits, lbits, nglobal, &m, &gmask)) return r;
  CK(h, cudaSetDevice(h->dev));
  return h->dtype == PTSBE_C64 ? shard_swap_impl<float2>(h, B, m, gbits, nswap)
                               : shard_swap_impl<double2>(h, B, m, gbits, nswap);
}

int ptsbe_shard_swap_local(ptsbe_engine* const* hs, int D, int B, int nswap, const int32_t* gbits,
                           const int32_t* lbits) {
  if (!hs || D < 2 || (D & (D - 1))) return PTSBE_ERR_VALIDATION;
  ptsbe_engine* h0 = hs[0];
  if (!h0) return PTSBE_ERR_VALIDATION;
  int nglobal = 0;
  while ((1 << nglobal) < D) ++nglobal;
  PartMap m;
  uint32_t gmask = 0;
  if (int r = part_map(h0, nswap, gbits, lbits, nglobal, &m, &gmask)) return r;
  for (int s = 0; s < D; ++s) {
    if (!hs[s] || hs[s]->dev != h0->dev || hs[s]->n != h0->n || hs[s]->dtype != h0->dtype || hs[s]->permuted)
      return fail(h0, PTSBE_ERR_VALIDATION, "shard %d: engines must share device, width, dtype and layout", s);
    if (B < 1 || B > hs[s]->cap) return fail(h0, PTSBE_ERR_VALIDATION, "batch %d exceeds shard %d", B, s);
  }
  CK(h0, cudaSetDevice(h0->dev));
  for (int s = 0; s < D; ++s) CK(h0, cudaStreamSynchronize(hs[s]->stream));
  const uint64_t part_len = 1ull << (h0->n - nswap);
  const unsigned grid = (unsigned)std::min<uint64_t>((part_len + 255) / 256, 8u * (unsigned)h0->num_sms);
  for (int s = 0; s < D; ++s) {
    const uint32_t own = spelled(s, gbits, nswap);
    for (uint32_t c = 0; c < (1u << nswap); ++c) {
      const int peer = shard_with(s, gbits, nswap, c);
      if (c == own || peer < s) continue;                // each pair once
      for (int b = 0; b < B; ++b) {
        if (h0->dtype == PTSBE_C64) {
          float2* a = reinterpret_cast<float2*>(hs[s]->states) + ((size_t)b << h0->n);
          float2* q = reinterpret_cast<float2*>(hs[peer]->states) + ((size_t)b << h0->n);
          part_swap<float2><<<grid, 256, 0, h0->stream>>>(a, q, m, c, own, part_len);
        } else {
          double2* a = reinterpret_cast<double2*>(hs[s]->states) + ((size_t)b << h0->n);
          double2* q = reinterpret_cast<double2*>(hs[peer]->states) + ((size_t)b << h0->n);
          part_swap<double2><<<grid, 256, 0, h0->stream>>>(a, q, m, c, own, part_len);
        }
        CKL(h0);
      }
    }
  }
  CK(h0, cudaStreamSynchronize(h0->stream));
  for (int s = 0; s < D; ++s) hs[s]->tsum_ok = false;
  return 0;
}

int ptsbe_slot_norms(ptsbe_engine* h, int B, double* out, int* out_slots) {
  if (!h || !out || !out_slots) return PTSBE_ERR_VALIDATION;
  if (h->pending_pass < 0) return fail(h, PTSBE_ERR_VALIDATION, "no pass waits for its norms");
  if (B != h->last_B) return fail(h, PTSBE_ERR_VALIDATION, "batch %d, the pending pass ran %d", B, h->last_B);
  const int ns = h->passes[h->pending_pass].n_slots;
  const int Bst = h->cap + 1;
  CK(h, cudaSetDevice(h->dev));
  for (int j = 0; j < ns; ++j)
    CK(h, cudaMemcpyAsync(out + (size_t)j * B, h->d_slotsum + (size_t)j * Bst, (size_t)B * 8, cudaMemcpyDeviceToHost,
                          h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  *out_slots = ns;
  return 0;
}

int ptsbe_finalize_norms(ptsbe_engine* h, int B, const double* sums) {
  if (!h || !sums) return PTSBE_ERR_VALIDATION;
  if (h->pending_pass < 0) return fail(h, PTSBE_ERR_VALIDATION, "no pass waits for its norms");
  if (B != h->last_B) return fail(h, PTSBE_ERR_VALIDATION, "batch %d, the pending pass ran %d", B, h->last_B);
  const PassHost& ph = h->passes[h->pending_pass];
  const int Bst = h->cap + 1;
  CK(h, cudaSetDevice(h->dev));
  for (int j = 0; j < ph.n_slots; ++j)
    CK(h, cudaMemcpyAsync(h->d_slotsum + (size_t)j * Bst, sums + (size_t)j * B, (size_t)B * 8, cudaMemcpyHostToDevice,
                          h->stream));
  norm_finalize_sums<<<(h->pending_E + 127) / 128, 128, 0, h->stream>>>(
      h->d_slotsum, ph.n_slots, Bst, h->d_slot_site + ph.slot_begin, h->d_nst, h->d_weight, h->d_status, h->d_fail,
      h->d_ent + h->pending_ent, h->pending_E);
  CKL(h);
  h->pending_pass = -1;
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ptsbe_set_host_mirror(ptsbe_engine* h, const uint8_t* sel, const int64_t* shots, int B) {
  if (!h || B < 0) return PTSBE_ERR_VALIDATION;
  h->mirror_sel = sel;
  h->mirror_shots = shots;
  h->mirror_B = B;
  return 0;
}

int ptsbe_get_weights(ptsbe_engine* h, int B, double* out_weight, int32_t* out_status) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (B < 0 || B > h->cap) return fail(h, PTSBE_ERR_VALIDATION, "batch %d exceeds capacity %d", B, h->cap);
  CK(h, cudaSetDevice(h->dev));
  if (out_weight) CK(h, cudaMemcpyAsync(out_weight, h->d_weight, (size_t)B * 8, cudaMemcpyDeviceToHost, h->stream));
  if (out_status) CK(h, cudaMemcpyAsync(out_status, h->d_status, (size_t)B * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ptsbe_gather_amplitudes(ptsbe_engine* h, int b, const uint64_t* idx, int64_t count, void* out) {
  if (!h || (count > 0 && (!idx || !out))) return PTSBE_ERR_VALIDATION;
  if (b < 0 || b >= h->cap) return fail(h, PTSBE_ERR_VALIDATION, "state %d out of range", b);
  if (count <= 0) return 0;
  const uint64_t nmask = (1ull << h->n) - 1;
  for (int64_t i = 0; i < count; ++i)
    if (idx[i] & ~nmask) return fail(h, PTSBE_ERR_VALIDATION, "index %llu outside 2^%d", (unsigned long long)idx[i], h->n);
  CK(h, cudaSetDevice(h->dev));
  int r = h->dtype == PTSBE_C64 ? rescale_if_needed<float>(h) : rescale_if_needed<double>(h);
  if (r) return r;
  uint64_t* d_idx = nullptr;
  void* d_out = nullptr;
  CK(h, cudaMallocAsync((void**)&d_idx, (size_t)count * 8, h->stream));
  CK(h, cudaMallocAsync(&d_out, (size_t)count * h->amp_bytes, h->stream));
  CK(h, cudaMemcpyAsync(d_idx, idx, (size_t)count * 8, cudaMemcpyHostToDevice, h->stream));
  const unsigned g = (unsigned)std::min<int64_t>((count + 255) / 256, 4096);
  const size_t off = (size_t)b << h->n;
  if (h->dtype == PTSBE_C64)
    gather_amps<float2><<<g, 256, 0, h->stream>>>(reinterpret_cast<const float2*>(h->states) + off, d_idx, count,
                                                  reinterpret_cast<float2*>(d_out));
  else
    gather_amps<double2><<<g, 256, 0, h->stream>>>(reinterpret_cast<const double2*>(h->states) + off, d_idx, count,
                                                   reinterpret_cast<double2*>(d_out));
  CKL(h);
  CK(h, cudaMemcpyAsync(out, d_out, (size_t)count * h->amp_bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaFreeAsync(d_idx, h->stream));
  CK(h, cudaFreeAsync(d_out, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

void* ptsbe_state_ptr(ptsbe_engine* h, int b) {
  if (!h || b < 0 || b >= h->cap) return nullptr;
  return (char*)h->states + (size_t)b * ((size_t)1 << h->n) * h->amp_bytes;
}

int ptsbe_sample(ptsbe_engine* h, int B, const int64_t* shots, int rng_mode, const uint64_t* rng_state,
                 const uint64_t* keys, uint64_t* out_idx, uint32_t* out_cnt, int64_t* out_nuniq, uint32_t flags) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (B < 0 || B > h->last_B) return fail(h, PTSBE_ERR_VALIDATION, "batch %d exceeds the %d prepared states", B, h->last_B);
  if (B == 0) return 0;
  CK(h, cudaSetDevice(h->dev));
  return h->dtype == PTSBE_C64
             ? sample_impl<float>(h, B, shots, rng_mode, rng_state, keys, out_idx, out_cnt, out_nuniq, flags)
             : sample_impl<double>(h, B, shots, rng_mode, rng_state, keys, out_idx, out_cnt, out_nuniq, flags);
}

int ptsbe_get_state(ptsbe_engine* h, int b, void* buf, uint32_t flags) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (b < 0 || b >= h->cap) return fail(h, PTSBE_ERR_VALIDATION, "state %d out of range", b);
  CK(h, cudaSetDevice(h->dev));
  int r = h->dtype == PTSBE_C64 ? rescale_if_needed<float>(h) : rescale_if_needed<double>(h);
  if (r) return r;
  const size_t bytes = ((size_t)1 << h->n) * h->amp_bytes;
  const char* src = (char*)h->states + (size_t)b * bytes;
  void* scratch = nullptr;
  if (h->permuted && !h->logical[b]) {   // logical order for the caller
    scratch = state_scratch(h);
    if (!scratch) return fail(h, PTSBE_ERR_CUDA, "cannot allocate %zu bytes of relayout scratch", bytes);
    if (int r = h->dtype == PTSBE_C64
                    ? permute_into<float2>(h, (const float2*)src, (float2*)scratch, h->layout)
                    : permute_into<double2>(h, (const double2*)src, (double2*)scratch, h->layout))
      return r;
    src = (const char*)scratch;
  }
  int e = copy_out(h, buf, src, bytes, flags);
  if (e) return e;
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

int ptsbe_set_state(ptsbe_engine* h, int b, const void* buf, uint32_t flags) {
  if (!h) return PTSBE_ERR_VALIDATION;
  if (b < 0 || b >= h->cap) return fail(h, PTSBE_ERR_VALIDATION, "state %d out of range", b);
  CK(h, cudaSetDevice(h->dev));
  const size_t bytes = ((size_t)1 << h->n) * h->amp_bytes;
  char* dst = (char*)h->states + (size_t)b * bytes;
  h->logical[b] = 0;
  if (h->permuted) {   // caller gives logical order; store physical
    void* scratch = state_scratch(h);
    if (!scratch) return fail(h, PTSBE_ERR_CUDA, "cannot allocate %zu bytes of relayout scratch", bytes);
    if (int e = copy_in(h, scratch, buf, bytes, flags)) return e;
    BitPerm fwd;     // physical bit perm[q] <- logical bit q
    fwd.n = h->n;
    for (int q = 0; q < h->n; ++q) fwd.src[h->layout.src[q]] = (int8_t)q;
    if (int r = h->dtype == PTSBE_C64 ? permute_into<float2>(h, (const float2*)scratch, (float2*)dst, fwd)
                                      : permute_into<double2>(h, (const double2*)scratch, (double2*)dst, fwd))
      return r;
  } else if (int e = copy_in(h, dst, buf, bytes, flags)) {
    return e;
  }
  const double one = 1.0;
  const int32_t zero = 0;
  CK(h, cudaMemcpyAsync(h->d_nst + b, &one, 8, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(h->d_status + b, &zero, 4, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  h->last_B = std::max(h->last_B, b + 1);
  h->final_general = false;
  h->tsum_ok = false;
  return 0;
}

int ptsbe_set_layout(ptsbe_engine* h, const int32_t* perm) {
  if (!h) return PTSBE_ERR_VALIDATION;
  h->permuted = false;
  h->layout.n = h->n;
  for (int q = 0; q < h->n; ++q) h->layout.src[q] = (int8_t)q;
  std::fill(h->logical.begin(), h->logical.end(), 0);
  if (!perm) return 0;
  uint64_t seen = 0;
  for (int q = 0; q < h->n; ++q) {
    if (perm[q] < 0 || perm[q] >= h->n || ((seen >> perm[q]) & 1))
      return fail(h, PTSBE_ERR_VALIDATION, "layout is not a permutation of %d qubits", h->n);
    seen |= 1ull << perm[q];
    h->layout.src[q] = (int8_t)perm[q];
    h->permuted = h->permuted || perm[q] != q;
  }
  return 0;
}

int ptsbe_plan(int n_qubits, int n_ops, const uint64_t* target_masks, const uint8_t* general, int tile_bits,
               int low_bits, int search_iters, uint64_t seed, int32_t* perm_io, int32_t* out_pass,
               uint64_t* out_masks, int max_passes) {
  if (n_qubits < 1 || n_qubits > 63 || n_ops < 0 || tile_bits < 1 || low_bits < 0 || !perm_io)
    return -PTSBE_ERR_VALIDATION;
  std::vector<plan::Op> ops(n_ops);
  // general[i]: bit 0 = renormalising site, bit 1 = gate (counts toward the
  // optional per-pass gate budget PTSBE_MAX_PASS_GATES, a tuning knob), bit 2 =
  // decision site (first op of its pass; ptsbe_run_conventional)
  for (int i = 0; i < n_ops; ++i)
    ops[i] = plan::Op{target_masks[i], general && (general[i] & 1) != 0, general && (general[i] & 2) ? 1 : 0,
                      general && (general[i] & 4) != 0};
  const char* cap_env = std::getenv("PTSBE_MAX_PASS_GATES");
  const int cap = cap_env ? std::atoi(cap_env) : 0;
  std::vector<int> perm(perm_io, perm_io + n_qubits);
  const int L = std::min(tile_bits, n_qubits), c = std::min(low_bits, L);
  plan::search(n_qubits, ops, perm, L, c, search_iters, seed, cap);
  std::vector<int> pass;
  std::vector<uint64_t> masks;
  const int P = plan::greedy(n_qubits, ops, perm, L, c, &pass, &masks, cap);
  if (P < 0) return -PTSBE_ERR_VALIDATION;
  if (P > max_passes) return -PTSBE_ERR_VALIDATION;
  for (int q = 0; q < n_qubits; ++q) perm_io[q] = perm[q];
  if (out_pass)
    for (int i = 0; i < n_ops; ++i) out_pass[i] = pass[i];
  if (out_masks)
    for (int p = 0; p < P; ++p) out_masks[p] = masks[p];
  return P;
}

int ptsbe_device_memory(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
  if (cudaSetDevice(device) != cudaSuccess) return PTSBE_ERR_CUDA;
  size_t f = 0, t = 0;
  if (cudaMemGetInfo(&f, &t) != cudaSuccess) return PTSBE_ERR_CUDA;
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = t;
  return 0;
}

int ptsbe_synchronize(ptsbe_engine* h) {
  if (!h) return PTSBE_ERR_VALIDATION;
  CK(h, cudaStreamSynchronize(h->stream));
  return 0;
}

void* ptsbe_stream(ptsbe_engine* h) { return h ? (void*)h->stream : nullptr; }

int ptsbe_profile(ptsbe_engine* h, int enable) {
  if (!h) return PTSBE_ERR_VALIDATION;
  h->profiling = enable != 0;
  h->ev_used = 0;
  h->pass_ms_total = 0.0;
  h->pass_launches = 0;
  h->pass_bytes_total = 0.0;
  h->ev_pass.clear();
  h->ev_bytes.clear();
  h->per_pass_ms.assign(h->passes.size(), 0.0);
  h->per_pass_bytes.assign(h->passes.size(), 0.0);
  return 0;
}

int ptsbe_profile_read(ptsbe_engine* h, double* total_ms, int64_t* launches) {
  if (!h) return PTSBE_ERR_VALIDATION;
  CK(h, cudaStreamSynchronize(h->stream));
  for (int i = 0; i + 1 < h->ev_used; i += 2) {
    float ms = 0.f;
    CK(h, cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
    h->pass_ms_total += ms;
    h->pass_launches++;
    const size_t k = (size_t)(i / 2);
    if (k < h->ev_pass.size()) {
      const int p = h->ev_pass[k];
      if (p >= (int)h->per_pass_ms.size()) {
        h->per_pass_ms.resize(p + 1, 0.0);
        h->per_pass_bytes.resize(p + 1, 0.0);
      }
      h->per_pass_ms[p] += ms;
      h->per_pass_bytes[p] += h->ev_bytes[k];
    }
  }
  h->ev_used = 0;
  h->ev_pass.clear();
  h->ev_bytes.clear();
  if (total_ms) *total_ms = h->pass_ms_total;
  if (launches) *launches = h->pass_launches;
  return 0;
}

double ptsbe_profile_bytes(ptsbe_engine* h) { return h ? h->pass_bytes_total : 0.0; }

int ptsbe_profile_passes(ptsbe_engine* h, double* ms, double* bytes, int max_passes) {
  if (!h) return -PTSBE_ERR_VALIDATION;
  const int n = (int)h->per_pass_ms.size();
  for (int p = 0; p < n && p < max_passes; ++p) {
    if (ms) ms[p] = h->per_pass_ms[p];
    if (bytes) bytes[p] = h->per_pass_bytes[p];
  }
  return n;
}

int ptsbe_info(ptsbe_engine* h, int64_t* out, int n) {
  if (!h || !out) return PTSBE_ERR_VALIDATION;
  int max_tile = 0, total_slots = 0;
  for (auto& P : h->passes) { max_tile = std::max(max_tile, P.L); total_slots += P.n_slots; }
  const int64_t vals[] = {h->n, h->dtype, h->cap, (int64_t)h->passes.size(), max_tile, h->n_sites,
                          h->sbits, total_slots, h->launches, h->gen_active ? 1 : 0, h->n_phases_total};
  for (int i = 0; i < n && i < (int)(sizeof vals / sizeof vals[0]); ++i) out[i] = vals[i];
  return 0;
}

int ptsbe_last_error(ptsbe_engine* h, char* buf, size_t len) {
  if (!buf || len == 0) return PTSBE_ERR_VALIDATION;
  const std::string& s = h ? h->err : std::string("null handle");
  std::snprintf(buf, len, "%s", s.c_str());
  return 0;
}

int ptsbe_pass_info(ptsbe_engine* h, int p, int64_t* out, int n) {
  if (!h || !out) return PTSBE_ERR_VALIDATION;
  if (p < 0 || p >= (int)h->passes.size()) return fail(h, PTSBE_ERR_VALIDATION, "pass %d out of range", p);
  const PassHost& P = h->passes[p];
  const int64_t thr = h->gen_active ? gen::threads_for(P.L, P.gb, P.n_slots > 0) : std::max(32, 1 << std::max(0, P.L - 4));
  const int64_t vals[] = {P.L, P.c, P.gb, P.n_phases, P.n_ops, P.n_slots, thr, h->gen_active ? 1 : 0};
  for (int i = 0; i < n && i < (int)(sizeof vals / sizeof vals[0]); ++i) out[i] = vals[i];
  return 0;
}

int64_t ptsbe_launch_count(ptsbe_engine* h) { return h ? h->launches : 0; }

int64_t ptsbe_format_records(int n_qubits, int64_t n_traj, const int64_t* traj_ids, const int64_t* offsets,
                             const uint64_t* indices, const uint32_t* counts, char* buf, int64_t cap) {
  return ptsbe_records::format(n_qubits, n_traj, traj_ids, offsets, indices, counts, buf, cap);
}

}  // extern "C"
