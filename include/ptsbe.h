/*
 * ptsbe.h -- C ABI of libptsbe.so, the sm_100a batched-execution engine of the
 * PTSBE (pre-trajectory sampling with batched execution) hot path.
 *
 * The reference ("trajsim", /root/reference/pkg/src/trajsim) is pure Python and
 * has no FFI; each entry point below replaces one Python function of its
 * hot path (file:line in the reference):
 *
 *   ptsbe_create / ptsbe_destroy  <- statevector.init_zero          statevector.py:64-69
 *                                    (device-resident batch of 2^n-amplitude states)
 *   ptsbe_load_program            <- the op loop of prepare_state   execute.py:85-97
 *                                    (gate + fixed Kraus stream, lowered to fused passes)
 *   ptsbe_run_batch               <- prepare_state x B              execute.py:74-98
 *                                    apply_gate/apply_matrix         statevector.py:118-126
 *                                    apply_kraus_normalized          statevector.py:136-145
 *   ptsbe_sample                  <- sample_shots x B               statevector.py:148-163
 *                                    ShotBatch.from_indices          statevector.py:44-47
 *   ptsbe_get_state/ptsbe_set_state <- ComplexState.amplitudes      statevector.py:18-32
 *   ptsbe_last_error              <- exception text                 errors.py:5-25
 *
 * Conventions
 *   - Every function returns a ptsbe_status; 0 is success.  Per-trajectory
 *     annihilation is NOT a call failure: it is reported in out_status[b].
 *   - The caller owns every pointer it passes; the handle owns device memory.
 *     Pointers are HOST pointers unless PTSBE_DEVICE_PTRS is set in `flags`,
 *     in which case they are device pointers on the handle's device.
 *   - One handle per (host thread, device); a handle is not thread-safe.
 *     Work is queued on the handle's own CUDA stream (ptsbe_stream).
 *   - Basis index bit q is qubit q (statevector.py:20).  For a 2-qubit op the
 *     first-listed target is the most significant bit of the 4x4 local index
 *     (statevector.py:86, circuit.py:25-26).
 */
#ifndef PTSBE_H
#define PTSBE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTSBE_ABI_VERSION 1

typedef enum {
  PTSBE_OK = 0,
  PTSBE_ERR_VALIDATION = 1,   /* -> ValidationError   (errors.py:17)  */
  PTSBE_ERR_ANNIHILATED = 2,  /* -> AnnihilatedStateError (errors.py:25), per trajectory */
  PTSBE_ERR_CUDA = 3,         /* -> ExecutionError    (errors.py:21)  */
  PTSBE_ERR_NCCL = 4          /* -> ExecutionError                     */
} ptsbe_status;

typedef enum { PTSBE_C64 = 0, PTSBE_C128 = 1 } ptsbe_dtype;

/* trajectory status values written to out_status[] */
#define PTSBE_TRAJ_OK 0
#define PTSBE_TRAJ_ANNIHILATED 2

/* flags */
#define PTSBE_DEVICE_PTRS 0x1u  /* pointer arguments are device pointers */
#define PTSBE_ZERO_VECTOR 0x4u  /* ptsbe_run_range from pass 0: start from the all-zero vector
                                   instead of |0...0> (every shard but shard 0) */
#define PTSBE_CONTINUE    0x8u  /* ptsbe_run_range from pass 0: apply the passes to the states as
                                   they are (set_state / a previous range) instead of |0...0> */
#define PTSBE_NO_SYNC     0x2u  /* do not synchronise the stream before returning
                                   (only meaningful with PTSBE_DEVICE_PTRS) */
#define PTSBE_DEFER_NORMS 0x20u /* ptsbe_run_range of ONE pass of a shard: leave the shard-local
                                   norms of its renormalising sites for ptsbe_slot_norms /
                                   ptsbe_finalize_norms (shards of one process) */
#define PTSBE_SHARDED     0x40u /* ptsbe_run_range of a shard in an NCCL shard group
                                   (ptsbe_shard_init): norms of renormalising sites are
                                   all-reduced over the group on the engine stream */
#define PTSBE_HOST_MIRROR 0x80u /* with PTSBE_DEVICE_PTRS: the host copies registered by
                                   ptsbe_set_host_mirror stand in for reading the device outcome
                                   table / shot counts back (no device->host sync per call) */
#define PTSBE_KEEP_SEL    0x10u /* continued ptsbe_run_range: keep the device outcome table as it
                                   is (sel may be NULL) -- e.g. outcomes chosen on device */

/* rng modes of ptsbe_sample */
#define PTSBE_RNG_PCG64   0  /* numpy PCG64 stream per trajectory: rng_state[4*b..] =
                                {state_hi, state_lo, inc_hi, inc_lo}; bit-exact uniforms
                                of Generator(PCG64).random(m)  (execute.py:44-45,145-146) */
#define PTSBE_RNG_PHILOX  1  /* device Philox4x32-10, key rng_state[b] (production) */
#define PTSBE_RNG_KEYS    2  /* caller supplies the uniforms as 53-bit integers
                                u = key * 2^-53 in `keys` (concatenated per trajectory) */

/* One entry of the program's op stream (gate or noise site), in application
 * order (execute.py:85-97). */
typedef struct {
  int32_t kind;   /* 0 = gate with fixed matrix, 1 = noise site (outcome chosen per trajectory) */
  int32_t arity;  /* 1 or 2 */
  int32_t t0;     /* first-listed target qubit (MSB of local index) */
  int32_t t1;     /* second target (arity 2), else -1 */
  int32_t ref;    /* kind 0: matrix index; kind 1: site id */
  int32_t pass;   /* index of the fused HBM pass that executes this op */
} ptsbe_op;

/* A noise channel as the device sees it: outcome k uses matrix mat_base + k. */
typedef struct {
  int32_t n_outcomes;
  int32_t mat_base;
  int32_t general;        /* 1: non-unitary Kraus, renormalise + weight (statevector.py:136-145) */
  int32_t arity;
  uint64_t identity_mask; /* bit k: outcome k is exactly the identity (skipped bit-exactly) */
} ptsbe_channel;

/* A fused pass: all ops with .pass == index act inside tiles spanned by qubit_mask. */
typedef struct {
  uint64_t qubit_mask;    /* tile qubit set; must contain qubits 0..low_bits-1 */
  int32_t tile_bits;      /* popcount(qubit_mask) */
  int32_t low_bits;       /* contiguous low qubits in the set (>= 3) */
} ptsbe_pass;

typedef struct ptsbe_engine ptsbe_engine;

int ptsbe_abi_version(void);

int ptsbe_create(int device, int n_qubits, int dtype, int batch_cap, ptsbe_engine** out);
int ptsbe_destroy(ptsbe_engine* h);

/* mats: n_mats matrices, each 4x4 complex128 row-major padded (32 doubles,
 * re/im interleaved); a 1-qubit matrix is the leading 2x2 block (entries 0,1,4,5). */
int ptsbe_load_program(ptsbe_engine* h,
                       const ptsbe_op* ops, int n_ops,
                       const double* mats, int n_mats,
                       const ptsbe_channel* chans, int n_chans,
                       const int32_t* site_chan, int n_sites,
                       const ptsbe_pass* passes, int n_passes);

/* Prepare B states (B <= batch_cap).  sel[b*n_sites + s] = Kraus outcome at
 * site s (0 = default).  Writes realized weights (execute.py:97) and status. */
int ptsbe_run_batch(ptsbe_engine* h, const uint8_t* sel, int B,
                    double* out_weight, int32_t* out_status, uint32_t flags);

/* Sample shots[b] shots from each prepared state (b < B).  Output is one
 * contiguous CSR stream: trajectory b's distinct outcomes occupy entries
 * [u_b, u_b + out_nuniq[b]) of out_idx / out_cnt, u_b = sum of earlier
 * out_nuniq, ascending basis index (qubit q = bit q) with its shot count.
 * out_idx / out_cnt need room for sum(shots) entries.  rng_state / keys
 * depend on rng_mode (see above). */
int ptsbe_sample(ptsbe_engine* h, int B, const int64_t* shots, int rng_mode,
                 const uint64_t* rng_state, const uint64_t* keys,
                 uint64_t* out_idx, uint32_t* out_cnt, int64_t* out_nuniq,
                 uint32_t flags);

/* Copy state b (normalised, engine dtype, interleaved re/im) to / from `buf`. */
int ptsbe_get_state(ptsbe_engine* h, int b, void* buf, uint32_t flags);
int ptsbe_set_state(ptsbe_engine* h, int b, const void* buf, uint32_t flags);

/* Apply the loaded program to the batch states as they are (no |0> init);
 * used by the single-state inner API (apply_matrix & co). */
int ptsbe_apply_program(ptsbe_engine* h, const uint8_t* sel, int B,
                        double* out_weight, int32_t* out_status, uint32_t flags);

/* Physical layout: logical qubit q is stored at physical bit perm[q] (NULL =
 * identity).  Program ops and pass masks are given in physical qubits; shots,
 * get_state and set_state stay in logical order (indices are mapped back and
 * re-sorted on device). */
int ptsbe_set_layout(ptsbe_engine* h, const int32_t* perm);

/* Fusion planner (host only; no GPU or handle needed).  Op i acts on the
 * LOGICAL qubits in target_masks[i]; general[i] bit 0 marks renormalising
 * sites (never reordered among themselves), bit 1 gates, bit 2 decision sites
 * (ptsbe_run_conventional: the site must open its pass).  perm_io: in = starting layout,
 * out = layout after `search_iters` steps of local search minimising the pass
 * count.  Writes out_pass[i] (pass of op i, ops keep stream order within a
 * pass) and out_masks[p] (PHYSICAL tile qubit set of pass p).  Returns the
 * number of passes, or a negative status. */
int ptsbe_plan(int n_qubits, int n_ops, const uint64_t* target_masks, const uint8_t* general,
               int tile_bits, int low_bits, int search_iters, uint64_t seed,
               int32_t* perm_io, int32_t* out_pass, uint64_t* out_masks, int max_passes);

/* ---- intra-trajectory state sharding (sharded.py drives these per shard) ----
 * A shard holds the 2^n amplitudes of one global-bit pattern of a 2^(n+k)
 * state; its program covers segments of local-only ops.
 *
 * Run passes [pass_begin, pass_end) of the loaded program; pass_begin == 0
 * starts from |0...0>, otherwise the B states continue where the previous
 * range stopped (a global<->local qubit swap may have happened in between). */
int ptsbe_run_range(ptsbe_engine* h, const uint8_t* sel, int B, int pass_begin, int pass_end,
                    double* out_weight, int32_t* out_status, uint32_t flags);
/* ---- conventional trajectories (Algorithm 1) <- trajectory.py:40-70 run_trajectory,
 * :138-219 the dense ensemble of sample_conventional.  Outcomes of unitary-mixture
 * sites are state independent (select_index over the mixture's probabilities on
 * the trajectory's uniform) and arrive in `sel`; the outcome of every GENERAL-channel
 * site is chosen on device from the state just before it: the reduced density
 * matrix rho of its targets gives every branch probability p_k = ||K_k psi||^2 =
 * tr(K_k^+ K_k rho) / tr(rho) (statevector.py:129-133) in one read, then
 * k = select_index(u[b*S + site], p) (trajectory.py:27-37) is written to the outcome
 * table, and the next fused pass applies K_k with renormalisation and weight
 * (statevector.py:136-145).  The program must be planned with every general site
 * opening its pass (ptsbe_plan bit 2), else PTSBE_ERR_VALIDATION.
 * u: B x S uniforms (only general sites' columns are read).  out_sel (optional):
 * the final B x S outcome table.  out_probs (optional): for the i-th decision site
 * in program order, p_k at out_probs[(i*B + b)*64 + k]. */
int ptsbe_run_conventional(ptsbe_engine* h, const uint8_t* sel, const double* u, int B, uint8_t* out_sel,
                           double* out_weight, int32_t* out_status, double* out_probs, uint32_t flags);
/* Copy the half of state b whose local bit `bit` equals `value` to (unpack = 0)
 * or from (unpack = 1) the contiguous device buffer `buf` (2^(n-1) amplitudes):
 * the data movement of a global<->local qubit swap. */
int ptsbe_exchange_half(ptsbe_engine* h, int b, int bit, int value, void* buf, int unpack);
/* Exact 2^-62 fixed-point sum of |a|^2 of each of the first B states (the
 * sampler's CDF total), for splitting shots across shards. */
int ptsbe_norm_totals(ptsbe_engine* h, int B, uint64_t* out_totals);
/* NCCL shard group (one shard per rank, one rank per GPU; `nccl_id` = 128 bytes from
 * ptsbe_nccl_unique_id on rank 0, broadcast by the caller).  NCCL is loaded at run time. */
int ptsbe_nccl_unique_id(void* out128);
int ptsbe_shard_init(ptsbe_engine* h, const void* nccl_id, int rank, int nranks);
/* Swap global bits gbits[j] (bits of the shard index = rank) with local bits lbits[j],
 * j < nswap <= 3, for the first B states: ONE all-to-all of 2^nswap parts per group of
 * shards (grouped ncclSend/ncclRecv on a comm stream, chunked and double-buffered so
 * the part packing overlaps the transfer; persistent buffers <= 2 GiB). */
int ptsbe_shard_swap(ptsbe_engine* h, int B, int nswap, const int32_t* gbits, const int32_t* lbits);
/* The same exchange between the D = 2^k shards of ONE process on one device
 * (handles hs[s] hold shard s): pairwise in-place part swaps, no buffers. */
int ptsbe_shard_swap_local(ptsbe_engine* const* hs, int D, int B, int nswap, const int32_t* gbits,
                           const int32_t* lbits);
/* Cross-shard norms for PTSBE_DEFER_NORMS runs: shard-local norm^2 of the pending pass's
 * renormalising slots (out[j*B + b], j < *out_slots <= 64), then the caller's sums
 * over all shards finalise weights / status / stored norms on every shard. */
int ptsbe_slot_norms(ptsbe_engine* h, int B, double* out, int* out_slots);
int ptsbe_finalize_norms(ptsbe_engine* h, int B, const double* sums);
/* Host copies of the device-resident inputs of the next PTSBE_HOST_MIRROR calls (the
 * caller keeps them alive): sel[B*n_sites] for ptsbe_run_batch's scheduling, shots[B]
 * for ptsbe_sample's shot layout.  With PTSBE_DEVICE_PTRS, ptsbe_sample's CSR output
 * (out_idx / out_cnt / out_nuniq) is compacted on device; the stream is not drained. */
int ptsbe_set_host_mirror(ptsbe_engine* h, const uint8_t* sel, const int64_t* shots, int B);
/* Realized weights and status of the first B rows (after a run / finalize). */
int ptsbe_get_weights(ptsbe_engine* h, int B, double* out_weight, int32_t* out_status);
/* Amplitudes of state b at `count` PHYSICAL basis indices (normalised; verification of
 * states too large to download). */
int ptsbe_gather_amplitudes(ptsbe_engine* h, int b, const uint64_t* idx, int64_t count, void* out);
/* Device address of state b (exchange buffers, debugging). */
void* ptsbe_state_ptr(ptsbe_engine* h, int b);

/* ---- offline tooling (no GPU): a host-only handle runs ptsbe_load_program's
 * validation, pass/phase planning and kernel generation, and keeps the
 * generated CUDA source instead of compiling it (tools/gen_offline.py
 * compiles it with nvcc for SASS inspection).  Compute calls on it fail. */
int ptsbe_create_host(int n_qubits, int dtype, ptsbe_engine** out);
/* Copies up to len-1 bytes of the generated source (NUL-terminated) into buf
 * (buf may be NULL); returns the full source length. */
int64_t ptsbe_codegen_source(ptsbe_engine* h, char* buf, size_t len);

/* Misc */
int ptsbe_device_memory(int device, uint64_t* free_bytes, uint64_t* total_bytes);
int ptsbe_synchronize(ptsbe_engine* h);
void* ptsbe_stream(ptsbe_engine* h);            /* cudaStream_t of the handle */
int ptsbe_info(ptsbe_engine* h, int64_t* out, int n);  /* {n, dtype, cap, n_passes, tile_bits, ...} */
/* Pass p of the loaded program: {tile bits L, contiguous low bits c, register bits per
 * phase, phases, ops, renormalising slots, threads per CTA, generated (1) / generic (0)}. */
int ptsbe_pass_info(ptsbe_engine* h, int p, int64_t* out, int n);
int ptsbe_last_error(ptsbe_engine* h, char* buf, size_t len);
/* Per-launch timing of the fused-pass kernel: when enabled, every pass launch
 * is bracketed by CUDA events on the handle's stream; profile_read syncs and
 * returns the accumulated kernel milliseconds and launch count. */
int ptsbe_profile(ptsbe_engine* h, int enable);
int ptsbe_profile_read(ptsbe_engine* h, double* total_ms, int64_t* launches);
/* Algorithmic bytes (one read + one write of every state a launch processes)
 * of the pass launches profiled since ptsbe_profile(h, 1). */
double ptsbe_profile_bytes(ptsbe_engine* h);
/* Per pass index: accumulated kernel milliseconds and algorithmic bytes of the
 * launches read by ptsbe_profile_read so far.  Returns the number of passes. */
int ptsbe_profile_passes(ptsbe_engine* h, double* ms, double* bytes, int max_passes);
/* Kernel launches issued by this handle since creation (for bench gpu_launches). */
int64_t ptsbe_launch_count(ptsbe_engine* h);

/* ---- dataset writer (host-only, no GPU) <- Dataset.write's records.jsonl
 * (execute.py:246-259, record order execute.py:181-223, bitstrings
 * statevector.py:44-53).  Formats the sampler's CSR output -- trajectory i owns
 * records [offsets[i], offsets[i+1]) of indices/counts and is written with id
 * traj_ids[i] -- as the reference's lines {"t":T,"b":"<n bits, qubit n-1
 * leftmost>","c":C}\n, each trajectory's records in ascending bitstring order,
 * on all host cores.  Returns the text's byte length; writes it (no NUL) when
 * buf != NULL and cap >= that length; -1 on invalid arguments (n_qubits
 * outside 1..64, decreasing offsets, negative ids, index >= 2^n_qubits). */
int64_t ptsbe_format_records(int n_qubits, int64_t n_traj, const int64_t* traj_ids, const int64_t* offsets,
                             const uint64_t* indices, const uint32_t* counts, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* PTSBE_H */
