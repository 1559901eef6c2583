/* stabkit_b200.h -- C ABI of the B200-native stabilizer-tableau engine.
 *
 * This is the drop-in boundary: the `stabkit::` C++ host classes
 * (the headers under include/stabkit/) and any foreign binding (ctypes, cgo, JNI ...) call
 * ONLY these entry points; behind them are hand-written sm_100a CUDA kernels
 * (paper_2507_03092_b200/csrc/).  There is no CPU fallback: every call that
 * computes fails with SK_ECUDA when no CUDA device is usable.
 *
 * Each entry point names the reference interface it replaces.  "ref:" paths
 * are relative to /root/reference ; SPEC = SPEC.md, the behavioural contract
 * for everything the reference ships only as specification.
 *
 * Conventions (ref: proj/include/stabkit/bitvec.hpp:26-35, pauli.hpp:28-31,53-54)
 *   - 64-bit words; qubit q lives in word q>>6, bit q&63; padding bits zero.
 *   - I=(0,0) X=(1,0) Z=(0,1) Y=(1,1); sign byte 1 means -1.
 *   - Host tableau/row arrays are ROW-MAJOR: row i occupies words
 *     [i*W, (i+1)*W) of the x array and of the z array, W = ceil(n/64).
 *     Tableau row order is SPEC:110: rows 0..n-1 stabilizers, n..2n-1
 *     destabilizers (the scratch row never leaves the chip).
 *   - Every function returns an sk_status; sk_last_error() gives the text.
 *     The C++ wrappers map the codes to the reference's exception types
 *     (ref: proj/include/stabkit/error.hpp:25-51).
 *   - Handles own device memory.  Host arrays are borrowed for the call.
 *   - One host thread drives a context; calls are ordered on the context's
 *     stream; calls that return data synchronise that stream.
 */
#ifndef STABKIT_B200_H
#define STABKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sk_status {
    SK_OK = 0,
    SK_EDIM = 1,         /* stabkit::DimensionError   (error.hpp:38-41) */
    SK_EUNSUPPORTED = 2, /* stabkit::UnsupportedError (error.hpp:43-46) */
    SK_EINVARIANT = 3,   /* stabkit::InvariantError   (error.hpp:48-51) */
    SK_ECUDA = 4,        /* CUDA runtime / no device: stabkit::Error */
    SK_ENCCL = 5,
    SK_EPARSE = 6,       /* stabkit::ParseError       (error.hpp:31-36) */
    SK_EARG = 7          /* null pointer / bad enum: stabkit::Error */
} sk_status;

/* Gate kinds.  M, T, TDG are circuit-level only. */
typedef enum sk_gate_kind {
    SK_H = 0, SK_S = 1, SK_SDG = 2, SK_X = 3, SK_Y = 4, SK_Z = 5,
    SK_CX = 6, SK_CZ = 7, SK_SWAP = 8, SK_M = 9, SK_T = 10, SK_TDG = 11
} sk_gate_kind;

typedef struct sk_gate {
    uint8_t kind;        /* sk_gate_kind */
    uint8_t pad[3];
    uint32_t q0;         /* target, or control of CX */
    uint32_t q1;         /* second qubit of CX/CZ/SWAP, else 0 */
} sk_gate;

typedef struct sk_ctx sk_ctx;
typedef struct sk_tableau sk_tableau;
typedef struct sk_program sk_program;
typedef struct sk_rows sk_rows;

/* Counters for the roofline report. */
typedef struct sk_counters {
    uint64_t n_rand, n_det;        /* measurements by branch                    */
    uint64_t k_rand, k_det;        /* rowsums performed in each branch          */
    uint64_t gate_hist[12];        /* gates applied, by sk_gate_kind            */
    uint64_t layers;               /* fused layer launches                      */
    uint64_t waves;                /* measurement scheduler waves               */
    uint64_t transposes;           /* column-major <-> row-major conversions    */
    uint64_t kernel_launches;      /* kernels launched by this library          */
    uint64_t meas_phase_ns[8];     /* measurement kernel, CTA 0 wall ns per phase: inspect, barrier, classify+det, barrier, random, barrier, window */
    /* "algorithmic bytes, per-kernel times" */
    uint64_t pred_evals;           /* commutation predicates evaluated by the grouping conflict kernels (config C4 roofline)      */
    double   algorithmic_bytes;    /* SURVEY 8d byte count of the gates and measurements run since the last reset, for the qubit
                                      count of the tableau used last (exact when one tableau size was in use)                      */
    double   class_ms[4];          /* device time of the last sk_program_run_profiled by kernel class: fused layers, transposes,
                                      k_measure_block, wave kernels (k_wave_cols + k_wave_rows) */
} sk_counters;

/* ---- context ---------------------------------------------------------- */
/* device: CUDA ordinal.  stream: a cudaStream_t to run on, or NULL to create
 * one.  Fails with SK_ECUDA if the device cannot be used. */
int32_t sk_ctx_create(int device, void* stream, sk_ctx** out);
void sk_ctx_destroy(sk_ctx* ctx);
const char* sk_last_error(const sk_ctx* ctx);
void* sk_ctx_stream(const sk_ctx* ctx);           /* the cudaStream_t in use */
int32_t sk_ctx_sync(sk_ctx* ctx);
int32_t sk_get_counters(sk_ctx* ctx, sk_counters* out);   /* syncs */
int32_t sk_reset_counters(sk_ctx* ctx);
const char* sk_version(void);

/* ---- tableau  (replaces SPEC:104-224 `tableau`) ------------------------ */
/* SPEC:125-133 new_identity.  n == 0 -> SK_EDIM. */
int32_t sk_tableau_create(sk_ctx* ctx, uint64_t n, sk_tableau** out);
void sk_tableau_destroy(sk_tableau* t);
int32_t sk_tableau_reset(sk_tableau* t);                 /* back to identity */
uint64_t sk_tableau_qubits(const sk_tableau* t);
/* Row-major 2n x W words for x and z, 2n sign bytes. */
int32_t sk_tableau_upload(sk_tableau* t, const uint64_t* x, const uint64_t* z, const uint8_t* sign);
int32_t sk_tableau_download(sk_tableau* t, uint64_t* x, uint64_t* z, uint8_t* sign);
/* EngineConfig.audit, the tableau invariants of SPEC:111-116 checked on the device: every pair of rows has the
 * symplectic product the CHP form demands (stabilizers commute, destabilizers commute, destabilizer i anticommutes with
 * stabilizer i and with nothing else).  *violations = number of row pairs (a < b) that break it; 0 for a valid tableau. */
int32_t sk_tableau_audit(sk_tableau* t, uint64_t* violations);

/* One fused layer of Clifford gates on pairwise-disjoint qubits: every
 * tableau word is read/written once per layer.  Replaces a loop of
 * apply_h/apply_s/apply_cx/apply_gate (row rules
 * ref: proj/src/pauli.cpp:146-187).  Qubit collision -> SK_EARG; M/T -> SK_EUNSUPPORTED. */
int32_t sk_apply_layer(sk_tableau* t, const sk_gate* gates, size_t ngates);
/* Any ordered Clifford sequence; layered internally (order per qubit kept). */
int32_t sk_apply_gates(sk_tableau* t, const sk_gate* gates, size_t ngates);

/* SPEC:175-185 measure_z with the counter RNG of rng.hpp:30-39:
 * random outcome = CounterRng{seed}.bit(ordinal). */
int32_t sk_measure_z(sk_tableau* t, uint32_t q, uint64_t seed, uint64_t ordinal,
                     uint8_t* outcome, uint8_t* deterministic);
/* m consecutive measurements; bit-identical to m sequential sk_measure_z
 * calls with ordinals ordinal0 .. ordinal0+m-1. */
int32_t sk_measure_batch(sk_tableau* t, const uint32_t* qubits, size_t m, uint64_t seed,
                         uint64_t ordinal0, uint8_t* outcomes, uint8_t* deterministic);
/* SPEC:165-173 rowsum(h, i) on tableau rows (h, i in [0, 2n)). Odd mod-4 sum -> SK_EINVARIANT. */
int32_t sk_tableau_rowsum(sk_tableau* t, uint64_t h, uint64_t i);

/* ---- engine  (replaces SPEC:294-362 `engine`: sim / sim2d) ------------- */
/* Compile a circuit once: validates it, fuses Clifford runs into layers,
 * groups measurement runs into blocks, uploads everything to the device.
 * mode 0 = sim (chunk marks ignored), 1 = sim2d (chunks that pass
 * validate_chunks become layers; others fall back and set bit 0 of
 * *warnings).  T/TDG -> SK_EUNSUPPORTED. */
int32_t sk_program_create(sk_ctx* ctx, uint64_t n, const sk_gate* gates, size_t ngates,
                          const uint32_t* chunk_marks, size_t nmarks, int mode,
                          sk_program** out, uint32_t* warnings);
void sk_program_destroy(sk_program* p);
uint64_t sk_program_measurements(const sk_program* p);
/* Runs the whole program on t from its current state (asynchronous; the
 * measurement record stays on the device until read). */
int32_t sk_program_run(sk_program* p, sk_tableau* t, uint64_t seed);
/* Same, with CUDA events around every launch and every kernel on the one stream, in order: class_ms = device ms spent in
 * {fused layers, transposes, k_measure_block, wave kernels (k_wave_cols + k_wave_rows)}.  Synchronises; for roofline
 * reporting, not for timing runs: an ordinary run overlaps the wave kernels with the transposition and the next layers. */
int32_t sk_program_run_profiled(sk_program* p, sk_tableau* t, uint64_t seed, float class_ms[4]);
/* SPEC:330-338 run_shots: `shots` runs from the identity tableau with seeds seed ^ shot_index.
 * ones[i] = number of shots in which measurement site i gave 1 (accumulated on the device);
 * records (optional, may be NULL) receives every shot's outcome bytes, [shots][measurements].
 * t ends in the state of the last shot.  shots == 0 -> SK_EARG.  Synchronises. */
int32_t sk_program_run_shots(sk_program* p, sk_tableau* t, uint64_t shots, uint64_t seed,
                             uint32_t* ones, uint8_t* records);
/* outcome / deterministic byte per M gate in circuit order (MeasurementRecord). */
int32_t sk_program_read_record(sk_program* p, uint8_t* outcomes, uint8_t* deterministic);
/* Convenience: identity tableau -> run -> record.  *out_t receives the final tableau. */
int32_t sk_sim(sk_ctx* ctx, uint64_t n, const sk_gate* gates, size_t ngates,
               const uint32_t* chunk_marks, size_t nmarks, int mode, uint64_t seed,
               sk_tableau** out_t, uint8_t* outcomes, uint8_t* deterministic, uint32_t* warnings);

/* ---- circuit_io / qec_gen host helpers ---------- */
/* Arrays returned through ** are malloc'ed by the library; release with sk_free. */
void sk_free(void* p);
/* SPEC:375-383.  final_data_measure != 0 appends `m` on the d*d data qubits
 * (BASELINE.json configs 1-3 "Z-basis measurement"). */
int32_t sk_circuit_surface_code(uint32_t d, uint32_t rounds, int final_data_measure,
                                uint64_t* n, sk_gate** gates, size_t* ngates,
                                uint32_t** chunk_marks, size_t* nmarks);
/* SPEC:385-393 */
int32_t sk_circuit_random_layered(uint64_t n, uint64_t seed, sk_gate** gates, size_t* ngates,
                                  uint32_t** chunk_marks, size_t* nmarks);
/* SPEC:242-250 parse_native (.stab text).  On error *err_line is the 1-based line. */
int32_t sk_circuit_parse_native(const char* text, size_t len, uint64_t* n, sk_gate** gates,
                                size_t* ngates, uint32_t** chunk_marks, size_t* nmarks,
                                size_t* err_line, char* err_msg, size_t err_cap);
/* SPEC:252-260 parse_qasm2_subset (OPENQASM 2.0 header, one qreg, optional cregs, h s sdg x y z cx cz swap t tdg,
 * `measure q[i] -> c[j];` -> M, `barrier` -> chunk mark).  Unsupported constructs (second qreg, parameterised or unknown
 * gates, `if`, `gate`, `reset`) -> SK_EUNSUPPORTED, malformed text -> SK_EPARSE; err_msg names the construct and line. */
int32_t sk_circuit_parse_qasm2(const char* text, size_t len, uint64_t* n, sk_gate** gates,
                               size_t* ngates, uint32_t** chunk_marks, size_t* nmarks,
                               size_t* err_line, char* err_msg, size_t err_cap);
/* SPEC:262-270.  violations: pairs (chunk index, gate index); kind 1 = collision, 2 = measurement.
 * A chunk that holds ONLY measurements is a measurement barrier region (every M is a full barrier), not a
 * chunk intended for sim2d: it is not reported, which is what SPEC:397 requires of the generators' output.  A
 * measurement next to Clifford gates in one chunk is a violation.  flags = SK_CHUNKS_STRICT reports the measurement-only
 * chunks too (the literal reading of SPEC:270's `chunk [m 0]` example). */
#define SK_CHUNKS_STRICT 1u
int32_t sk_circuit_validate_chunks(uint64_t n, const sk_gate* gates, size_t ngates,
                                   const uint32_t* chunk_marks, size_t nmarks,
                                   uint32_t** viol_chunk, uint32_t** viol_gate, uint8_t** viol_kind,
                                   size_t* nviol);
int32_t sk_circuit_validate_chunks_ex(uint64_t n, const sk_gate* gates, size_t ngates,
                                      const uint32_t* chunk_marks, size_t nmarks, uint32_t flags,
                                      uint32_t** viol_chunk, uint32_t** viol_gate, uint8_t** viol_kind,
                                      size_t* nviol);

/* ---- Pauli row sets on the device (grouping + Clifford+T pass) ---------- */
/* A resizable block of signed n-qubit Pauli rows (T_tab / layer / term list). */
int32_t sk_rows_create(sk_ctx* ctx, uint64_t n, uint64_t capacity, sk_rows** out);
void sk_rows_destroy(sk_rows* r);
uint64_t sk_rows_count(const sk_rows* r);
int32_t sk_rows_upload(sk_rows* r, const uint64_t* x, const uint64_t* z, const uint8_t* sign, uint64_t m);
int32_t sk_rows_download(sk_rows* r, uint64_t* x, uint64_t* z, uint8_t* sign);
/* Appends m rows behind the current ones (T_tab grows by one row per T gate; PAPER Alg. 2).  SK_EDIM when the
 * capacity given to sk_rows_create is exceeded. */
int32_t sk_rows_append(sk_rows* r, const uint64_t* x, const uint64_t* z, const uint8_t* sign, uint64_t m);
/* ref: proj/src/pauli.cpp:117-140 commutes_with / qubitwise_commutes_with over a tile of the pair matrix: bit (j - j0) of
 * out_bits[(i - i0) * words + ...] is set iff rows i and j CONFLICT (mode 0: anticommute, mode 1: not qubit-wise commuting),
 * i in [i0, i0+ni), j in [j0, j0+nj), words = ceil(nj/64) per output row (host buffer).  The grouping driver itself
 * consumes conflicts on the fly (group-major kernel); the tile is the API for callers that want the matrix. */
int32_t sk_commute_matrix_tile(sk_rows* r, int mode, uint64_t i0, uint64_t ni, uint64_t j0, uint64_t nj, uint64_t* out_bits);
/* ref: proj/src/pauli.cpp:146-187 applied to every row (Algorithm 2 inner loop). */
int32_t sk_rows_conj_layer(sk_rows* r, const sk_gate* gates, size_t ngates);
/* ref: proj/src/pauli.cpp:215-237 commutation_vector: bit i set iff p anticommutes with row i. */
int32_t sk_commutation_vector(sk_rows* r, const uint64_t* px, const uint64_t* pz, uint64_t* out_bits);
/* ref: proj/src/pauli.cpp:239-254 rowsum_plus_i on every row that anticommutes with (p, psign). */
int32_t sk_rowsum_plus_i_where_anticommuting(sk_rows* r, const uint64_t* px, const uint64_t* pz,
                                             uint8_t psign, uint64_t* n_updated);
/* ref: proj/src/pauli.cpp:142-144 same_axis: first duplicate pair in scan order. found=0 if none. */
int32_t sk_find_first_duplicate(sk_rows* r, int* found, uint64_t* i, uint64_t* j);
/* ref: proj/src/pauli.cpp:100-106 weight, summed over rows. */
int32_t sk_weight_sum(sk_rows* r, uint64_t* out);

/* SPEC:444-452 group_greedy on terms ALREADY in sorted order (rows of r);
 * mode 0 = GC, 1 = QWC; group_of[i] = first-fit group of row i. */
int32_t sk_group_first_fit(sk_rows* r, int mode, uint32_t* group_of, uint64_t* ngroups);
/* SPEC:454-462 verify_grouping: number of violating intra-group pairs. */
int32_t sk_verify_grouping(sk_rows* r, int mode, const uint32_t* group_of, uint64_t* nviolations);

/* SPEC:545-553 transpile (Algorithms 2-4).  Results are read back with the
 * accessors below.  Mid-circuit M -> SK_EUNSUPPORTED. */
typedef struct sk_pbc sk_pbc;
/* The DEFAULT (sk_transpile, flags 0) is the unitary-exact form: SPEC:575-589 makes the dense-statevector check
 * (verify_transpile, TV < 1e-9) the arbiter of every sign convention, and that check requires (a) the INVERSE
 * gate in Algorithm 2's backward walk (S <-> S^dagger; moving an axis P from behind G to in front of it gives G^dagger P G) and
 * (b) a T row to stay behind every rotation it anticommutes with (it joins the layer right after the last layer holding an
 * anticommuting member).  Algorithm 4 and rowsum+i are as published.
 * SK_TRANSPILE_PUBLISHED selects Algorithms 2-3 verbatim (G's own CHP rule in the backward walk; "first layer from P_0 it
 * commutes with", PAPER Alg. 2-3) -- NOT unitarily equivalent in general (smallest counter-examples:
 * `h s t h`, `t h t h t h`); kept for comparison with the paper's text only.  SK_TRANSPILE_EXACT (bit 0) names the default
 * explicitly and is accepted for source compatibility. */
int32_t sk_transpile(sk_ctx* ctx, uint64_t n, const sk_gate* gates, size_t ngates, sk_pbc** out);
#define SK_TRANSPILE_EXACT 1u
#define SK_TRANSPILE_PUBLISHED 2u
int32_t sk_transpile_ex(sk_ctx* ctx, uint64_t n, const sk_gate* gates, size_t ngates, uint32_t flags, sk_pbc** out);
void sk_pbc_destroy(sk_pbc* p);
/* stats: initial_t, final_rotations_rowcount, final_rotations_pauliweight, layers, passes */
int32_t sk_pbc_stats(sk_pbc* p, uint64_t out5[5]);
uint64_t sk_pbc_layer_rows(sk_pbc* p, uint64_t layer);
int32_t sk_pbc_layer_download(sk_pbc* p, uint64_t layer, uint64_t* x, uint64_t* z, uint8_t* sign);
/* final M_tab, 2n rows row-major (measurement_rows are rows 0..n-1) */
int32_t sk_pbc_mtab_download(sk_pbc* p, uint64_t* x, uint64_t* z, uint8_t* sign);

/* ---- commutation grouping with the pair matrix sharded by row blocks ------
 * Replaces nothing in the reference (single-process): it is the multi-GPU form of sk_group_first_fit.  Every
 * shard holds the replicated rows and group assignment; per block of 1024 terms shard s of S evaluates the predicates
 * (proj/src/pauli.cpp:117-140) against the groups of the bitmap words w with w % S == s, the driver ORs the shards' bitmaps
 * (allreduce-SUM over disjoint words: ncclAllReduce / torch.distributed, or in process) and every shard resolves the block.
 * Rows of at most 128 qubits (config C4).  d_bitmap: device buffer of sk_group_shard_bitmap_words() u32. */
typedef struct sk_group_shard sk_group_shard;
int32_t sk_group_shard_create(sk_rows* r, int mode, uint32_t shard, uint32_t nshards, sk_group_shard** out);
void sk_group_shard_destroy(sk_group_shard* g);
uint64_t sk_group_shard_blocks(const sk_group_shard* g);
uint64_t sk_group_shard_bitmap_words(const sk_group_shard* g);
int32_t sk_group_shard_conflicts(sk_group_shard* g, uint64_t block, uint32_t* d_bitmap);
int32_t sk_group_shard_resolve(sk_group_shard* g, uint64_t block, uint32_t* d_bitmap);
int32_t sk_group_shard_result(sk_group_shard* g, uint32_t* group_of, uint64_t* ngroups);

/* ---- row sharding of one tableau across GPUs ------ */
/* A shard owns the slots [slot_lo, slot_hi): stabilizer i AND destabilizer i for every i in the
 * range (the deterministic branch of SPEC:183 then needs no remote row).  One shard per GPU /
 * process; Clifford gates never communicate (rows are independent).  A measurement is
 * assembled by the host driver from the calls below plus three small exchanges:
 *   pivot search  -> allreduce-min of d_cand over the shards
 *   random branch -> owner's pivot row broadcast, every shard rowsums
 *   deterministic -> allgather of the partial products, multiplied in shard order
 * Every d_* argument is a DEVICE pointer supplied by the caller (the exchange buffers of its
 * communication library), used on the context's stream; results are bit-identical to the unsharded
 * sk_measure_batch. */
typedef struct sk_shard sk_shard;
int32_t sk_shard_create(sk_ctx* ctx, uint64_t n, uint64_t slot_lo, uint64_t slot_hi, sk_shard** out);  /* identity rows */
void sk_shard_destroy(sk_shard* s);
int32_t sk_shard_reset(sk_shard* s);
/* Any ordered Clifford sequence on this shard's rows (same kernel and layering as sk_apply_gates). */
int32_t sk_shard_apply_gates(sk_shard* s, const sk_gate* gates, size_t ngates);
/* d_cand[j] (int32) = smallest GLOBAL stabilizer index in this shard with an x on qubits[j], else 0x7f7f7f7f. */
int32_t sk_shard_pivot_search(sk_shard* s, const uint32_t* qubits, size_t m, int32_t* d_cand);
/* 64-bit words per partial product / pivot row buffer: x[Wp] z[Wp] phase pad, Wp = W rounded up to even. */
uint64_t sk_shard_partial_words(const sk_shard* s);
/* d_part[j] = product of this shard's partner stabilizers of measurement j (identity if none). */
int32_t sk_shard_det_partial(sk_shard* s, const uint32_t* qubits, size_t m, uint64_t* d_part);
/* d_gathered = [nshards][m][partial_words] in shard order -> outcome bytes (host). Synchronises. */
int32_t sk_shard_det_combine(sk_shard* s, const uint64_t* d_gathered, uint32_t nshards, size_t m, uint8_t* outcomes);
/* Owner only: stabilizer p (global index) -> d_row[partial_words]. */
int32_t sk_shard_pivot_row(sk_shard* s, uint64_t p, uint64_t* d_row);
/* Every shard: rowsum(h, pivot) on its rows with an x on q (ref: proj/src/pauli.cpp:189-205 phase sum);
 * the owner then stores destabilizer p := pivot row and stabilizer p := (-1)^outcome Z_q. */
int32_t sk_shard_random_update(sk_shard* s, uint32_t q, uint64_t p, const uint64_t* d_row, uint8_t outcome);
/* This shard's rows, row-major: stabilizers slot_lo..slot_hi-1, then their destabilizers. Synchronises. */
int32_t sk_shard_download(sk_shard* s, uint64_t* x, uint64_t* z, uint8_t* sign);
/* Replicated elimination of a random measurement block: a shard's rows as one contiguous device block (stabilizer rows, destabilizer
 * rows, sign words of the two halves; sk_shard_export_words() 64-bit words), the blocks of all shards placed into a full
 * sk_tableau (import_block per shard, then commit), sk_measure_batch on it -- identical on every rank -- and the rows back
 * (export_block -> sk_shard_import_rows).  One allgather of the tableau per random block instead of an exchange per measurement. */
uint64_t sk_shard_export_words(const sk_shard* s);
int32_t sk_shard_export_rows(sk_shard* s, uint64_t* d_buf);
int32_t sk_shard_import_rows(sk_shard* s, const uint64_t* d_buf);
int32_t sk_tableau_import_block(sk_tableau* t, uint64_t slot_lo, uint64_t slot_hi, const uint64_t* d_buf);
int32_t sk_tableau_commit_blocks(sk_tableau* t);
int32_t sk_tableau_export_block(sk_tableau* t, uint64_t slot_lo, uint64_t slot_hi, uint64_t* d_buf);
/* rowsums performed: out2[0] random branch, out2[1] deterministic branch. Synchronises. */
int32_t sk_shard_counters(sk_shard* s, uint64_t out2[2]);
/* Plain device buffers for the exchange, so that a host binding needs no CUDA headers of its own.
 * sk_dev_copy kind: 0 host->device, 1 device->host (both synchronise), 2 device->device (stream ordered). */
int32_t sk_dev_alloc(sk_ctx* ctx, size_t bytes, void** out);
void sk_dev_free(sk_ctx* ctx, void* p);
int32_t sk_dev_copy(sk_ctx* ctx, void* dst, const void* src, size_t bytes, int kind);

#ifdef __cplusplus
}
#endif
#endif /* STABKIT_B200_H */
