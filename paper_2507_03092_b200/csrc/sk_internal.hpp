// sk_internal.hpp -- host-side internals shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <functional>

#include "common.cuh"
#include "stabkit_b200.h"

struct sk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // measurement pipeline: k_wave_cols runs on `side` next to the C -> R transposition, k_wave_rows under the next gate layers
    cudaStream_t side = nullptr;
    cudaStream_t copy = nullptr;            // sk_sim: host -> device uploads of large programs, beside the kernels of earlier segments
    cudaEvent_t ev_fork = nullptr, ev_cols = nullptr, ev_rows = nullptr, ev_side = nullptr;
    bool side_pending = false;              // work on `side` that `stream` has not waited for yet
    int no_tr_regs = 0;                     // SK_TRANSPOSE_REGS=0: shuffle transposition kernel only (A/B aid)
    int no_fuse_h = 0;                      // SK_FUSE_H=0: programs keep their H ; CX.. ; H windows as written (no XCX rewriting)
    int no_pipe = 0;                        // SK_PIPELINE=0: the two wave kernels on the main stream, in order
    int num_sms = 0;
    int max_smem_optin = 0;
    int prof = 0;                           // SK_DEBUG_PROF: device-side phase timers (slows the kernel)
    int no_graph = 0;                       // SK_NO_GRAPH=1: sk_program_run enqueues plain launches instead of replaying a CUDA graph
    int no_fold = 0;                        // SK_NO_FOLD=1: the measurement kernel gathers every panel in a phase of its own
    int row_cap = 0;                        // SK_ROW_CAP=<k>: row-form factorisation only up to k active rows (tests: exercises the regather path)
    uint64_t tableau_uid = 0;
    int pdl = 1;                            // programmatic dependent launch of the layer and transpose kernels (SK_PDL=0 disables)
    int no_wave_kernel = 0;                 // SK_WAVE_KERNEL=0: wave mode only inside the cooperative measurement kernel
    int no_repl = 0;                        // SK_PANEL_REPL=0: panel mode without the replicated level-form path (general path only)
    int seq_rows = 0;                       // SK_PANEL_SEQ=1: step-by-step row-form panel factorisation instead of the level form
    int force_columns = 0;                  // SK_PANEL_COLUMNS=1: column-form panel factorisation only (testing aid)
    int meas_grid_override = 0;             // SK_MEAS_GRID: CTAs of the measurement kernel (profiling aid)
    std::string err;
    // growable device scratch
    void* d_gates = nullptr; size_t d_gates_cap = 0;
    void* d_tmp = nullptr; size_t d_tmp_cap = 0;
    void* h_pin = nullptr; size_t h_pin_cap = 0;   // pinned host staging (sk_sim: ordered gates + measured qubits)
    skd::u32* d_err = nullptr;              // generic error word for small kernels
    void* d_ws = nullptr;                   // skd::MeasWs: barrier, wave slots, device-side counters
    // host-side counters (device-side ones live in MeasWs)
    sk_counters cnt{};
    uint64_t last_n = 0;                    // qubit count of the tableau used last (for sk_counters.algorithmic_bytes)
    double class_ms[4] = {0, 0, 0, 0};      // last sk_program_run_profiled: layers, transposes, k_measure_block, wave kernels
    std::function<void(int)>* prof_mark = nullptr;      // set while a profiled run enqueues: event + class of the launches before it
    std::vector<uint32_t> q_epoch; uint32_t epoch = 0;   // qubit-collision scratch
};

#define SK_FAIL(ctx, code, ...)                                   \
    do {                                                          \
        char _b[512]; snprintf(_b, sizeof _b, __VA_ARGS__);       \
        (ctx)->err = _b; return (code);                           \
    } while (0)

#define SK_CUDA(ctx, call)                                                                 \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) SK_FAIL(ctx, SK_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

// Frees the device pointers registered with it when the scope ends (early SK_CUDA / SK_FAIL returns included).
struct SkDevScope {
    std::vector<void**> slots;
    template <class T> void own(T** p) { slots.push_back(reinterpret_cast<void**>(p)); }
    ~SkDevScope() { for (void** p : slots) if (*p) { cudaFree(*p); *p = nullptr; } }
};

int32_t sk_ctx_reserve_gates(sk_ctx* ctx, size_t bytes);
int32_t sk_ctx_reserve_tmp(sk_ctx* ctx, size_t bytes);

// layering of an ordered Clifford run into layers of disjoint qubits (order per
// qubit preserved => same tableau as gate-by-gate application).  Appends the
// re-ordered gates to `out` and the layer sizes to `layer_sizes`.
void sk_layer_run(const sk_gate* g, size_t ng, uint64_t n, std::vector<uint32_t>& scratch,
                  std::vector<sk_gate>& out, std::vector<uint32_t>& layer_sizes);

static inline bool sk_is_two_qubit(uint8_t k) { return k == SK_CX || k == SK_CZ || k == SK_SWAP; }
