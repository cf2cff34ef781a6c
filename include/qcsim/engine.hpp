// qcsim/engine.hpp -- Algorithm 1 of arXiv:1811.05630 on the GPU.
//
// The reference specifies the engine but ships no header
// or source for it; names follow SPEC.md (EngineConfig, RunMetrics, run,
// gather_state).  Every gate pass -- decode, normalize, apply the lowered
// action, sq_norm, re-encode every slice -- runs on the device
// (libqcsim_b200.so); the compressed state stays resident in HBM.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/codec.hpp"
#include "qcsim/statevec.hpp"

struct qcsim_engine;

namespace qcsim {

enum class NormPolicy { EveryGate, EveryKGates, Off };

struct EngineConfig {
    int slice_bits = -1; // < 0: default_slice_bits(n)
    CodecConfig codec{CodecMode::Absolute, 1e-5, 16, Predictor::PreviousValue};
    bool compression_enabled = true;
    int workers = 1; // accepted for API parity; all slices run concurrently
    NormPolicy norm_policy = NormPolicy::EveryGate;
    int norm_every_k = 1;
    double norm_drift_tolerance = 0.02;
    int device = 0;
    int rank = 0, world = 1; // slice sharding
    uint64_t wave_bytes = 0; // dense working-set budget of a gate pass (0: 45% of the device)
};

struct RunMetrics {
    double min_compression_ratio = 0.0;
    double mean_compression_ratio = 0.0;
    std::vector<double> per_gate_min_ratio; // one entry per gate pass since the load
    double wall_seconds = 0.0;
    double baseline_wall_seconds = 0.0; // measure_overhead: the compression-off run
    double overhead_factor = 0.0;       // measure_overhead: wall_seconds / baseline_wall_seconds
    uint64_t peak_compressed_bytes = 0;
    uint64_t dense_bytes = 0;
    double final_norm = 0.0;
    uint64_t compress_calls = 0;
    uint64_t gates = 0;
    uint64_t index_bytes = 0;
    uint64_t fallback_planes = 0;
};

// One row of the per-gate report (SPEC.md:383 CSV: gate_index, min_ratio,
// mean_ratio, seconds) plus the state's bytes after the pass.  Row 0 is the
// initial compression (gate_index -1).
struct GateMetrics {
    long long gate_index = 0;
    double min_ratio = 0.0, mean_ratio = 0.0, seconds = 0.0;
    uint64_t compressed_bytes = 0, index_bytes = 0;
};

class Engine {
  public:
    Engine(int num_qubits, const EngineConfig &config);
    ~Engine();
    Engine(const Engine &) = delete;
    Engine &operator=(const Engine &) = delete;

    void load(const StateVector &initial);        // dense or compressed slices
    void load_basis(uint64_t basis_index);
    RunMetrics run(const Circuit &circuit);        // gate passes
    RunMetrics run(const std::vector<GateAction> &actions);
    RunMetrics metrics() const;
    std::vector<GateMetrics> gate_metrics() const;
    StateVector gather_state(int guard_qubits = 28) const; // dense StateVector
    std::vector<CompressedPlanes> compressed_slices() const; // checkpoint
    std::vector<double> slice_norms() const;                 // cached sq_norm per slice (statevec.hpp:72)
    // Resume from a checkpoint: the slices' QCB1 planes, their cached sq_norm
    // and the number of gates already applied (qcsim_engine_load_blocks).
    void resume(const std::vector<CompressedPlanes> &slices, const std::vector<double> &sq_norms,
                uint64_t gates_done = 0);

    int num_qubits() const { return n_; }
    int slice_bits() const { return s_; }

  private:
    qcsim_engine *h_ = nullptr;
    int n_ = 0, s_ = 0;
};

// compresses `initial`, applies every gate, returns the
// engine holding the final compressed state plus the metrics.
std::pair<std::unique_ptr<Engine>, RunMetrics> run(const Circuit &circuit, const EngineConfig &config,
                                                   const StateVector &initial);

// SPEC.md:353-361 (Fig. 2): runs the circuit twice on the same
// device -- compression on (config) and off -- and returns the compressed
// run's metrics with baseline_wall_seconds / overhead_factor filled.
RunMetrics measure_overhead(const Circuit &circuit, const EngineConfig &config, const StateVector &initial);

// Metrics report: a JSON object with every RunMetrics field
// plus the per-gate rows, and the CSV export (gate_index, min_ratio,
// mean_ratio, seconds).
std::string metrics_json(const RunMetrics &m, const std::vector<GateMetrics> &rows);
std::string metrics_csv(const std::vector<GateMetrics> &rows);

} // namespace qcsim
