// qcsim/reference.hpp -- dense single-array simulator (correctness oracle).
//
// Same declarations as /root/reference/proj/include/qcsim/reference.hpp:32-50
// (declared upstream, never implemented there; implemented here on the host
// with the pinned gate arithmetic of DESIGN.md §3).
#pragma once

#include <cstdint>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/statevec.hpp"

namespace qcsim {

struct DenseState {
    int num_qubits = 0;
    std::vector<Amplitude> amps;
};

DenseState make_dense_basis(int num_qubits, uint64_t basis_index);
void apply_action_dense(const GateAction &action, std::vector<Amplitude> &amps);
DenseState ref_run(const Circuit &circuit, DenseState initial, int guard_qubits = 24);
double success_probability(const DenseState &state, uint64_t basis_index);

} // namespace qcsim
