// B200 cost model (model.cpp): the reference's CostModel
// (cost_model.hpp:14-33) re-parameterised for this executor, and its
// calibrate() (calibrate.cpp:67-181) fitting it to measured latencies.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "program.hpp"

namespace cecoll {

// Times in ns, bandwidths in bytes/s of algorithmic HBM traffic (read+write).
// Defaults: round-1 probes (tools/phase_probe.cu, profiles/b200_cost_model.conf;
// MEASURED_PEAKS.json), before any fit.
struct B200Model {
  double t_kernel = 2050;   // device: one kernel boundary, back to back
  double t_graph = 4000;    // device: one recorded-graph launch
  double t_branch = 900;    // device: each further parallel branch of a recorded graph
  double t_node = 1500;     // device: each serial memcpy node on a branch
  double t_trigger = 4000;  // prelaunch: caller-stream ready write + gate observation + completion join
  double bw_copy = 6.3e12;  // SM mover, copy items
  double bw_fan = 5.9e12;   // SM mover, fan / broadcast items (write-bound)
  double bw_ce = 6.0e12;    // driver memcpy nodes (device-local copies run on SMs on one GPU)
  double bw_lanes = 6.3e12; // one item kernel per lane, running concurrently (chunks >= 4 MiB)
  double bw_swap = 6.3e12;  // in-place swap items in one register-mover kernel (merged / prelaunch)
  double l2_boost = 1.3;    // every bandwidth, when the collective's buffers fit in L2
  double l2_bytes = 96.0 * (1 << 20);  // that footprint (126 MB L2, fixed, not fitted)
  double folded_max_bytes = 8.0 * (1 << 20);  // prelaunch bodies up to this traffic are one folded kernel
  double prelaunch_gain_threshold = 0.002;    // winner_grid's tie-break (cost_model.hpp:30)
  double t_stream = 3000;  // device: fill / drain of an SM mover table beyond one wave
  double stream_min_bytes = 148.0 * 32768;  // one wave: 32 KiB tiles, one CTA per SM (fixed, not fitted)
  double l2_boost_swap = 1.3;  // bw_swap's factor when the buffers fit in L2 (in-place: writes hit read lines)
};

struct Measurement {
  Kind kind;
  Impl impl;
  int64_t s;
  int n;
  double ns;
};

struct FitResult {
  B200Model model;
  double residual = 0;
  std::string report;
};

B200Model default_model();
// Device time of one collective (back to back) with n co-resident ranks.
double predict_ns(const B200Model& m, Kind kind, Impl impl, int64_t s, int n);
std::vector<Impl> model_candidates(Kind kind);
Impl model_winner(const B200Model& m, Kind kind, int64_t s, int n);
double model_score(const B200Model& m, const std::vector<Measurement>& meas, std::string* report);
FitResult calibrate_b200(const std::vector<Measurement>& meas, uint64_t seed, int iterations);

}  // namespace cecoll
