// C shim over the reference's simulator — TEST / ANALYSIS INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile with the reference's own sim.cpp and
// cost_model.cpp (plus program/compiler/topology/verifier) into
// oracle/_ref/libdmasim_sim.so when nlohmann/json.hpp is available. Used by
// oracle/b200_model.py to run the reference's fluid simulator with the
// B200-measured phase latencies (tools/phase_probe.cu) and compare its
// predictions with the measured sweep.
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>

#include "dmasim/compiler.hpp"
#include "dmasim/cost_model.hpp"
#include "dmasim/sim.hpp"
#include "dmasim/topology.hpp"

using namespace dmasim;

extern "C" {

// out5: total, control, schedule, copy, sync (critical-path ns). Returns 0 or -1.
int sim_run(const char* kind, const char* impl, std::int64_t s, int n, const char* cost_text,
            double link_bandwidth, double* out5) {
  try {
    auto k = parse_collective(kind);
    auto im = parse_implementation(impl);
    if (!k || !im) return -1;
    std::map<std::string, std::string> over;
    if (link_bandwidth > 0) {
      std::ostringstream o;
      o.precision(17);
      o << link_bandwidth;
      over["link_bandwidth_bytes_per_s"] = o.str();
    }
    NodeTopology topo = build_topology(n, over);
    std::istringstream in(cost_text ? cost_text : "");
    CostModel cost = cost_text ? load_cost_model(in) : CostModel{};
    if (cost.engine_throughput_cap < topo.link_bandwidth) cost.engine_throughput_cap = topo.link_bandwidth;
    CollectiveSpec spec{*k, s, n, false};
    CommandProgram program = compile(*im, spec, topo);
    SimOptions opts;
    opts.record_events = false;
    Timeline t = simulate(program, topo, cost, opts);
    out5[0] = t.total_ns();
    auto get = [&](Phase p) {
      auto it = t.critical_path_ns.find(p);
      return it == t.critical_path_ns.end() ? 0.0 : it->second;
    };
    out5[1] = get(Phase::Control);
    out5[2] = get(Phase::Schedule);
    out5[3] = get(Phase::Copy);
    out5[4] = get(Phase::Sync);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
