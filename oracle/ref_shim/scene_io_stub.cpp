// scene_io stub — TEST INFRASTRUCTURE ONLY (oracle/_ref).  The reference's scene_io.cpp needs
// nlohmann/json (absent: gitignored vendor/ tree).  It is not on the PBA hot path (SURVEY.md §8f row 3
// is served by paper_1704_06967_b200/scene_io.py); these definitions only satisfy the linker for
// tests/test_synth.cpp, whose two scene_io test cases are excluded from the oracle/_ref run.
#include "pba/scene_io.hpp"

namespace pba {
namespace {
[[noreturn]] void unavailable(const char* what) {
  throw Error(std::string(what) + ": scene_io is not built in oracle/_ref (needs nlohmann/json)");
}
}  // namespace
SceneSpec parse_scene_spec(const std::string&) { unavailable("parse_scene_spec"); }
SceneSpec load_scene_spec(const std::string&) { unavailable("load_scene_spec"); }
void save_scene(const RenderedScene&, const std::string&) { unavailable("save_scene"); }
RenderedScene load_scene(const std::string&) { unavailable("load_scene"); }
ParamRms compute_param_rms(const std::vector<Pose>&, const std::vector<double>&, const std::vector<Pose>&,
                           const std::vector<double>&) {
  unavailable("compute_param_rms");
}
void write_metrics_csv(const SolveReport&, const std::vector<Pose>&, const std::vector<double>&,
                       const std::string&, bool) {
  unavailable("write_metrics_csv");
}
void write_final_json(const SolveReport&, const std::string&, bool) { unavailable("write_final_json"); }
}  // namespace pba
