// cmd_solve (reference run.hpp:375-480) smoke driver: the reference's own
// production caller of ggr() (table load, FD config + validation, solve, PHC
// recomputation, prompt rendering, dedup, cache replay, cost, schedule file).
// Built twice from this one source by proj/tests/Makefile: against the
// drop-in headers (bin/cmd_solve_smoke, GPU path) and against the unmodified
// reference headers alone (bin/cmd_solve_smoke_ref, CPU); tests/
// test_dropin_cpp.py requires identical reports (minus wall time) and
// identical schedule files.
//
//   cmd_solve_smoke TABLE [FD_JSON|-] [SOLVER] [SCHEDULE_OUT] [THRESHOLD]

#include <iostream>
#include <sstream>
#include <string>

#include "prefixopt/run.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: cmd_solve_smoke TABLE [FD_JSON|-] [SOLVER] [SCHEDULE_OUT] [THRESHOLD]\n";
    return 2;
  }
  prefixopt::RunConfig cfg;
  cfg.input_path = argv[1];
  if (argc > 2 && std::string(argv[2]) != "-") cfg.fd_config_path = argv[2];
  if (argc > 3) cfg.solver = argv[3];
  if (argc > 4) cfg.schedule_out = argv[4];
  if (argc > 5) cfg.ggr.hitcount_stop_threshold = std::stoull(argv[5]);
  cfg.system_prompt = "You are a data analyst. Use the provided JSON data to answer the user query.";
  cfg.question = "Is this movie suitable for kids? Answer Yes or No.";
  try {
    std::ostringstream diag;
    prefixopt::RunReport rep = prefixopt::cmd_solve(cfg, diag);
    auto j = prefixopt::run_report_to_json(rep);
    j["solver"].erase("wall_ms");
    std::cout << j.dump(1) << "\n" << diag.str();
  } catch (const std::exception& e) {
    std::cout << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
