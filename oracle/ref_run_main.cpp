// TEST INFRASTRUCTURE ONLY: a process around the reference's own CLI entry
// point hood::cli::run (cli.cpp:144-190), built by `make -C oracle ref` from
// the UNMODIFIED reference sources into oracle/_ref/hood_ref_run.  The
// reference's stream writers (write_trace_round, cli.cpp:108-118) run here in a
// normal process, where libstdc++ streams work (they do not inside a
// ctypes-loaded library on this image).  tests/golden/make_golden.py uses it to
// record the reference's trace files; nothing on the product path runs it.
//
//   hood_ref_run <points file> <trace file>   -> the run output on stdout
#include <iostream>
#include <string>

#include "hood/cli.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: hood_ref_run <points> <trace>\n";
    return 2;
  }
  hood::cli::RunOptions o;
  o.input = argv[1];
  o.trace_path = argv[2];
  o.mode = hood::cli::Mode::parallel;
  return hood::cli::run(o, std::cout, std::cerr);
}
