// oracle/_ref/run_experiment "<key=value;...>" out.csv
// Runs the reference's run_experiment (harness.cpp:249-302) and its own
// aggregate CSV writer (harness.cpp:311-342).  Test infrastructure: the
// golden for the byte-identical-CSV parity test (tests/test_report_format.py).
#include <cstdio>
#include <cstdlib>

extern "C" int ref_run_experiment(const char* cfg_text, const char* csv_path, double* out_seconds,
                                  int* out_diverged);
extern "C" const char* ref_last_error();

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s <config key=value;...> <out.csv>\n", argv[0]);
    return 64;
  }
  double sec = 0.0;
  int diverged = 0;
  const int rc = ref_run_experiment(argv[1], argv[2], &sec, &diverged);
  if (rc) std::fprintf(stderr, "reference raised: %s\n", ref_last_error());
  else std::printf("%.6f %d\n", sec, diverged);
  return rc;
}
