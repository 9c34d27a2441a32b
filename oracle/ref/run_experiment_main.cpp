// oracle/_ref/run_experiment "<key=value;...>" out.csv [summary.json [replicate.csv [r]]]
// Runs the reference's run_experiment (harness.cpp:249-302) and its own
// writers: the aggregate CSV (harness.cpp:311-342), summary_json
// (:367-427) and write_replicate_csv of replicate r (default 0, :344-365).
// Test infrastructure: the goldens for the byte-identical writer parity
// tests (tests/test_report_format.py).
#include <cstdio>
#include <cstdlib>

extern "C" int ref_run_experiment(const char* cfg_text, const char* csv_path, double* out_seconds,
                                  int* out_diverged);
extern "C" int ref_run_experiment_outputs(const char* cfg_text, const char* csv_path,
                                          const char* json_path, const char* rep_csv_path,
                                          int rep_index);
extern "C" const char* ref_last_error();

int main(int argc, char** argv) {
  if (argc < 3 || argc > 6) {
    std::fprintf(stderr, "usage: %s <config key=value;...> <out.csv> [summary.json [rep.csv [r]]]\n",
                 argv[0]);
    return 64;
  }
  int rc;
  if (argc == 3) {
    double sec = 0.0;
    int diverged = 0;
    rc = ref_run_experiment(argv[1], argv[2], &sec, &diverged);
    if (!rc) std::printf("%.6f %d\n", sec, diverged);
  } else {
    rc = ref_run_experiment_outputs(argv[1], argv[2], argv[3], argc > 4 ? argv[4] : nullptr,
                                    argc > 5 ? std::atoi(argv[5]) : 0);
  }
  if (rc) std::fprintf(stderr, "reference raised: %s\n", ref_last_error());
  return rc;
}
