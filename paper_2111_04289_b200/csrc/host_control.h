// Host-side control of the LMStream micro-batch loop (C++17, no CUDA).
//
//  * Admission: Algorithm 1 ConstructMicroBatch with Eq. 6,
//    CG(dN) / OS(tN) modes of the earlier revision (P:6), readings
//    R11/R15/R16/R22 of DESIGN.md §3.
//  * Planner: Algorithm 2 MapDevice with Eq. 7-9 and Table III.
//  * Regression: Eq. 10 online OLS of the inflection point.
//  * Metrics: Eq. 4 AvgThPut, Eq. 5 MaxLat, nearest-rank percentiles.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace lms {

enum class Mode : int32_t { LMStream = 0, Deadline = 1, Trigger = 2, Manual = 3 };

struct DatasetInfo {
  uint64_t id;
  double ingest_time;
  uint64_t nbytes;
};

// ---------------------------------------------------------------- Eq. 6 / Alg. 1
// Eq. 6: max_j buff_j + (sum_j bytes_j) / avg_thput.
double est_max_lat(const double* buff_s, const uint64_t* bytes, uint64_t n, double avg_thput);

enum AdmitReason : int32_t {
  kAdmitForced = 0, kAdmitBootstrap = 1, kAdmitTarget = 2, kAdmitTumblingBootstrap = 3,
  kAdmitCap = 4, kAdmitTrigger = 5, kAdmitFlush = 6, kBuffer = -1, kPoll = -2
};

constexpr uint64_t kCapDatasets = 4096;

struct AdmitResult {
  bool admit = false;
  double est = 0.0 / 0.0;   // NaN when not computed
  int32_t reason = kPoll;
};

// One Algorithm 1 decision over tmp = buffered U new (creation order).
AdmitResult admit_decision(Mode mode, double slide_s, double deadline_s, double now_s,
                           const double* ingest_s, const uint64_t* bytes, uint64_t n,
                           double avg_thput, const double* maxlat_hist, uint64_t n_hist);

// ---------------------------------------------------------------- Alg. 2
struct Dag {
  std::vector<uint8_t> kind;
  std::vector<std::vector<int32_t>> preds;
};
double base_cost(int32_t op_kind);                       // Table III, < 0 if unknown
// Children-first topological order; empty + false on cycle / not one root.
bool traverse(const Dag& dag, std::vector<int32_t>& order);
bool map_device(const Dag& dag, double part, double infpt, double btc, std::vector<uint8_t>& dev);
Dag query_dag(int32_t kind);                             // SPEC S:153 catalog

// ---------------------------------------------------------------- Eq. 10
bool infpt_fit(const double* thput, const double* lat, const double* infpt, uint64_t n,
               double b[3]);
double infpt_predict(const double b[3], double thput, double lat);

// Asynchronous Eq. 10 refit ("LMStream handles the optimization process
// asynchronously ... the results only need to be returned before the next processing phase").
// One persistent worker thread per handle: submit() hands over the history snapshot at a
// batch's completion and returns at once; collect() — called when the next batch is planned,
// the first consumer of InfPT — waits for that fit and reports how long the fit took and how
// long the caller was blocked on it (Table V "optimization blocking").
class RefitWorker {
 public:
  struct Job {
    std::vector<double> thput, lat, infpt;   // Eq. 10 training rows (history)
    double target_thput = 0, target_lat = 0; // test inputs
  };
  RefitWorker() = default;
  RefitWorker(const RefitWorker&) = delete;
  RefitWorker& operator=(const RefitWorker&) = delete;
  ~RefitWorker();
  void submit(Job&& job);
  bool pending() const { return submitted_; }
  // Waits for the last submitted job.  Returns true with the predicted InfPT when the fit
  // succeeded (false: insufficient / degenerate history, InfPT unchanged).
  bool collect(double& infpt, double& fit_s, double& block_s);

 private:
  void loop();
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  Job job_;
  bool has_job_ = false, done_ = false, stop_ = false, submitted_ = false, ok_ = false;
  double out_ = 0, fit_s_ = 0;
};

double percentile_nearest_rank(std::vector<double> v, double p);

}  // namespace lms
