// Host-side control of the LMStream micro-batch loop.  See host_control.h.
#include "host_control.h"

#include <chrono>

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>

namespace lms {

double est_max_lat(const double* buff_s, const uint64_t* bytes, uint64_t n, double avg_thput) {
  // Eq. 6: EstMaxLat_i = max_j Buff_(i,j) + sum_j Part_(i,j) / AvgThPut_{i-1}
  double mb = -std::numeric_limits<double>::infinity();
  double total = 0.0;
  for (uint64_t j = 0; j < n; j++) {
    mb = std::max(mb, buff_s[j]);
    total += (double)bytes[j];
  }
  return mb + total / avg_thput;
}

AdmitResult admit_decision(Mode mode, double slide_s, double deadline_s, double now_s,
                           const double* ingest_s, const uint64_t* bytes, uint64_t n,
                           double avg_thput, const double* maxlat_hist, uint64_t n_hist) {
  AdmitResult r;
  // Alg. 1 "if there is no new data: do polling" — reading R22: only when nothing is buffered.
  if (n == 0) { r.reason = kPoll; return r; }
  if (n >= kCapDatasets) { r.admit = true; r.reason = kAdmitCap; return r; }
  if (!(avg_thput > 0.0)) { r.admit = true; r.reason = kAdmitBootstrap; return r; }   // R15
  std::vector<double> buff(n);
  for (uint64_t j = 0; j < n; j++) buff[j] = now_s - ingest_s[j];                    // Buff_(i,j)
  r.est = est_max_lat(buff.data(), bytes, n, avg_thput);
  bool sliding;
  double target;
  if (mode == Mode::Deadline) { sliding = deadline_s > 0.0; target = deadline_s; }   // R16
  else { sliding = slide_s > 0.0; target = slide_s; }
  if (sliding) {
    if (r.est >= target) { r.admit = true; r.reason = kAdmitTarget; return r; }
  } else {
    if (n_hist < 2) { r.admit = true; r.reason = kAdmitTumblingBootstrap; return r; } // R11
    double s = 0.0;
    for (uint64_t k = 0; k < n_hist; k++) s += maxlat_hist[k];
    if (r.est >= s / (double)n_hist) { r.admit = true; r.reason = kAdmitTarget; return r; }
  }
  r.reason = kBuffer;   // "do buffering": bufferedFiles = tmpMicroBatch
  return r;
}

// ---------------------------------------------------------------- Alg. 2

double base_cost(int32_t k) {
  // Table III: Aggregation/Filtering/Shuffling 1.0; Projection/Join/Expand 0.9;
  // Scan (CSV)/Sorting 0.8.  Kinds: Scan0 Filter1 Project2 HashAgg3 HashJoin4 Sort5 Shuffle6 Expand7.
  static const double c[8] = {0.8, 1.0, 0.9, 1.0, 0.9, 0.8, 1.0, 0.9};
  return (k >= 0 && k < 8) ? c[k] : -1.0;
}

bool traverse(const Dag& dag, std::vector<int32_t>& order) {
  const int n = (int)dag.kind.size();
  order.clear();
  std::vector<int> succ(n, 0);
  for (int o = 0; o < n; o++)
    for (int p : dag.preds[o]) {
      if (p < 0 || p >= n) return false;
      succ[p]++;
    }
  int root = -1;
  for (int o = 0; o < n; o++)
    if (succ[o] == 0) { if (root >= 0) return false; root = o; }
  if (root < 0) return false;
  std::vector<int> state(n, 0);
  bool ok = true;
  std::function<void(int)> visit = [&](int o) {
    if (!ok) return;
    if (state[o] == 1) { ok = false; return; }
    if (state[o] == 2) return;
    state[o] = 1;
    for (int p : dag.preds[o]) visit(p);   // "Searching sequentially from the child node"
    state[o] = 2;
    order.push_back(o);
  };
  visit(root);
  return ok && (int)order.size() == n;
}

bool map_device(const Dag& dag, double part, double infpt, double btc, std::vector<uint8_t>& dev) {
  std::vector<int32_t> order;
  if (!traverse(dag, order)) return false;
  const int root = order.back();
  dev.assign(dag.kind.size(), 1);   // "Initially, map every operation in opDAG to the GPU"
  for (int o : order) {
    const double base = base_cost(dag.kind[o]);
    double cpu = base * (part / infpt);          // Eq. 7
    double gpu = base * (infpt / part);          // Eq. 8
    const double trans = btc * (part / infpt);   // Eq. 9
    bool prev_cpu = false;
    for (int p : dag.preds[o]) prev_cpu |= (dev[p] == 0);
    if (dag.preds[o].empty() || o == root || prev_cpu) gpu += trans;
    else cpu += trans;
    if (gpu > cpu) dev[o] = 0;
  }
  return true;
}

Dag query_dag(int32_t kind) {
  // LR1* diamond Scan -> Project x2 -> HashJoin -> Project; LR2S Scan -> Project ->
  // Shuffle -> HashAggregate -> Filter; CM1* Scan -> Project -> Shuffle -> HashAggregate -> Sort;
  // CM2S Scan -> Filter -> Shuffle -> HashAggregate.
  Dag d;
  auto add = [&](uint8_t k, std::vector<int32_t> p) { d.kind.push_back(k); d.preds.push_back(p); };
  switch (kind) {
    case 0: case 1:
      add(0, {}); add(2, {0}); add(2, {0}); add(4, {1, 2}); add(2, {3}); break;
    case 2:
      add(0, {}); add(2, {0}); add(6, {1}); add(3, {2}); add(1, {3}); break;
    case 3: case 4:
      add(0, {}); add(2, {0}); add(6, {1}); add(3, {2}); add(5, {3}); break;
    case 5:
      add(0, {}); add(1, {0}); add(6, {1}); add(3, {2}); break;
    default: break;
  }
  return d;
}

// ---------------------------------------------------------------- Eq. 10

bool infpt_fit(const double* thput, const double* lat, const double* infpt, uint64_t n, double b[3]) {
  // Eq. 10 OLS on regressors (1, thput[MB/s], lat[s]) in long double.  The regressors
  // are centred first (the normal equations of the intercept decouple: b0 = mean(y) - b1
  // mean(t) - b2 mean(l)), which removes the cancellation of the raw normal equations when
  // the cumulative AvgThPut (Eq. 4) settles; singular 2x2 -> insufficient history.
  if (n < 3) return false;
  long double mt = 0, ml = 0, my = 0;
  for (uint64_t r = 0; r < n; r++) { mt += thput[r] / 1e6L; ml += lat[r]; my += infpt[r]; }
  mt /= n; ml /= n; my /= n;
  long double stt = 0, sll = 0, stl = 0, sty = 0, sly = 0;
  for (uint64_t r = 0; r < n; r++) {
    const long double t = thput[r] / 1e6L - mt, l = lat[r] - ml, y = infpt[r] - my;
    stt += t * t; sll += l * l; stl += t * l; sty += t * y; sly += l * y;
  }
  const long double det = stt * sll - stl * stl;
  if (!(stt > 0) || !(sll > 0) || det <= stt * sll * 1e-15L) return false;
  const long double b1 = (sty * sll - sly * stl) / det, b2 = (sly * stt - sty * stl) / det;
  b[0] = (double)(my - b1 * mt - b2 * ml);
  b[1] = (double)b1;
  b[2] = (double)b2;
  return true;
}

double infpt_predict(const double b[3], double thput, double lat) {
  const double v = b[0] + b[1] * (thput / 1e6) + b[2] * lat;
  return std::min(16.0 * 1024 * 1024, std::max(1024.0, v));   // clamp
}

// ---------------------------------------------------------------- asynchronous Eq. 10 refit

static double mono_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

RefitWorker::~RefitWorker() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  if (th_.joinable()) th_.join();
}

void RefitWorker::submit(Job&& job) {
  {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !has_job_; });      // at most one fit outstanding
    job_ = std::move(job);
    has_job_ = true;
    done_ = false;
    submitted_ = true;
  }
  if (!th_.joinable()) th_ = std::thread(&RefitWorker::loop, this);
  cv_.notify_all();
}

bool RefitWorker::collect(double& infpt, double& fit_s, double& block_s) {
  const double t0 = mono_s();
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [&] { return done_; });
  block_s = mono_s() - t0;
  submitted_ = false;
  fit_s = fit_s_;
  if (ok_) infpt = out_;
  return ok_;
}

void RefitWorker::loop() {
  std::unique_lock<std::mutex> lk(mu_);
  while (true) {
    cv_.wait(lk, [&] { return stop_ || has_job_; });
    if (stop_) return;
    Job j = std::move(job_);
    lk.unlock();
    const double t0 = mono_s();
    double b[3];
    const bool ok = infpt_fit(j.thput.data(), j.lat.data(), j.infpt.data(), j.thput.size(), b);
    const double v = ok ? infpt_predict(b, j.target_thput, j.target_lat) : 0.0;
    const double dt = mono_s() - t0;
    lk.lock();
    ok_ = ok;
    out_ = v;
    fit_s_ = dt;
    has_job_ = false;
    done_ = true;
    cv_.notify_all();
  }
}

double percentile_nearest_rank(std::vector<double> v, double p) {
  std::sort(v.begin(), v.end());
  const double n = (double)v.size();
  long rank = (long)std::ceil(p / 100.0 * n - 1e-12);
  rank = std::max(1L, std::min(rank, (long)v.size()));
  return v[rank - 1];
}

}  // namespace lms
