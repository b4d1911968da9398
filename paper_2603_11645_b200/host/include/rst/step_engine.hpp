// rst/step_engine.hpp -- the run context every strategy receives
// (reference: include/rst/step_engine.hpp:36-93).
//
// On the B200 engine there is no host thread pool: a "step" is a
// device-wide barrier of the CUDA pipeline (kernel boundary or grid
// barrier) and `work` counts element updates. The counters are filled from
// the device statistics after each call, so code that reads steps()/work()
// keeps working. `workers` is accepted for signature compatibility and
// ignored; `device` selects the GPU.
#pragma once

#include <chrono>
#include <cstdint>

namespace rst {

struct StepReport {
  std::int64_t steps = 0;
  std::int64_t work = 0;
  double wall_ms = 0.0;
};

class StepEngine {
 public:
  explicit StepEngine(int workers = 1, int device = 0)
      : workers_(workers < 1 ? 1 : workers), device_(device),
        start_(std::chrono::steady_clock::now()) {}
  StepEngine(const StepEngine&) = delete;
  StepEngine& operator=(const StepEngine&) = delete;

  int workers() const { return workers_; }
  int device() const { return device_; }
  std::int64_t steps() const { return steps_; }
  std::int64_t work() const { return work_; }
  // Device-side figures of the last call.
  double device_ms() const { return device_ms_; }
  std::int64_t launches() const { return launches_; }

  void charge(std::int64_t extra_steps, std::int64_t extra_work = 0) {
    steps_ += extra_steps;
    work_ += extra_work;
  }
  void record_device(std::int64_t steps, std::int64_t work, std::int64_t launches, double ms) {
    steps_ += steps;
    work_ += work;
    launches_ += launches;
    device_ms_ = ms;
  }
  StepReport report() const {
    StepReport r;
    r.steps = steps_;
    r.work = work_;
    r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start_)
                    .count();
    return r;
  }

 private:
  int workers_;
  int device_;
  std::int64_t steps_ = 0;
  std::int64_t work_ = 0;
  std::int64_t launches_ = 0;
  double device_ms_ = 0.0;
  std::chrono::steady_clock::time_point start_;
};

}  // namespace rst
