// GPU execution API (new in this framework; no reference counterpart beyond
// the simulate() entry points it implements, ref simulate.hpp:23-36).
//
// An Executor owns one et_runtime (include/et_runtime.h): it flattens every
// sampled schedule of a lowered kernel into device arrays once, binds a tile
// operation to every call, and then runs one persistent-kernel launch per
// step at any covered binding without re-lowering or recompiling.
#pragma once

#include <memory>

#include "et_runtime.h"
#include "etsim/simulate.hpp"

namespace etsim {

struct ExecConfig {
    int device = 0;
    int num_workers = 0;        // 0: the kernel's num_sms
    bool record_trace = true;   // per-slot %globaltimer records
    bool enable_prefetch = true;
    Int watchdog_ns = 2'000'000'000;
    Int tick_ns = 0;            // synthetic task body: ns per duration unit
    Int seed = 0;               // duration-model seed for synthetic bodies
    Int step_limit = 0;         // > 0: SimError::StepLimit after this many tasks
    int max_batch = 1;          // largest GEMV batch (<= 8 on the mma.sync GEMV path)
    Int l2_prefetch_bytes = -1; // per worker L2 run-ahead beyond the smem ring (-1: default)
};

struct StepStats {
    int sample_index = -1;
    Int tasks_executed = 0;
    Int noop_tasks = 0;
    Int pushes = 0;
    Int pops = 0;
    double kernel_ms = 0;
};

class Executor {
public:
    Executor(const StaticMegakernel& k, const ExecConfig& cfg);
    // Dynamic scheduler: one device program per sampled binding (any covered
    // binding runs on the next-larger sample with masked no-ops); data-dependent
    // routing is resolved on the device.
    Executor(const DynamicMegakernel& k, const std::vector<ShapeBinding>& samples, const ExecConfig& cfg);
    // Ahead-of-time program image (et_save_program / et_load_program): a static
    // executor saved once loads without lowering or flattening; the graph rides
    // along as the image's metadata (reference JSON), so traces keep working.
    static std::unique_ptr<Executor> load_program(const std::string& path, const ExecConfig& cfg);
    void save_program(const std::string& path) const;
    ~Executor();
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;

    // One op per call (index = call index); calls left unbound run the
    // synthetic body.
    void bind_ops(const std::vector<et_op>& ops);
    void set_runtime_tensor(const std::string& name, const std::vector<Int>& values);
    void set_realization(const RoutingRealization& r);
    std::vector<Int> runtime_tensor(const std::string& name, size_t n) const;

    StepStats run(const ShapeBinding& binding);                     // synchronous, throws on failure
    void launch(const ShapeBinding& binding, void* stream = nullptr);  // enqueue only
    StepStats sync();

    Trace trace() const;                    // last step, reference Trace form (measured ns)
    std::vector<et_trace_rec> raw_trace() const;  // last step, device records in slot / task order
    std::vector<Int> final_counters() const;
    const StaticMegakernel& kernel() const;
    bool dynamic() const;
    int num_workers() const;
    double upload_ms() const;
    void set_debug(int bits);  // diagnostics: megakernel debug bits (et_set_debug)
    void set_l2_prefetch(Int bytes);  // producer L2 run-ahead per worker (et_set_l2_prefetch)

private:
    Executor();
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

// Throws etsim::Error / SimError according to an et_status code.
void raise_status(int code, const std::string& what);

bool gpu_available();

}  // namespace etsim
