// Experiment drivers behind the C ABI's iluamg_run_* entry points: the same
// reports (ordered scalars + CSV tables, %.16e numbers) as the reference's
// src/driver.cpp, produced by the device solve phase.
#pragma once

#include "../host/config.hpp"
#include "solver.hpp"

#include <string>
#include <utility>
#include <vector>

namespace ilug {

struct ReportTable {
    std::string name;
    std::vector<std::string> columns;
    std::vector<std::vector<std::string>> rows;
    std::string csv() const;
};

struct Report {
    std::vector<std::pair<std::string, std::string>> scalars;
    std::vector<ReportTable> tables;
    int status = 0;
    void add(const std::string& k, const std::string& v) { scalars.emplace_back(k, v); }
    void add(const std::string& k, const char* v) { scalars.emplace_back(k, std::string(v)); }
    void add(const std::string& k, double v);
    void add(const std::string& k, i64 v) { add(k, std::to_string(v)); }
    void add(const std::string& k, bool v) { add(k, std::string(v ? "true" : "false")); }
    const std::string* find(const std::string& k) const;
    std::string text() const;
    std::string json() const;
};

std::string format_num(double v); ///< %.16e

/// Binds the config's device (device.id) and owns one stream for a run.
struct DeviceContext {
    cudaStream_t stream = nullptr;
    explicit DeviceContext(const Config& c);
    ~DeviceContext();
    DeviceContext(const DeviceContext&) = delete;
    DeviceContext& operator=(const DeviceContext&) = delete;
};

Report run_solve(const Csr& A, const Config& cfg, const std::string& label);
Report run_bench_trisolve(const Csr& A, const Config& cfg, const std::string& label);
Report run_schur_solve(const Csr& A, const Config& cfg, const std::string& label);
Report run_analyze(const Csr& A, const Config& cfg, const std::string& label);

} // namespace ilug
