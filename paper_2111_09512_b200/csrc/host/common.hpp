// Shared host-side vocabulary: error kinds, thread pool helpers, index types.
//
// Error semantics mirror the reference (include/iluamg/error.hpp:11-34):
// invalid/io map to status 2 and numeric to 3 at the C ABI; no exception
// crosses the ABI (csrc/host/capi.cpp).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace ilug {

using i64 = std::int64_t;
using i32 = std::int32_t;
using Vec = std::vector<double>;

enum class ErrorKind { invalid, io, numeric };

class Error : public std::runtime_error {
public:
    Error(ErrorKind k, const std::string& m) : std::runtime_error(m), kind_(k) {}
    ErrorKind kind() const noexcept { return kind_; }

private:
    ErrorKind kind_;
};

[[noreturn]] inline void fail_invalid(const std::string& m) { throw Error(ErrorKind::invalid, m); }
[[noreturn]] inline void fail_io(const std::string& m) { throw Error(ErrorKind::io, m); }
[[noreturn]] inline void fail_numeric(const std::string& m) { throw Error(ErrorKind::numeric, m); }

/// Worker count for host setup loops (ILUG_THREADS overrides).
int host_threads();

/// Static block partition of [0, n) over the worker pool; fn(begin, end, tid).
/// Every loop that uses it writes disjoint outputs, so results never depend on
/// the thread count (bitwise reproducibility is a parity requirement).
void parallel_ranges(i64 n, const std::function<void(i64, i64, int)>& fn, i64 grain = 4096);

/// ILUG_TRACE_SETUP=1: wall time of setup phases on stderr (diagnostics only).
class SetupTimer {
public:
    explicit SetupTimer(const char* scope);
    void mark(const char* phase, i64 level = -1);
    bool on() const { return on_; }

private:
    const char* scope_;
    bool on_;
    double t_;
};

} // namespace ilug
