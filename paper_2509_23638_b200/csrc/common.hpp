// Internal helpers shared by the host C++ and the CUDA translation units.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "ps_api.h"

namespace ps {

// Internal error type: carries the C-ABI status; converted at the boundary (capi.cpp).
struct Error : std::runtime_error {
  ps_status status;
  Error(ps_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(ps_status s, const std::string& msg) { throw Error(s, msg); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) fail(PS_EINVAL, msg);
}

void set_last_error(const std::string& msg);

// Runs f, mapping exceptions to ps_status (tools/prescope_main.cpp:427-434 semantics).
template <typename F>
ps_status guarded(F&& f) noexcept {
  try {
    f();
    return PS_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return PS_EINVAL;
  } catch (const std::out_of_range& e) {
    set_last_error(e.what());
    return PS_ERANGE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PS_ERUNTIME;
  } catch (...) {
    set_last_error("unknown exception");
    return PS_ERUNTIME;
  }
}

}  // namespace ps
