// Error taxonomy shared by the host side of the C ABI. Codes follow the
// reference fe2rom::ErrorCode (common.hpp:26-37); the ABI returns
// 1 + ordinal and keeps the message for fe2_last_error().
#pragma once

#include <stdexcept>
#include <string>

namespace fe2 {

enum class Code { config, geometry, mesh, material, solver, numeric, rank, bc, io, provenance };

struct Failure : std::runtime_error {
  Failure(Code c, const std::string& what) : std::runtime_error(what), code(c) {}
  Code code;
};

inline void check(bool ok, Code c, const std::string& what) {
  if (!ok) throw Failure(c, what);
}

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return 1 + static_cast<int>(e.code);
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1 + static_cast<int>(Code::numeric);
  }
}

}  // namespace fe2
