// Internal glue between the C ABI translation units.
#pragma once
#include <string>

#include "../../include/sdrt.h"
#include "mesh.h"
#include "refel.h"

struct sdrt_mesh {
  sdrt::Mesh m;
};
struct sdrt_operators {
  sdrt::Operators o;
};

namespace sdrt {
void set_error(const std::string& msg);
}

#define SDRT_TRY(...)                                              \
  try {                                                             \
    __VA_ARGS__                                                     \
  } catch (const std::invalid_argument& e) {                        \
    sdrt::set_error(e.what());                                      \
    return SDRT_E_INVALID_ARG;                                      \
  } catch (const std::exception& e) {                               \
    std::string w = e.what();                                       \
    sdrt::set_error(w);                                             \
    if (w.find("unsupported") != std::string::npos ||               \
        w.find("no simplex rule") != std::string::npos)             \
      return SDRT_E_UNSUPPORTED;                                    \
    if (w.find("ill-conditioned") != std::string::npos)             \
      return SDRT_E_ILL_CONDITIONED;                                \
    return SDRT_E_INTERNAL;                                         \
  }
