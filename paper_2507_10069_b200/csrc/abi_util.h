// abi_util.h — error plumbing shared by the extern "C" entry points.
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include "host_cache.h"

namespace emm_abi {
void set_error(const std::string& s);
}

// Run `body`; map C++ exceptions to EMM_E_* status codes + emm_last_error().
#define EMM_GUARD(body)                                   \
  try {                                                   \
    body;                                                 \
    return 0;                                             \
  } catch (const emm::CacheError& e) {                    \
    emm_abi::set_error(e.msg);                            \
    return e.code;                                        \
  } catch (const std::bad_alloc&) {                       \
    emm_abi::set_error("host allocation failed");         \
    return 4;                                             \
  } catch (const std::exception& e) {                     \
    emm_abi::set_error(e.what());                         \
    return 5;                                             \
  }
