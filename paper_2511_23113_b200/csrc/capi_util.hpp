// Shared exception -> status translation for the C ABI translation units.
#pragma once

#include <exception>
#include <new>
#include <string>

#include "core.hpp"

namespace dbsp_capi {

int record(int code, const char* what);

template <class F>
int guard(F&& body) {
  try {
    body();
    return dbsp_core::kOk;
  } catch (const dbsp_core::Error& e) {
    return record(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return record(dbsp_core::kInternal, "out of host memory");
  } catch (const std::exception& e) {
    return record(dbsp_core::kInternal, e.what());
  } catch (...) {
    return record(dbsp_core::kInternal, "unknown exception");
  }
}

}  // namespace dbsp_capi
