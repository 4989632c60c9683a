// Exception -> status-code conversion at the C ABI (no C++ exception crosses it).
#pragma once

#include <exception>
#include <new>
#include <string>

#include "common.cuh"

namespace rp {

void set_last_error(const std::string& msg);

template <class F>
int guard(F&& f) {
  try {
    f();
    return RP_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("out of memory: ") + e.what());
    return RP_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return RP_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown error");
    return RP_ERR_INTERNAL;
  }
}

}  // namespace rp
