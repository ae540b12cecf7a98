// Error plumbing for the C ABI: C++ exceptions never cross the boundary; each
// entry point returns a status code and leaves the message in a thread-local
// slot (ppb_last_error), so the C++ drop-in shim can rethrow the reference's
// exception type with the reference's text.
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/pipeplan_b200.h"

void ppb_set_error(const std::string& msg);

// Run `f` and translate exceptions to PPB_* codes.
template <class F>
int ppb_guard(F&& f) {
    try {
        f();
        return PPB_OK;
    } catch (const std::invalid_argument& e) {
        ppb_set_error(e.what());
        return PPB_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        ppb_set_error(e.what());
        return PPB_ERR_OUT_OF_RANGE;
    } catch (const std::runtime_error& e) {
        ppb_set_error(e.what());
        return PPB_ERR_RUNTIME;
    } catch (const std::exception& e) {
        ppb_set_error(e.what());
        return PPB_ERR_RUNTIME;
    } catch (...) {
        ppb_set_error("unknown error");
        return PPB_ERR_RUNTIME;
    }
}
