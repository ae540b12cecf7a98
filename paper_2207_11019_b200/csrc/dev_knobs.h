// Development knobs: timing probes that drop work (wrong results) and the
// alternative paths that measured slower than the default (numbers next to
// each use).  They exist only in a -DPPB_DEV_KNOBS build (`make DEV=1`); in
// the release library (the one the tests, smoke() and bench.py load) every
// knob is a compile-time constant off, so no environment variable can change
// what a training step computes.
#pragma once

#ifdef PPB_DEV_KNOBS
#include <cstdlib>
namespace ppb {
inline bool dev_knob(const char* name) {
    const char* e = std::getenv(name);
    return e != nullptr && *e != '\0' && *e != '0';
}
inline unsigned dev_knob_uint(const char* name) {
    const char* e = std::getenv(name);
    return e != nullptr ? static_cast<unsigned>(std::strtoul(e, nullptr, 0)) : 0u;
}
}  // namespace ppb
#else
namespace ppb {
constexpr bool dev_knob(const char*) { return false; }
constexpr unsigned dev_knob_uint(const char*) { return 0u; }
}  // namespace ppb
#endif
