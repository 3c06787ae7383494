// error.hpp -- the error family of the host layer.  Same taxonomy and names as the
// reference's sf::Error hierarchy (proj/include/sf/error.hpp:9-59) so that callers'
// catch clauses keep their meaning; the C-ABI status codes of sfb200.h map onto it.
#pragma once

#include <stdexcept>
#include <string>

#if defined(__GNUC__)
#define SFB_PUBLIC __attribute__((visibility("default")))  // one typeinfo across shared objects
#else
#define SFB_PUBLIC
#endif

namespace sfb {

struct SFB_PUBLIC Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct SFB_PUBLIC OrderError : Error { using Error::Error; };       // bad stencil / space order
struct SFB_PUBLIC LocationError : Error { using Error::Error; };    // sparse point outside the grid
struct SFB_PUBLIC BindingError : Error { using Error::Error; };     // operator inputs incomplete
struct SFB_PUBLIC ParameterError : Error { using Error::Error; };   // bad user parameter
struct SFB_PUBLIC StabilityError : Error { using Error::Error; };   // CFL violated or NaN at run time
struct SFB_PUBLIC CapabilityError : Error { using Error::Error; };  // no usable B200 / kernel image

// throws the member of the family that corresponds to a C-ABI status code
[[noreturn]] void raise_status(int code, const std::string& message);

}  // namespace sfb
