// stabkit/error.hpp -- exception hierarchy of the stabkit host API.
// API-compatible with the reference header (ref: proj/include/stabkit/error.hpp:25-51):
// same type names, same base/derived relations, ParseError carries `line` (0 = no location).
// Added: throw_status(), which turns an sk_status from the C ABI (stabkit_b200.h) back into
// the matching exception, so no exception ever crosses the C boundary.
#pragma once
#include <cstddef>
#include <stdexcept>
#include <string>

namespace stabkit {

class Error : public std::runtime_error {
  public:
    explicit Error(const std::string& message) : std::runtime_error(message) {}
    explicit Error(const char* message) : std::runtime_error(message) {}
};

// malformed text input; `line` is 1-based, 0 when unknown
class ParseError : public Error {
  public:
    ParseError(size_t line_number, const std::string& what)
        : Error(line_number == 0 ? what : "line " + std::to_string(line_number) + ": " + what), line(line_number) {}
    size_t line;
};

class DimensionError : public Error { public: using Error::Error; };     // size / index mismatch
class UnsupportedError : public Error { public: using Error::Error; };   // valid construct, wrong code path
class InvariantError : public Error { public: using Error::Error; };     // internal consistency failure

// sk_status -> exception (1 EDIM, 2 EUNSUPPORTED, 3 EINVARIANT, 5 ENCCL -> Error, 6 EPARSE, anything else Error)
[[noreturn]] inline void throw_status(int code, const std::string& message) {
    switch (code) {
        case 1: throw DimensionError(message);
        case 2: throw UnsupportedError(message);
        case 3: throw InvariantError(message);
        case 5: throw Error("NCCL: " + message);            // SK_ENCCL (stabkit/nccl_exchange.hpp)
        case 6: throw ParseError(0, message);
        default: throw Error(message);
    }
}

}  // namespace stabkit
