// memplan — drop-in planner API of the B200 chunk runtime.
// Error vocabulary. Mirrors the reference contract proj/include/memplan/errors.hpp:10-37:
// every domain failure is a memplan::Error whose name() is the stable
// identifier the CLI prints (exit code 1) and whose what() reads
// "<Name>: <message>".
#pragma once

#include <stdexcept>
#include <string>
#include <utility>

namespace memplan {

class Error : public std::runtime_error {
 public:
  Error(std::string name, const std::string& msg)
      : std::runtime_error(name + ": " + msg), tag_(std::move(name)) {}
  const std::string& name() const { return tag_; }

 private:
  std::string tag_;
};

namespace detail {
// Fixed-string tag so each error type carries its own stable name.
template <std::size_t N>
struct Tag {
  char text[N];
  constexpr Tag(const char (&s)[N]) {
    for (std::size_t i = 0; i < N; ++i) text[i] = s[i];
  }
};
template <Tag T>
class NamedError : public Error {
 public:
  explicit NamedError(const std::string& msg) : Error(T.text, msg) {}
};
}  // namespace detail

// Trace / profile / plan input that cannot be parsed or has unknown keys.
class MalformedTrace : public detail::NamedError<"MalformedTrace"> { using NamedError::NamedError; };
// A structural invariant of a trace, profile or configuration does not hold.
class InvariantViolation : public detail::NamedError<"InvariantViolation"> { using NamedError::NamedError; };
class BlockOutOfRange : public detail::NamedError<"BlockOutOfRange"> { using NamedError::NamedError; };
class ZeroBandwidth : public detail::NamedError<"ZeroBandwidth"> { using NamedError::NamedError; };
// A packing unit (whole block / parameter op) is larger than the chunk.
class ChunkTooSmall : public detail::NamedError<"ChunkTooSmall"> { using NamedError::NamedError; };
class NoFeasibleChunkSize : public detail::NamedError<"NoFeasibleChunkSize"> { using NamedError::NamedError; };
class OutOfRange : public detail::NamedError<"OutOfRange"> { using NamedError::NamedError; };
class InfeasibleLayout : public detail::NamedError<"InfeasibleLayout"> { using NamedError::NamedError; };
class NoFeasibleConfig : public detail::NamedError<"NoFeasibleConfig"> { using NamedError::NamedError; };
class DeadlockDetected : public detail::NamedError<"DeadlockDetected"> { using NamedError::NamedError; };
class LedgerUnderflow : public detail::NamedError<"LedgerUnderflow"> { using NamedError::NamedError; };
class UnknownPreset : public detail::NamedError<"UnknownPreset"> { using NamedError::NamedError; };

}  // namespace memplan
