// dmc/errors.hpp — the reference error taxonomy (reference
// include/dmc/errors.hpp:24-61): dmc::Error{code(), kind()} and its 19
// subclasses with the same codes, so a reference caller's catch clauses work
// unchanged.  detail::raise() maps a libdmcg return code + "<Kind>: <message>"
// string (dmcg_last_error / dmcg_parse_error / dmcg_host_error) back onto the
// matching subclass.
#pragma once

#include <stdexcept>
#include <string>

namespace dmc {

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& kind, const std::string& what)
      : std::runtime_error(kind + ": " + what), code_(code), kind_(kind) {}
  int code() const { return code_; }
  const std::string& kind() const { return kind_; }

 private:
  int code_;
  std::string kind_;
};

#define DMC_DEFINE_ERROR(Name, Code)                                              \
  class Name : public Error {                                                     \
   public:                                                                        \
    explicit Name(const std::string& what) : Error(Code, #Name, what) {}          \
  }

DMC_DEFINE_ERROR(DimensionMismatch, 5);
DMC_DEFINE_ERROR(IndexOutOfRange, 4);
DMC_DEFINE_ERROR(DegenerateFace, 4);
DMC_DEFINE_ERROR(ValidationError, 4);
DMC_DEFINE_ERROR(ConfigError, 5);
DMC_DEFINE_ERROR(InvalidBits, 5);
DMC_DEFINE_ERROR(InvalidCount, 5);
DMC_DEFINE_ERROR(BlockSizeError, 5);
DMC_DEFINE_ERROR(ConvergenceFailure, 9);
DMC_DEFINE_ERROR(RankDeficiency, 9);
DMC_DEFINE_ERROR(SignMisalignment, 9);
DMC_DEFINE_ERROR(SingularSystem, 9);
DMC_DEFINE_ERROR(CorruptPayload, 6);
DMC_DEFINE_ERROR(CorruptStream, 6);
DMC_DEFINE_ERROR(VersionMismatch, 7);
DMC_DEFINE_ERROR(ParseError, 3);
DMC_DEFINE_ERROR(VertexCountMismatch, 3);
DMC_DEFINE_ERROR(ConnectivityMismatch, 3);
DMC_DEFINE_ERROR(IoError, 8);
// B200-only failures (libdmcg codes 10 / 11): a CUDA runtime or launch error,
// and a request outside the GPU path (per_mesh_gft, raw payloads, ...).
DMC_DEFINE_ERROR(CudaError, 10);
DMC_DEFINE_ERROR(Unsupported, 11);

#undef DMC_DEFINE_ERROR

namespace detail {
// Throws the subclass named by the message's "<Kind>: " prefix (falling back
// to a plain dmc::Error with the libdmcg code).
[[noreturn]] inline void raise(int code, const std::string& msg) {
  const size_t colon = msg.find(": ");
  const std::string kind = colon == std::string::npos ? std::string() : msg.substr(0, colon);
  const std::string what = colon == std::string::npos ? msg : msg.substr(colon + 2);
#define DMC_RAISE_IF(Name) \
  if (kind == #Name) throw Name(what)
  DMC_RAISE_IF(DimensionMismatch);
  DMC_RAISE_IF(IndexOutOfRange);
  DMC_RAISE_IF(DegenerateFace);
  DMC_RAISE_IF(ValidationError);
  DMC_RAISE_IF(ConfigError);
  DMC_RAISE_IF(InvalidBits);
  DMC_RAISE_IF(InvalidCount);
  DMC_RAISE_IF(BlockSizeError);
  DMC_RAISE_IF(ConvergenceFailure);
  DMC_RAISE_IF(RankDeficiency);
  DMC_RAISE_IF(SignMisalignment);
  DMC_RAISE_IF(SingularSystem);
  DMC_RAISE_IF(CorruptPayload);
  DMC_RAISE_IF(CorruptStream);
  DMC_RAISE_IF(VersionMismatch);
  DMC_RAISE_IF(ParseError);
  DMC_RAISE_IF(VertexCountMismatch);
  DMC_RAISE_IF(ConnectivityMismatch);
  DMC_RAISE_IF(IoError);
  DMC_RAISE_IF(CudaError);
  DMC_RAISE_IF(Unsupported);
#undef DMC_RAISE_IF
  if (code == 10) throw CudaError(what);
  if (code == 11) throw Unsupported(what);
  throw Error(code, kind.empty() ? "Error" : kind, what);
}
}  // namespace detail

}  // namespace dmc
