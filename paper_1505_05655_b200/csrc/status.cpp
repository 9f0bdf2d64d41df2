// status.cpp -- names and response codes of gpcx::Errc.  The name table is
// gpc::errc_name (proj/src/error.cpp:5-36); the response code table is the
// closed set of proj/src/registry.cpp:38-60.
#include "status.hpp"

namespace gpcx {

const char* errc_name(Errc code) {
  static const char* const kNames[kErrcCount] = {
      "FieldTooLong",     "InvalidCharacter", "BadMarker",       "MalformedPadding",
      "DuplicateKey",     "BadToken",         "MissingParam",    "BadValue",
      "Overflow",         "Truncated",        "PayloadMismatch", "UnknownTask",
      "DuplicateFlag",    "TaskFailed",       "BadImage",        "InsufficientPoints",
      "Singular",         "OrderTooHigh",     "ConnectFailed",   "BindFailed",
      "TimedOut",         "IoError",          "UnsafeName",      "SizeMismatch",
      "BadFormat",        "TooLarge",         "ServerError"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < kErrcCount) ? kNames[i] : "Unknown";
}

std::string response_code(Errc code) {
  switch (code) {
    case Errc::UnknownTask: return "UNKNOWN_TASK";
    case Errc::MissingParam: return "MISSING_PARAM";
    case Errc::PayloadMismatch: return "PAYLOAD_MISMATCH";
    case Errc::Overflow:
    case Errc::TooLarge: return "TOO_LARGE";
    case Errc::FieldTooLong:
    case Errc::InvalidCharacter:
    case Errc::BadMarker:
    case Errc::MalformedPadding:
    case Errc::DuplicateKey:
    case Errc::BadToken:
    case Errc::BadValue: return "BAD_HEADER";
    default: return "TASK_FAILED";
  }
}

}  // namespace gpcx
