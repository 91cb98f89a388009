// tangram/event_log.hpp -- drop-in for the reference's scheduler event sink
// (event_log.hpp:29-45).  Same construction (output stream + policy name)
// and enabled(); the drop-in SloScheduler fills it with the batcher's JSON
// lines (keys sorted, "policy" added), byte-identical to the reference's
// nlohmann dump() lines, so no JSON library is needed.
#pragma once

#include <ostream>
#include <string>
#include <utility>

namespace tangram {

class EventLog {
 public:
  EventLog() = default;
  EventLog(std::ostream* out, std::string policy) : out_(out), policy_(std::move(policy)) {}

  bool enabled() const { return out_ != nullptr; }
  const std::string& policy() const { return policy_; }

  // Appends already-formatted JSON lines (each ending in '\n').
  void write_lines(const std::string& lines) {
    if (out_ != nullptr) (*out_) << lines;
  }

 private:
  std::ostream* out_ = nullptr;
  std::string policy_;
};

}  // namespace tangram
