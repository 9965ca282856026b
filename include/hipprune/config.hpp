// hipprune (B200) — config.hpp (subset of reference include/hipprune/config.hpp):
// the Appendix C plan presets. The CLI's config-file / override plumbing stays on
// the Python side (hipprune.run_report / config_hash).
#pragma once

#include <string>

#include "hipprune/pruning.hpp"

namespace hipprune {

// "3k", "5k", "fast", "flash" (config.cpp:64-86)
PruningPlan preset_plan(const std::string& name);

}  // namespace hipprune
