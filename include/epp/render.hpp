// epp-b200 planner: SVG Gantt view of simulated or measured traces
// (API of proj/include/epp/render.hpp:12-16).
#pragma once

#include <string>
#include <vector>

#include "epp/pipeline.hpp"

namespace epp {

std::string render_svg(const std::vector<SimTrace>& traces);

}  // namespace epp
