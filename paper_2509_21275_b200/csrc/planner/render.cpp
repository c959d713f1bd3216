// epp-b200 planner: SVG Gantt chart of traces (one lane per stage, one bar
// per F/B/R event, one memory sparkline per stage).  Used to eyeball
// simulated vs measured GPU traces; the element classes ("bar", "mem") and
// lane labels ("stage N") follow the reference's render contract
// (proj/include/epp/render.hpp:12-16, tests/test_docs.cpp:95-157).
#include <algorithm>
#include <sstream>

#include "epp/render.hpp"

namespace epp {

namespace {

const char* event_colour(EventKind k) {
    switch (k) {
        case EventKind::Forward: return "#4c78a8";
        case EventKind::Backward: return "#f58518";
        case EventKind::Recompute: return "#e45756";
    }
    return "#999999";
}

}  // namespace

std::string render_svg(const std::vector<SimTrace>& traces) {
    if (traces.empty()) throw ContractError("nothing to render");
    for (const SimTrace& t : traces)
        if (t.events.empty() || t.memory_series.empty())
            throw ContractError("cannot render a trace without events");

    constexpr double kWidth = 1000.0, kLeft = 80.0, kLane = 28.0, kSpark = 18.0;
    int lanes = 0;
    for (const SimTrace& t : traces) lanes += static_cast<int>(t.memory_series.size());
    const double height = 40.0 + lanes * (kLane + kSpark) + 20.0 * traces.size();

    std::ostringstream svg;
    svg << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << kWidth + kLeft + 20
        << "\" height=\"" << height << "\">\n";
    double y = 20.0;
    for (size_t u = 0; u < traces.size(); ++u) {
        const SimTrace& t = traces[u];
        const double span = t.makespan > 0 ? t.makespan : 1.0;
        const double sx = kWidth / span;
        svg << "<text x=\"4\" y=\"" << y << "\">unit " << u << " makespan " << t.makespan
            << " s</text>\n";
        y += 8.0;
        const int stages = static_cast<int>(t.memory_series.size());
        for (int p = 0; p < stages; ++p) {
            const double top = y + p * (kLane + kSpark);
            svg << "<text x=\"4\" y=\"" << top + kLane * 0.7 << "\">stage " << p + 1
                << "</text>\n";
            for (const SimEvent& e : t.events) {
                if (e.stage != p + 1) continue;
                svg << "<rect class=\"bar\" x=\"" << kLeft + e.start * sx << "\" y=\"" << top
                    << "\" width=\"" << std::max(0.5, (e.end - e.start) * sx)
                    << "\" height=\"" << kLane - 4 << "\" fill=\"" << event_colour(e.kind)
                    << "\"><title>" << to_string(e.kind) << " chunk " << e.chunk_id
                    << "</title></rect>\n";
            }
            double peak = 1.0;
            for (const auto& pt : t.memory_series[p]) peak = std::max(peak, pt.second);
            svg << "<polyline class=\"mem\" fill=\"none\" stroke=\"#54a24b\" points=\"";
            for (const auto& pt : t.memory_series[p])
                svg << kLeft + pt.first * sx << ","
                    << top + kLane + kSpark - 2 - (kSpark - 4) * pt.second / peak << " ";
            svg << "\"/>\n";
        }
        y += stages * (kLane + kSpark) + 12.0;
    }
    svg << "</svg>\n";
    return svg.str();
}

}  // namespace epp
