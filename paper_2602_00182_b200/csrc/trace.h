// Per-CTA timeline record (timing instrumentation: detgpu_set_option "trace", tools/trace_step.py).
#pragma once
#include <cstdint>

namespace detgpu {

struct TraceRec {
    uint32_t tag;          // kernel class << 24 | linear CTA index
    uint32_t sm;
    uint64_t t[15];        // globaltimer ns: [0] CTA start, [1] dependency wait released,
                           // [2..13] kernel-specific phase marks (0 = unused), [14] CTA end
};
constexpr int kTraceMarks = 14;

}  // namespace detgpu
