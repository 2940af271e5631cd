// logs.cu — the reference's decision-log wire format for GPU replays, so replay
// output drops into the reference's report tooling unchanged:
//   decisions_csv  metrics.hpp:145-157 (schema and field order)
//   fmt_num        csvio.hpp:17-21     ("%.10g" through the C library's printf)
//   to_string      controller.hpp:72-82 (reason strings)
//   fnv1a64        rng.hpp:22-28        (the per-file hash run manifests record,
//                                        commands.hpp:26-39, csvio.hpp:69-71)
// Host code only: formatting is a few hundred bytes per logged step and stays off
// the device, exactly as the reference formats after its simulation.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "pals_internal.cuh"

namespace {

const char* reason_string(int r) {
    switch (r) {
        case PALS_REASON_QOS_FEASIBLE: return "qos-feasible-max-efficiency";
        case PALS_REASON_FALLBACK_MAX_T: return "fallback-max-throughput";
        case PALS_REASON_BUDGET_MAX_T: return "budget-constrained-max-throughput";
        case PALS_REASON_HOLD: return "hold-hysteresis";
        case PALS_REASON_ORACLE: return "oracle-exhaustive";
    }
    return "?";
}

void put_num(std::string& out, double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.10g", v);
    out += buf;
}

}  // namespace

extern "C" {

int pals_decisions_csv(const pals_replay_spec* spec, const pals_profile* plant, int32_t n_models,
                       const double* caps, int32_t n_caps, const int32_t* batches,
                       int32_t n_batches, const pals_trace_summary* summaries,
                       const pals_step_log* logs, const pals_step_detail* details, char* buf,
                       int64_t buf_size, int64_t* out_len) {
    using namespace pals;
    if (!spec || !out_len) return set_error(PALS_ECONFIG, "pals_decisions_csv: null argument");
    const int64_t nl = std::max<int64_t>(0, std::min<int64_t>(spec->n_log_traces, spec->n_traces));
    if (nl > 0 && (!plant || n_models <= 0 || !caps || n_caps <= 0 || !batches ||
                   n_batches <= 0 || !summaries || !logs || !details))
        return set_error(PALS_ECONFIG, "pals_decisions_csv: null argument");
    const int64_t n_cands = (int64_t)n_caps * n_batches;
    std::string out = "node,model,t_s,cap_w,batch,tp,ep,dp,applied,reason,err_norm,bias\n";
    out.reserve(out.size() + (size_t)(nl * std::max(0, spec->n_steps)) * 96);
    for (int64_t i = 0; i < nl; ++i) {
        const int m = summaries[i].model;
        if (m < 0 || m >= n_models)
            return set_error(PALS_ECONFIG, "pals_decisions_csv: summary model out of range");
        const pals_profile& p = plant[m];
        const std::string node = std::to_string(spec->first_trace + i);
        const std::string tail_dims = "," + std::to_string(p.deploy_tp) + "," +
                                      std::to_string(p.deploy_ep) + "," +
                                      std::to_string(p.deploy_dp) + ",";
        for (int k = 0; k < spec->n_steps; ++k) {
            const int64_t o = i * (int64_t)spec->n_steps + k;
            const pals_step_log& lg = logs[o];
            if (lg.idx < 0 || lg.idx >= n_cands)
                return set_error(PALS_ECONFIG, "pals_decisions_csv: candidate index out of range");
            const double t1 = (double)k * spec->interval_s + spec->interval_s;  // replay t1
            out += node;
            out += ',';
            out += p.name;
            out += ',';
            put_num(out, t1);
            out += ',';
            put_num(out, caps[lg.idx / n_batches]);
            out += ',';
            out += std::to_string(batches[lg.idx % n_batches]);
            out += tail_dims;
            out += lg.applied ? "1," : "0,";
            out += reason_string(lg.reason);
            out += ',';
            put_num(out, details[o].err_norm);
            out += ',';
            put_num(out, details[o].bias);
            out += '\n';
        }
    }
    *out_len = (int64_t)out.size();
    if (buf && buf_size > 0) std::memcpy(buf, out.data(), (size_t)std::min<int64_t>(buf_size, *out_len));
    return PALS_OK;
}

uint64_t pals_fnv1a64(const void* data, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const unsigned char* b = (const unsigned char*)data;
    for (int64_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

}  // extern "C"
