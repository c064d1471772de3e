// ttsvd/report.hpp — the run report of report.hpp:20-183: one row per (step,
// phase), CSV schema `variant,shape,rmax,eps,phase,step,seconds,flops,bytes,
// rank`, and the JSON array form (written and parsed here without a JSON
// library: the rows are flat objects of strings and numbers, doubles as %.17g
// so every round trip is bit-exact).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "errors.hpp"
#include "perf_model.hpp"
#include "shape.hpp"
#include "tt_svd.hpp"

namespace ttsvd {

struct ReportRow {
    std::string variant, shape;
    index_t rmax = 0;
    double eps = 0;
    std::string phase;
    index_t step = 0;
    double seconds = 0;
    std::uint64_t flops = 0, bytes = 0;
    index_t rank = 0;
};

inline const char* kReportHeader = "variant,shape,rmax,eps,phase,step,seconds,flops,bytes,rank";

namespace report_detail {
inline std::string g17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
inline std::string quoted(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}
// the field order shared by both formats
inline std::vector<std::pair<const char*, std::string>> fields(const ReportRow& r, bool json) {
    auto str = [&](const std::string& s) { return json ? quoted(s) : s; };
    return {{"variant", str(r.variant)},          {"shape", str(r.shape)},     {"rmax", std::to_string(r.rmax)},
            {"eps", g17(r.eps)},                  {"phase", str(r.phase)},     {"step", std::to_string(r.step)},
            {"seconds", g17(r.seconds)},          {"flops", std::to_string(r.flops)},
            {"bytes", std::to_string(r.bytes)},   {"rank", std::to_string(r.rank)}};
}
inline void assign(ReportRow& r, const std::string& key, const std::string& v) {
    if (key == "variant") r.variant = v;
    else if (key == "shape") r.shape = v;
    else if (key == "rmax") r.rmax = std::stoll(v);
    else if (key == "eps") r.eps = std::strtod(v.c_str(), nullptr);
    else if (key == "phase") r.phase = v;
    else if (key == "step") r.step = std::stoll(v);
    else if (key == "seconds") r.seconds = std::strtod(v.c_str(), nullptr);
    else if (key == "flops") r.flops = std::strtoull(v.c_str(), nullptr, 10);
    else if (key == "bytes") r.bytes = std::strtoull(v.c_str(), nullptr, 10);
    else if (key == "rank") r.rank = std::stoll(v);
    else throw IoError("report: unknown field '" + key + "'");
}
inline std::size_t write(std::ostream& out, const std::string& s, const char* who) {
    out << s;
    if (!out) throw IoError(std::string(who) + ": write failed");
    return s.size();
}
}  // namespace report_detail

// one row per step and phase, phases in the order tsqr, small-svd, tsmm,
// reorder; flops / bytes from the cost model of each phase
inline std::vector<ReportRow> rows_from_recorder(const RunRecorder& rec, const std::string& variant,
                                                 const std::string& shape, index_t rmax, double eps,
                                                 const Counters* = nullptr) {
    std::vector<ReportRow> rows;
    for (const StepRecord& s : rec.steps) {
        const double secs[4] = {s.t_tsqr, s.t_small_svd, s.t_tsmm, s.t_reorder};
        const char* names[4] = {"tsqr", "small-svd", "tsmm", "reorder"};
        for (int p = 0; p < 4; ++p) {
            ReportRow r;
            r.variant = variant;
            r.shape = shape;
            r.rmax = rmax;
            r.eps = eps;
            r.phase = names[p];
            r.step = s.step;
            r.seconds = secs[p];
            r.rank = s.rank;
            const auto rows_u = static_cast<std::uint64_t>(s.rows), cols_u = static_cast<std::uint64_t>(s.cols);
            if (p == 0) {
                r.flops = static_cast<std::uint64_t>(tsqr_cost(static_cast<double>(s.rows), static_cast<double>(s.cols),
                                                               static_cast<double>(BlockParams::for_cols(s.cols).n_b))
                                                         .n_flops);
                r.bytes = 8 * rows_u * cols_u;
            } else if (p == 2) {
                r.flops = 2 * rows_u * cols_u * static_cast<std::uint64_t>(s.rank);
                r.bytes = 8 * rows_u * (cols_u + static_cast<std::uint64_t>(s.rank));
            }
            rows.push_back(std::move(r));
        }
    }
    return rows;
}

inline std::size_t emit_csv(const std::vector<ReportRow>& rows, std::ostream& out) {
    std::string s = std::string(kReportHeader) + "\n";
    for (const ReportRow& r : rows) {
        std::string line;
        for (const auto& [k, v] : report_detail::fields(r, false)) line += (line.empty() ? "" : ",") + v;
        s += line + "\n";
    }
    return report_detail::write(out, s, "emit_csv");
}

inline std::size_t emit_json(const std::vector<ReportRow>& rows, std::ostream& out) {
    std::string s = "[";
    for (std::size_t i = 0; i < rows.size(); ++i) {
        s += i ? ",\n  {" : "\n  {";
        bool first = true;
        for (const auto& [k, v] : report_detail::fields(rows[i], true)) {
            s += std::string(first ? "" : ", ") + "\"" + k + "\": " + v;
            first = false;
        }
        s += "}";
    }
    s += rows.empty() ? "]\n" : "\n]\n";
    return report_detail::write(out, s, "emit_json");
}

inline std::size_t emit_report(const std::vector<ReportRow>& rows, const std::string& format, std::ostream& out) {
    if (format == "csv") return emit_csv(rows, out);
    if (format == "json") return emit_json(rows, out);
    throw IoError("emit_report: unknown format '" + format + "'");
}

inline std::vector<ReportRow> parse_csv(std::istream& in) {
    std::string line;
    if (!std::getline(in, line)) throw IoError("parse_csv: empty input");
    if (line != kReportHeader) throw IoError("parse_csv: unexpected header");
    static const char* keys[10] = {"variant", "shape", "rmax", "eps", "phase", "step", "seconds", "flops", "bytes", "rank"};
    std::vector<ReportRow> rows;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::vector<std::string> f(1);
        for (char c : line) {
            if (c == ',') f.emplace_back();
            else f.back() += c;
        }
        if (f.size() != 10) throw IoError("parse_csv: bad row");
        ReportRow r;
        for (int i = 0; i < 10; ++i) report_detail::assign(r, keys[i], f[static_cast<std::size_t>(i)]);
        rows.push_back(std::move(r));
    }
    return rows;
}

// the array of flat objects emit_json writes (strings and numbers only)
inline std::vector<ReportRow> parse_json(std::istream& in) {
    const std::string s((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::size_t i = 0;
    auto ws = [&] {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
    };
    auto expect = [&](char c) {
        ws();
        if (i >= s.size() || s[i] != c) throw IoError(std::string("parse_json: expected '") + c + "'");
        ++i;
    };
    auto string_at = [&] {
        expect('"');
        std::string o;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\' && i + 1 < s.size()) ++i;
            o += s[i++];
        }
        expect('"');
        return o;
    };
    std::vector<ReportRow> rows;
    expect('[');
    ws();
    if (i < s.size() && s[i] == ']') return rows;
    for (;;) {
        expect('{');
        ReportRow r;
        for (;;) {
            const std::string key = string_at();
            expect(':');
            ws();
            std::string val;
            if (i < s.size() && s[i] == '"') {
                val = string_at();
            } else {
                while (i < s.size() && s[i] != ',' && s[i] != '}' && s[i] != ' ' && s[i] != '\n') val += s[i++];
            }
            report_detail::assign(r, key, val);
            ws();
            if (i < s.size() && s[i] == ',') {
                ++i;
                continue;
            }
            expect('}');
            break;
        }
        rows.push_back(std::move(r));
        ws();
        if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
        }
        expect(']');
        break;
    }
    return rows;
}

}  // namespace ttsvd
