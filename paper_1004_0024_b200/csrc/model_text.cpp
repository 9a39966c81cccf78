#include "model_text.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <unordered_set>
#include <vector>

namespace isingb200 {

namespace {

// One whitespace-separated field of a line; the views point into the document.
std::vector<std::string_view> split_fields(std::string_view line) {
    std::vector<std::string_view> fields;
    size_t at = 0;
    while (at < line.size()) {
        while (at < line.size() && (line[at] == ' ' || line[at] == '\t')) ++at;
        size_t end = at;
        while (end < line.size() && line[end] != ' ' && line[end] != '\t') ++end;
        if (end > at) fields.push_back(line.substr(at, end - at));
        at = end;
    }
    return fields;
}

bool to_u32(std::string_view field, uint32_t& out) {
    if (field.empty()) return false;
    const char* last = field.data() + field.size();
    const auto res = std::from_chars(field.data(), last, out, 10);
    return res.ec == std::errc() && res.ptr == last;
}

// Decimal or hexadecimal float literal, whole field (strtof reads both, and rounds to nearest).
bool to_f32(std::string_view field, float& out) {
    if (field.empty()) return false;
    const std::string copy(field);
    char* end = nullptr;
    out = std::strtof(copy.c_str(), &end);
    return end == copy.c_str() + copy.size();
}

void append_hex(std::string& doc, float v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%a", double(v));  // same literal the reference writes (model_io.cpp:18-22)
    doc += buf;
}

struct Problem {
    size_t line;
    [[noreturn]] void operator()(const std::string& what) const {
        throw ParseError("line " + std::to_string(line) + ": " + what);
    }
};

struct PendingEdge {
    uint32_t a, b;
    float coupling;
    bool tau;
};

}  // namespace

std::string model_to_text(const HostModel& m) {
    std::string doc = "ising-model v1\nspins " + std::to_string(m.n_spins) + "\n";
    if (m.layers != 0) doc += "layers " + std::to_string(m.layers) + " " + std::to_string(m.per_layer) + "\n";
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        uint32_t bits;
        std::memcpy(&bits, &m.h[i], sizeof bits);
        if (bits == 0) continue;  // +0.0 only: -0.0 is written, so the round trip keeps every bit
        doc += "h " + std::to_string(i) + " ";
        append_hex(doc, m.h[i]);
        doc += "\n";
    }
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        const uint32_t end = m.offsets[i + 1], first_tau = end - m.tau_counts[i];
        for (uint32_t e = m.offsets[i]; e < end; ++e) {
            if (m.targets[e] <= i) continue;  // each undirected edge once, from its lower endpoint
            doc += "edge " + std::to_string(i) + " " + std::to_string(m.targets[e]) + " ";
            append_hex(doc, m.couplings[e]);
            doc += e >= first_tau ? " tau\n" : " space\n";
        }
    }
    return doc;
}

HostModel model_from_text(std::string_view text) {
    bool seen_header = false, seen_spins = false, seen_layers = false;
    uint32_t n = 0, layers = 0, per_layer = 0;
    std::vector<float> h;
    std::vector<char> h_given;
    std::vector<PendingEdge> edges;
    std::unordered_set<uint64_t> edge_keys;

    size_t line_no = 0, at = 0;
    while (at < text.size()) {
        size_t nl = text.find('\n', at);
        if (nl == std::string_view::npos) nl = text.size();
        std::string_view line = text.substr(at, nl - at);
        at = nl + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        const std::vector<std::string_view> f = split_fields(line);
        if (f.empty()) continue;
        const Problem fail{line_no};

        if (!seen_header) {
            if (f.size() != 2 || f[0] != "ising-model" || f[1] != "v1") fail("expected header 'ising-model v1'");
            seen_header = true;
        } else if (f[0] == "spins") {
            if (seen_spins) fail("duplicate spins line");
            if (f.size() != 2 || !to_u32(f[1], n) || n == 0) fail("malformed spins line");
            seen_spins = true;
            h.assign(n, 0.0f);
            h_given.assign(n, 0);
        } else if (!seen_spins) {
            fail("spins line must precede '" + std::string(f[0]) + "'");
        } else if (f[0] == "layers") {
            if (seen_layers) fail("duplicate layers line");
            if (f.size() != 3 || !to_u32(f[1], layers) || !to_u32(f[2], per_layer)) fail("malformed layers line");
            if (layers < 4 || uint64_t(layers) * per_layer != n) {
                fail("layers * per_layer must equal spins with layers >= 4");
            }
            seen_layers = true;
        } else if (f[0] == "h") {
            uint32_t i = 0;
            float v = 0.0f;
            if (f.size() != 3 || !to_u32(f[1], i) || !to_f32(f[2], v)) fail("malformed h line");
            if (i >= n) fail("h index out of range");
            if (h_given[i]) fail("duplicate h line for spin " + std::to_string(i));
            h_given[i] = 1;
            h[i] = v;
        } else if (f[0] == "edge") {
            PendingEdge e{};
            if (f.size() != 5 || !to_u32(f[1], e.a) || !to_u32(f[2], e.b) || !to_f32(f[3], e.coupling) ||
                (f[4] != "space" && f[4] != "tau")) {
                fail("malformed edge line");
            }
            if (e.a >= n || e.b >= n) fail("edge endpoint out of range");
            if (e.a >= e.b) fail("edge endpoints must satisfy i < j");
            if (!edge_keys.insert(uint64_t(e.a) << 32 | e.b).second) {
                fail("duplicate edge " + std::to_string(e.a) + "-" + std::to_string(e.b));
            }
            e.tau = f[4] == "tau";
            if (e.tau && !seen_layers) fail("tau edge in a model without layers");
            edges.push_back(e);
        } else {
            fail("unknown line '" + std::string(f[0]) + "'");
        }
    }
    if (!seen_header) throw ParseError("line 1: empty document, expected 'ising-model v1'");
    if (!seen_spins) throw ParseError("line " + std::to_string(line_no) + ": missing spins line");

    // ---- canonical CSR: per spin the space edges by target, then (layered) tau up, tau down
    struct Half {
        uint32_t target;
        float coupling;
    };
    std::vector<std::vector<Half>> space(n), tau(n);
    for (const PendingEdge& e : edges) {
        auto& side = e.tau ? tau : space;
        side[e.a].push_back({e.b, e.coupling});
        side[e.b].push_back({e.a, e.coupling});
    }
    HostModel m;
    m.n_spins = n;
    m.h = std::move(h);
    m.layers = seen_layers ? layers : 0;
    m.per_layer = seen_layers ? per_layer : 0;
    m.offsets.assign(1, 0);
    m.tau_counts.assign(n, 0);
    for (uint32_t i = 0; i < n; ++i) {
        std::sort(space[i].begin(), space[i].end(), [](const Half& x, const Half& y) { return x.target < y.target; });
        if (seen_layers) {
            if (tau[i].size() != 2) {
                throw Error("spin " + std::to_string(i) + " has " + std::to_string(tau[i].size()) +
                            " tau edges, expected 2");
            }
            const uint32_t up = ((i / per_layer + 1) % layers) * per_layer + i % per_layer;
            if (tau[i][0].target != up) std::swap(tau[i][0], tau[i][1]);
            m.tau_counts[i] = 2;
        }
        for (const auto* side : {&space[i], &tau[i]}) {
            for (const Half& half : *side) {
                m.targets.push_back(half.target);
                m.couplings.push_back(half.coupling);
            }
        }
        m.offsets.push_back(uint32_t(m.targets.size()));
    }
    try {
        finalize_model(m);
    } catch (const Error& e) {
        throw Error(std::string("model failed validation after load: ") + e.what());
    }
    return m;
}

void save_model_text(const HostModel& m, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("save_model: cannot open " + path);
    out << model_to_text(m);
    out.flush();
    if (!out) throw IoError("save_model: write failed for " + path);
}

HostModel load_model_text(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("load_model: cannot open " + path);
    const std::string doc((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    try {
        return model_from_text(doc);
    } catch (const ParseError& e) {
        throw ParseError(path + ": " + e.what());
    } catch (const Error& e) {
        throw Error(path + ": " + e.what());
    }
}

}  // namespace isingb200
