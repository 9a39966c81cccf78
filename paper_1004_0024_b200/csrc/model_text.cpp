#include "model_text.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <tuple>
#include <vector>

namespace isingb200 {

namespace {

// ------------------------------------------------------------------------------------------
// Reading is a small state machine over the lines of the document: a table maps the keyword of
// a line to a handler, every handler validates its own arity and ranges, and all complaints go
// through Reader::reject, which stamps the 1-based line number (ref: model_io.cpp:28-30 for the
// message format; the wording of each complaint is the reference's, so that callers matching on
// it keep working).
// ------------------------------------------------------------------------------------------
struct HalfEdge {
    uint32_t spin;
    uint32_t target;
    float coupling;
    uint8_t rank;  // 0 space, 1 tau towards the next layer, 2 tau towards the previous layer
};

class Reader {
  public:
    explicit Reader(std::string_view document) : rest_(document) {}

    HostModel run() {
        while (next_line()) {
            if (words_.empty()) continue;
            if (!header_ok_) {
                if (!(words_.size() == 2 && words_[0] == "ising-model" && words_[1] == "v1")) {
                    reject("expected header 'ising-model v1'");
                }
                header_ok_ = true;
                continue;
            }
            dispatch();
        }
        if (!header_ok_) throw ParseError("line 1: empty document, expected 'ising-model v1'");
        if (!spins_known_) throw ParseError("line " + std::to_string(line_) + ": missing spins line");
        return assemble();
    }

  private:
    using Handler = void (Reader::*)();

    void dispatch() {
        static constexpr std::array<std::pair<std::string_view, Handler>, 4> table{{
            {"spins", &Reader::take_spins},
            {"layers", &Reader::take_layers},
            {"h", &Reader::take_field},
            {"edge", &Reader::take_edge},
        }};
        const std::string_view key = words_[0];
        const auto hit = std::find_if(table.begin(), table.end(), [&](const auto& row) { return row.first == key; });
        if (key != "spins" && !spins_known_) reject("spins line must precede '" + std::string(key) + "'");
        if (hit == table.end()) reject("unknown line '" + std::string(key) + "'");
        (this->*hit->second)();
    }

    void take_spins() {
        if (spins_known_) reject("duplicate spins line");
        uint32_t count = 0;
        if (words_.size() != 2 || !number(1, count) || count == 0) reject("malformed spins line");
        n_ = count;
        spins_known_ = true;
        field_.assign(n_, 0.0f);
        field_line_.assign(n_, 0);
    }

    void take_layers() {
        if (layers_ != 0) reject("duplicate layers line");
        uint32_t count = 0, width = 0;
        if (words_.size() != 3 || !number(1, count) || !number(2, width)) reject("malformed layers line");
        if (count < 4 || uint64_t(count) * width != n_) reject("layers * per_layer must equal spins with layers >= 4");
        layers_ = count;
        width_ = width;
    }

    void take_field() {
        uint32_t spin = 0;
        float value = 0.0f;
        if (words_.size() != 3 || !number(1, spin) || !real(2, value)) reject("malformed h line");
        if (spin >= n_) reject("h index out of range");
        if (field_line_[spin] != 0) reject("duplicate h line for spin " + std::to_string(spin));
        field_line_[spin] = line_;
        field_[spin] = value;
    }

    void take_edge() {
        uint32_t a = 0, b = 0;
        float coupling = 0.0f;
        const bool shape = words_.size() == 5 && number(1, a) && number(2, b) && real(3, coupling) &&
                           (words_[4] == "space" || words_[4] == "tau");
        if (!shape) reject("malformed edge line");
        if (std::max(a, b) >= n_) reject("edge endpoint out of range");
        if (a >= b) reject("edge endpoints must satisfy i < j");
        const uint64_t key = uint64_t(a) * n_ + b;
        if (std::binary_search(seen_sorted_.begin(), seen_sorted_.end(), key) ||
            std::find(seen_recent_.begin(), seen_recent_.end(), key) != seen_recent_.end()) {
            reject("duplicate edge " + std::to_string(a) + "-" + std::to_string(b));
        }
        remember(key);
        const bool tau = words_[4] == "tau";
        if (tau && layers_ == 0) reject("tau edge in a model without layers");
        // a tau edge ranks by the direction it has seen from each endpoint
        halves_.push_back({a, b, coupling, uint8_t(tau ? direction(a, b) : 0)});
        halves_.push_back({b, a, coupling, uint8_t(tau ? direction(b, a) : 0)});
    }

    // 1 when `to` is `from`'s partner in the next layer (periodic), else 2
    uint8_t direction(uint32_t from, uint32_t to) const {
        const uint32_t up = ((from / width_ + 1) % layers_) * width_ + from % width_;
        return to == up ? 1 : 2;
    }

    // duplicate detection without a node-based set: a sorted run plus a short unsorted tail
    void remember(uint64_t key) {
        seen_recent_.push_back(key);
        if (seen_recent_.size() >= 64) {
            const size_t old = seen_sorted_.size();
            seen_sorted_.insert(seen_sorted_.end(), seen_recent_.begin(), seen_recent_.end());
            std::sort(seen_sorted_.begin() + long(old), seen_sorted_.end());
            std::inplace_merge(seen_sorted_.begin(), seen_sorted_.begin() + long(old), seen_sorted_.end());
            seen_recent_.clear();
        }
    }

    HostModel assemble() {
        // canonical adjacency = half-edges ordered by (spin, space before tau-next before tau-previous,
        // target); stable, so nothing depends on the order of the lines
        std::stable_sort(halves_.begin(), halves_.end(), [](const HalfEdge& x, const HalfEdge& y) {
            return std::tie(x.spin, x.rank, x.target) < std::tie(y.spin, y.rank, y.target);
        });
        HostModel m;
        m.n_spins = n_;
        m.layers = layers_;
        m.per_layer = layers_ != 0 ? width_ : 0;
        m.h = std::move(field_);
        m.offsets.assign(size_t(n_) + 1, 0);
        m.tau_counts.assign(n_, 0);
        m.targets.reserve(halves_.size());
        m.couplings.reserve(halves_.size());
        for (const HalfEdge& half : halves_) {
            ++m.offsets[half.spin + 1];
            m.tau_counts[half.spin] = uint8_t(m.tau_counts[half.spin] + (half.rank != 0 ? 1 : 0));
            m.targets.push_back(half.target);
            m.couplings.push_back(half.coupling);
        }
        for (uint32_t spin = 0; spin < n_; ++spin) {
            m.offsets[spin + 1] += m.offsets[spin];
            if (layers_ != 0 && m.tau_counts[spin] != 2) {
                throw Error("spin " + std::to_string(spin) + " has " + std::to_string(m.tau_counts[spin]) +
                            " tau edges, expected 2");
            }
        }
        try {
            finalize_model(m);
        } catch (const Error& problem) {
            throw Error(std::string("model failed validation after load: ") + problem.what());
        }
        return m;
    }

    // ---- line and word plumbing
    bool next_line() {
        if (rest_.empty()) return false;
        const size_t cut = rest_.find('\n');
        std::string_view line = rest_.substr(0, cut);
        rest_.remove_prefix(cut == std::string_view::npos ? rest_.size() : cut + 1);
        ++line_;
        words_.clear();
        const char* const blanks = " \t\r";
        for (size_t from = line.find_first_not_of(blanks); from != std::string_view::npos;) {
            const size_t to = line.find_first_of(blanks, from);
            words_.push_back(line.substr(from, to == std::string_view::npos ? to : to - from));
            from = to == std::string_view::npos ? to : line.find_first_not_of(blanks, to);
        }
        return true;
    }

    bool number(size_t index, uint32_t& out) const {
        const std::string_view w = words_[index];
        const auto parsed = std::from_chars(w.data(), w.data() + w.size(), out, 10);
        return !w.empty() && parsed.ec == std::errc() && parsed.ptr == w.data() + w.size();
    }

    // decimal or hexadecimal literal filling the whole word (strtof reads both, to nearest)
    bool real(size_t index, float& out) const {
        const std::string word(words_[index]);
        char* stop = nullptr;
        out = std::strtof(word.c_str(), &stop);
        return !word.empty() && stop == word.c_str() + word.size();
    }

    [[noreturn]] void reject(const std::string& why) const {
        throw ParseError("line " + std::to_string(line_) + ": " + why);
    }

    std::string_view rest_;
    std::vector<std::string_view> words_;
    size_t line_ = 0;
    bool header_ok_ = false, spins_known_ = false;
    uint32_t n_ = 0, layers_ = 0, width_ = 0;
    std::vector<float> field_;
    std::vector<size_t> field_line_;
    std::vector<HalfEdge> halves_;
    std::vector<uint64_t> seen_sorted_, seen_recent_;
};

// "%a" of the value widened to double: the literal the reference writes (ref: model_io.cpp:18-22)
void put_hex(std::string& doc, float value) {
    char text[40];
    const int length = std::snprintf(text, sizeof text, "%a", double(value));
    doc.append(text, size_t(length));
}

void put_line(std::string& doc, std::initializer_list<uint32_t> numbers, const char* keyword, float value,
              const char* suffix) {
    doc += keyword;
    for (uint32_t v : numbers) {
        doc += ' ';
        doc += std::to_string(v);
    }
    doc += ' ';
    put_hex(doc, value);
    doc += suffix;
}

}  // namespace

std::string model_to_text(const HostModel& m) {
    std::string doc;
    doc.reserve(64 + size_t(m.n_spins) * 24 + m.targets.size() * 20);
    doc += "ising-model v1\nspins ";
    doc += std::to_string(m.n_spins);
    doc += '\n';
    if (m.layers != 0) {
        doc += "layers " + std::to_string(m.layers) + ' ' + std::to_string(m.per_layer) + '\n';
    }
    // fields: every bit pattern other than +0.0 (a negative zero is written and so survives)
    for (uint32_t spin = 0; spin < m.n_spins; ++spin) {
        uint32_t pattern = 0;
        std::memcpy(&pattern, &m.h[spin], sizeof pattern);
        if (pattern != 0) put_line(doc, {spin}, "h", m.h[spin], "\n");
    }
    // each undirected edge once, from its lower endpoint, in adjacency order
    for (uint32_t spin = 0; spin < m.n_spins; ++spin) {
        const uint32_t stop = m.offsets[spin + 1];
        for (uint32_t slot = m.offsets[spin]; slot < stop; ++slot) {
            if (m.targets[slot] <= spin) continue;
            const bool tau = stop - slot <= m.tau_counts[spin];
            put_line(doc, {spin, m.targets[slot]}, "edge", m.couplings[slot], tau ? " tau\n" : " space\n");
        }
    }
    return doc;
}

HostModel model_from_text(std::string_view text) { return Reader(text).run(); }

void save_model_text(const HostModel& m, const std::string& path) {
    const std::string doc = model_to_text(m);
    std::ofstream file(path, std::ios::binary | std::ios::trunc);
    if (!file.is_open()) throw IoError("save_model: cannot open " + path);
    file.write(doc.data(), std::streamsize(doc.size()));
    file.close();
    if (file.fail()) throw IoError("save_model: write failed for " + path);
}

HostModel load_model_text(const std::string& path) {
    std::ifstream file(path, std::ios::binary);
    if (!file.is_open()) throw IoError("load_model: cannot open " + path);
    const std::string doc{std::istreambuf_iterator<char>(file), std::istreambuf_iterator<char>()};
    try {
        return model_from_text(doc);
    } catch (const ParseError& problem) {
        throw ParseError(path + ": " + problem.what());
    } catch (const Error& problem) {
        throw Error(path + ": " + problem.what());
    }
}

}  // namespace isingb200
