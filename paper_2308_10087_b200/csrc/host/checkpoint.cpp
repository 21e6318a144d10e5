// Checkpoint files (save_checkpoint / load_checkpoint, nn.cpp:82-124; format
// nn.hpp:497-531) and the resumable training state built on them. The header is
// written exactly as the reference's JSON library dumps it (compact, keys in
// sorted order), so files are byte-compatible in both directions.
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>

#include "gnnsim_b200.hpp"

namespace gnnsim {

namespace {

std::string json_escape(const std::string& s) {
    std::string o;
    for (char c : s) {
        if (c == '"' || c == '\\') {
            o += '\\';
            o += c;
        } else if (c == '\b' || c == '\f' || c == '\n' || c == '\r' || c == '\t') {
            // nlohmann::json dump: the short escapes for these five, \u00XX for the rest
            o += '\\';
            o += c == '\b' ? 'b' : c == '\f' ? 'f' : c == '\n' ? 'n' : c == '\r' ? 'r' : 't';
        } else if (static_cast<unsigned char>(c) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", unsigned(static_cast<unsigned char>(c)));
            o += buf;
        } else {
            o += c;
        }
    }
    return o;
}

// Minimal reader for the header: {"tensors":[{key:value,...},...]} with string
// and unsigned-integer values, any key order.
struct HeaderReader {
    const std::string& s;
    size_t i = 0;
    [[noreturn]] void fail() const { throw std::runtime_error("checkpoint: malformed header"); }
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    void expect(char c) {
        ws();
        if (i >= s.size() || s[i] != c) fail();
        ++i;
    }
    bool peek(char c) {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string str() {
        expect('"');
        std::string o;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                if (++i >= s.size()) fail();
                if (s[i] == 'u') {
                    if (i + 4 >= s.size()) fail();
                    uint32_t cp = uint32_t(std::stoul(s.substr(i + 1, 4), nullptr, 16));
                    i += 5;
                    // surrogate pair -> one code point; then UTF-8 (as nlohmann parses it)
                    if (cp >= 0xD800 && cp < 0xDC00 && i + 5 < s.size() && s[i] == '\\' && s[i + 1] == 'u') {
                        const uint32_t lo = uint32_t(std::stoul(s.substr(i + 2, 4), nullptr, 16));
                        if (lo >= 0xDC00 && lo < 0xE000) {
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                            i += 6;
                        }
                    }
                    if (cp < 0x80) {
                        o += char(cp);
                    } else if (cp < 0x800) {
                        o += char(0xC0 | (cp >> 6));
                        o += char(0x80 | (cp & 0x3F));
                    } else if (cp < 0x10000) {
                        o += char(0xE0 | (cp >> 12));
                        o += char(0x80 | ((cp >> 6) & 0x3F));
                        o += char(0x80 | (cp & 0x3F));
                    } else {
                        o += char(0xF0 | (cp >> 18));
                        o += char(0x80 | ((cp >> 12) & 0x3F));
                        o += char(0x80 | ((cp >> 6) & 0x3F));
                        o += char(0x80 | (cp & 0x3F));
                    }
                    continue;
                }
                const char e = s[i];
                o += e == 'b' ? '\b' : e == 'f' ? '\f' : e == 'n' ? '\n' : e == 'r' ? '\r' : e == 't' ? '\t' : e;
                ++i;
                continue;
            }
            o += s[i++];
        }
        expect('"');
        return o;
    }
    uint64_t num() {
        ws();
        size_t j = i;
        while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
        if (j == i) fail();
        const uint64_t v = std::stoull(s.substr(i, j - i));
        i = j;
        return v;
    }
};

}  // namespace

void save_checkpoint(const std::string& path, const std::vector<std::string>& names,
                     const std::vector<const float*>& data,
                     const std::vector<std::pair<uint64_t, uint64_t>>& shapes) {
    if (names.size() != data.size() || names.size() != shapes.size())
        throw std::invalid_argument("save_checkpoint: names/data/shapes differ in length");
    std::string h = "{\"tensors\":[";
    for (size_t t = 0; t < names.size(); ++t) {
        if (t) h += ',';
        h += "{\"cols\":" + std::to_string(shapes[t].second) + ",\"name\":\"" + json_escape(names[t]) +
             "\",\"rows\":" + std::to_string(shapes[t].first) + "}";
    }
    h += "]}";
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot write " + path);
    const uint64_t hl = h.size();
    f.write(reinterpret_cast<const char*>(&hl), 8);
    f.write(h.data(), std::streamsize(h.size()));
    for (size_t t = 0; t < data.size(); ++t)
        f.write(reinterpret_cast<const char*>(data[t]), std::streamsize(shapes[t].first * shapes[t].second * 4));
    if (!f) throw std::runtime_error("write failed: " + path);
}

std::vector<CheckpointTensor> load_checkpoint(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot read " + path);
    uint64_t hl = 0;
    f.read(reinterpret_cast<char*>(&hl), 8);
    if (!f || hl > (1ull << 30)) throw std::runtime_error("truncated checkpoint header: " + path);
    std::string h(hl, '\0');
    f.read(h.data(), std::streamsize(hl));
    if (!f) throw std::runtime_error("truncated checkpoint header: " + path);
    HeaderReader r{h};
    std::vector<CheckpointTensor> out;
    r.expect('{');
    if (r.str() != "tensors") r.fail();
    r.expect(':');
    r.expect('[');
    while (!r.peek(']')) {
        CheckpointTensor t;
        r.expect('{');
        while (!r.peek('}')) {
            const std::string key = r.str();
            r.expect(':');
            if (key == "name") t.name = r.str();
            else if (key == "rows") t.rows = r.num();
            else if (key == "cols") t.cols = r.num();
            else r.fail();
            if (r.peek(',')) r.expect(',');
        }
        r.expect('}');
        out.push_back(std::move(t));
        if (r.peek(',')) r.expect(',');
    }
    r.expect(']');
    r.expect('}');
    for (auto& t : out) {
        t.data.resize(t.rows * t.cols);
        f.read(reinterpret_cast<char*>(t.data.data()), std::streamsize(t.data.size() * 4));
        if (!f) throw std::runtime_error("truncated checkpoint data: " + path);
    }
    return out;
}

void save_train_state(const std::string& path, const TrainState& st) {
    if (st.adam_m.size() != st.params.size() || st.adam_v.size() != st.params.size())
        throw std::invalid_argument("save_train_state: optimizer state does not match the parameters");
    std::vector<std::string> names;
    std::vector<const float*> data;
    std::vector<std::pair<uint64_t, uint64_t>> shapes;
    const float head[2] = {float(st.epoch), float(st.optimizer_step)};
    if (st.epoch > (1u << 24) || st.optimizer_step > (1ull << 24))
        throw std::invalid_argument("save_train_state: epoch / step beyond exact f32 range");
    names.push_back("train.state");
    data.push_back(head);
    shapes.push_back({1, 2});
    auto add = [&](const std::string& n, const LayerParams<float>& p) {
        names.push_back(n + ".weight");
        data.push_back(p.weight.data());
        shapes.push_back({p.weight.rows(), p.weight.cols()});
        if (!p.bias.empty()) {
            names.push_back(n + ".bias");
            data.push_back(p.bias.data());
            shapes.push_back({1, p.bias.size()});
        }
    };
    for (size_t l = 0; l < st.params.size(); ++l) add("layer" + std::to_string(l), st.params[l]);
    for (size_t l = 0; l < st.params.size(); ++l) {
        const std::string n = "layer" + std::to_string(l);
        for (const char* which : {"adam_m", "adam_v"}) {
            const auto& p = std::string(which) == "adam_m" ? st.adam_m[l] : st.adam_v[l];
            names.push_back(n + ".weight." + which);
            data.push_back(p.weight.data());
            shapes.push_back({p.weight.rows(), p.weight.cols()});
            if (!p.bias.empty()) {
                names.push_back(n + ".bias." + which);
                data.push_back(p.bias.data());
                shapes.push_back({1, p.bias.size()});
            }
        }
    }
    for (const auto& h : st.history) {
        names.push_back("history.w" + std::to_string(h.worker) + ".k" + std::to_string(h.which) + ".l" +
                        std::to_string(h.layer));
        data.push_back(h.rows.data());
        shapes.push_back({h.width ? h.rows.size() / h.width : 0, h.width});
    }
    save_checkpoint(path, names, data, shapes);
}

TrainState load_train_state(const std::string& path, const std::vector<LayerSpec>& specs) {
    std::map<std::string, CheckpointTensor> by;
    for (auto& t : load_checkpoint(path)) by[t.name] = std::move(t);
    auto take = [&](const std::string& n, uint64_t rows, uint64_t cols) -> std::vector<float>& {
        auto it = by.find(n);
        if (it == by.end()) throw std::invalid_argument("train state " + path + ": missing tensor " + n);
        if (it->second.rows != rows || it->second.cols != cols)
            throw std::invalid_argument("train state " + path + ": tensor " + n + " has the wrong shape");
        return it->second.data;
    };
    TrainState st;
    const auto& head = take("train.state", 1, 2);
    st.epoch = uint32_t(head[0]);
    st.optimizer_step = uint64_t(head[1]);
    for (size_t l = 0; l < specs.size(); ++l) {
        const uint32_t k = specs[l].k_in(), o = specs[l].out_dim;
        const std::string n = "layer" + std::to_string(l);
        for (int which = 0; which < 3; ++which) {
            const std::string sfx = which == 0 ? "" : (which == 1 ? ".adam_m" : ".adam_v");
            LayerParams<float> p;
            p.weight = MatF(k, o);
            const auto& w = take(n + ".weight" + sfx, k, o);
            std::memcpy(p.weight.data(), w.data(), w.size() * 4);
            if (specs[l].has_bias()) p.bias = take(n + ".bias" + sfx, 1, o);
            (which == 0 ? st.params : (which == 1 ? st.adam_m : st.adam_v)).push_back(std::move(p));
        }
    }
    for (auto& [name, t] : by) {  // history.wW.kK.lL (sorted by name: a stable order)
        unsigned w = 0, k = 0, l = 0;
        if (name.rfind("history.", 0) != 0) continue;
        if (std::sscanf(name.c_str(), "history.w%u.k%u.l%u", &w, &k, &l) != 3)
            throw std::invalid_argument("train state " + path + ": bad history tensor name " + name);
        TrainState::HistoryRows h;
        h.worker = w;
        h.which = k;
        h.layer = l;
        h.width = uint32_t(t.cols);
        h.rows = std::move(t.data);
        st.history.push_back(std::move(h));
    }
    return st;
}

}  // namespace gnnsim
