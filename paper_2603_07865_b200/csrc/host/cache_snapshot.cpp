// Cache Manager directory snapshot (CacheManager::save_snapshot / load_snapshot,
// cache.cpp:211-295) over the device arena — SURVEY §8f row 3.
//
//   <dir>/manifest.jsonl  one JSON object per entry (nlohmann::json::dump, keys sorted):
//                         admitted_h, attempts, duration_s, id, importance, last_update_h,
//                         prompt_embedding (base64 of little-endian f32, core.cpp:222-279),
//                         quality, recent_skips, reuse_count, segments [{length_s, level, start_s}]
//   <dir>/<id>.emb        SWEM (core.cpp:183-220): full embedding, the segment rows, the clip
//                         embedding
//   <dir>/<id>.clip       SWSC (cache.cpp:177-209): f64 duration, u32 latent_rate, u64 seed,
//                         f32 skip_fraction_used, u32 n, n x f32 latent
//
// Load mirrors the reference: the ledger is replaced, the index is rebuilt empty with the
// context's IVF configuration (IvfIndex::build({}, C, seed, nprobe) — the rebuild interval returns
// to IvfIndex's default 1024, as after the reference's load) and every entry's STORED segment
// rows are inserted in ascending id order (index_entry), straight into the device arena; the
// SimClip latent goes into the entry's latent slot when the context's slots are [1][T][1] (the
// reference's 1-D latent). Save reads the rows back from the arena.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "host_policy.hpp"

namespace sw {
void set_last_error(const std::string& m);
}

namespace {

// ---------------------------------------------------------------- minimal JSON (the manifest)
struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0.0;
    bool b = false;
    std::string str;  // also the raw number text (integers above 2^53 stay exact)
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;

    const JVal& at(const char* key) const {
        for (const auto& kv : obj)
            if (kv.first == key) return kv.second;
        throw std::runtime_error(std::string("manifest: missing key ") + key);
    }
    uint64_t as_u64() const {
        if (kind != Num) throw std::runtime_error("manifest: expected a number");
        return std::strtoull(str.c_str(), nullptr, 10);
    }
};

struct JParser {
    const char* p;
    const char* e;
    void ws() {
        while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    [[noreturn]] void bad() { throw std::runtime_error("manifest: malformed JSON"); }
    JVal parse() {
        ws();
        if (p >= e) bad();
        JVal v;
        if (*p == '{') {
            v.kind = JVal::Obj;
            ++p;
            ws();
            if (p < e && *p == '}') {
                ++p;
                return v;
            }
            for (;;) {
                ws();
                JVal k = parse();
                if (k.kind != JVal::Str) bad();
                ws();
                if (p >= e || *p != ':') bad();
                ++p;
                v.obj.emplace_back(k.str, parse());
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == '}') {
                    ++p;
                    return v;
                }
                bad();
            }
        }
        if (*p == '[') {
            v.kind = JVal::Arr;
            ++p;
            ws();
            if (p < e && *p == ']') {
                ++p;
                return v;
            }
            for (;;) {
                v.arr.push_back(parse());
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == ']') {
                    ++p;
                    return v;
                }
                bad();
            }
        }
        if (*p == '"') {
            v.kind = JVal::Str;
            ++p;
            while (p < e && *p != '"') {
                if (*p == '\\') {
                    ++p;
                    if (p >= e) bad();
                    const char c = *p;
                    v.str.push_back(c == 'n' ? '\n' : c == 't' ? '\t' : c == 'r' ? '\r' : c);
                } else {
                    v.str.push_back(*p);
                }
                ++p;
            }
            if (p >= e) bad();
            ++p;
            return v;
        }
        if (!std::strncmp(p, "true", 4) || !std::strncmp(p, "false", 5)) {
            v.kind = JVal::Bool;
            v.b = *p == 't';
            p += v.b ? 4 : 5;
            return v;
        }
        if (!std::strncmp(p, "null", 4)) {
            p += 4;
            return v;
        }
        const char* s = p;
        while (p < e && (std::strchr("+-.eE", *p) || (*p >= '0' && *p <= '9'))) ++p;
        if (p == s) bad();
        v.kind = JVal::Num;
        v.str.assign(s, p);
        v.num = std::strtod(v.str.c_str(), nullptr);
        return v;
    }
};

// shortest text that parses back to the same double; nlohmann's dump adds ".0" to integral
// values, so the manifest reads the same to both parsers
std::string jnum(double x) {
    char buf[40];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, x);
        if (std::strtod(buf, nullptr) == x) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

// ---------------------------------------------------------------- base64 (core.cpp:222-265)
const char kB64[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";

std::string b64_floats(const std::vector<float>& v) {
    const uint8_t* d = reinterpret_cast<const uint8_t*>(v.data());
    const size_t len = v.size() * 4;
    std::string out;
    for (size_t i = 0; i < len; i += 3) {
        uint32_t x = (uint32_t)d[i] << 16;
        if (i + 1 < len) x |= (uint32_t)d[i + 1] << 8;
        if (i + 2 < len) x |= d[i + 2];
        out.push_back(kB64[(x >> 18) & 63]);
        out.push_back(kB64[(x >> 12) & 63]);
        out.push_back(i + 1 < len ? kB64[(x >> 6) & 63] : '=');
        out.push_back(i + 2 < len ? kB64[x & 63] : '=');
    }
    return out;
}

std::vector<float> floats_b64(const std::string& t) {
    std::vector<uint8_t> out;
    uint32_t buf = 0;
    int bits = 0;
    for (char c : t) {
        if (c == '=' || c == '\n' || c == '\r') continue;
        int v = c >= 'A' && c <= 'Z'   ? c - 'A'
                : c >= 'a' && c <= 'z' ? c - 'a' + 26
                : c >= '0' && c <= '9' ? c - '0' + 52
                : c == '+'             ? 62
                : c == '/'             ? 63
                                       : -1;
        if (v < 0) throw std::runtime_error("invalid base64 character");
        buf = (buf << 6) | (uint32_t)v;
        bits += 6;
        if (bits >= 8) {
            bits -= 8;
            out.push_back((uint8_t)((buf >> bits) & 0xff));
        }
    }
    if (out.size() % 4) throw std::runtime_error("embedding blob not a multiple of 4 bytes");
    std::vector<float> f(out.size() / 4);
    std::memcpy(f.data(), out.data(), out.size());
    return f;
}

// ---------------------------------------------------------------- binary payloads
std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

void spit(const std::string& path, const std::string& bytes) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot write " + path);
    f.write(bytes.data(), (std::streamsize)bytes.size());
    if (!f) throw std::runtime_error("short write to " + path);
}

struct Rd {
    const uint8_t* p;
    const uint8_t* e;
    template <typename T>
    T get() {
        if ((size_t)(e - p) < sizeof(T)) throw std::runtime_error("snapshot payload truncated");
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
};

template <typename T>
void put(std::string& out, T v) {
    out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

std::vector<std::vector<float>> read_swem(const std::string& path) {
    const std::string b = slurp(path);
    Rd r{reinterpret_cast<const uint8_t*>(b.data()), reinterpret_cast<const uint8_t*>(b.data()) + b.size()};
    if (b.size() < 4 || std::memcmp(b.data(), "SWEM", 4))
        throw std::runtime_error("not an embedding file (bad magic): " + path);
    r.p += 4;
    const uint32_t count = r.get<uint32_t>(), dim = r.get<uint32_t>();
    std::vector<std::vector<float>> out(count, std::vector<float>(dim));
    for (auto& v : out)
        for (auto& x : v) x = r.get<float>();
    return out;
}

void write_swem(const std::string& path, const std::vector<const std::vector<float>*>& vecs) {
    std::string out("SWEM");
    const uint32_t dim = vecs.empty() ? 0 : (uint32_t)vecs[0]->size();
    put<uint32_t>(out, (uint32_t)vecs.size());
    put<uint32_t>(out, dim);
    for (const auto* v : vecs) {
        if (v->size() != dim) throw std::runtime_error("ragged embedding dimensions");
        for (float f : *v) put<float>(out, f);
    }
    spit(path, out);
}

std::string entry_path(const std::string& dir, uint64_t id, const char* ext) {
    return dir + "/" + std::to_string(id) + ext;
}

int fail(int code, const std::string& m) {
    sw::set_last_error(m);
    return code;
}

}  // namespace

extern "C" {

int swcm_save_snapshot(const swcm_cache* h, const char* dir) {
    if (!h || !dir) return fail(SW_EINVAL, "swcm_save_snapshot: null argument");
    try {
        const std::string d(dir);
        if (mkdir(dir, 0755) != 0 && errno != EEXIST)
            throw std::runtime_error("cannot create snapshot directory " + d);
        std::ostringstream man;
        for (const auto& kv : h->entries) {
            const swh::Entry& e = kv.second;
            const int n = (int)e.segs.size();
            std::vector<float> rows((size_t)std::max(n, 1) * h->dim);
            const int got = sw_arena_read_rows(h->ctx, e.id, rows.data(), n);
            if (got != n) throw std::runtime_error("arena rows of entry " + std::to_string(e.id) +
                                                   " do not match the ledger");
            std::vector<std::vector<float>> seg_rows((size_t)n);
            for (int i = 0; i < n; ++i)
                seg_rows[i].assign(rows.begin() + (size_t)i * h->dim,
                                   rows.begin() + (size_t)(i + 1) * h->dim);
            // keys in nlohmann's (std::map) order
            man << "{\"admitted_h\":" << jnum(e.admitted_h)
                << ",\"attempts\":" << e.refinement_attempts
                << ",\"duration_s\":" << jnum(e.duration_s) << ",\"id\":" << e.id
                << ",\"importance\":" << jnum(e.importance)
                << ",\"last_update_h\":" << jnum(e.last_update_h)
                << ",\"prompt_embedding\":\"" << b64_floats(e.prompt) << "\""
                << ",\"quality\":" << jnum(e.quality) << ",\"recent_skips\":[";
            bool first = true;
            for (double s : e.recent_skips) {
                man << (first ? "" : ",") << jnum(s);
                first = false;
            }
            man << "],\"reuse_count\":" << e.reuse_count << ",\"segments\":[";
            for (int i = 0; i < n; ++i)
                man << (i ? "," : "") << "{\"length_s\":" << jnum(e.segs[i].length)
                    << ",\"level\":" << e.segs[i].level << ",\"start_s\":" << jnum(e.segs[i].start)
                    << "}";
            man << "]}\n";
            // blobs: full embedding, the segment rows, the clip embedding
            std::vector<const std::vector<float>*> blobs;
            blobs.push_back(&e.clip_embedding);  // full_embedding == clip.embedding
            for (const auto& v : seg_rows) blobs.push_back(&v);
            blobs.push_back(&e.clip_embedding);
            write_swem(entry_path(d, e.id, ".emb"), blobs);
            std::string clip("SWSC");
            put<double>(clip, e.duration_s);
            put<uint32_t>(clip, (uint32_t)e.latent_rate);
            put<uint64_t>(clip, e.clip_seed);
            put<float>(clip, (float)e.clip_skip);
            put<uint32_t>(clip, (uint32_t)e.clip_latent.size());
            for (float f : e.clip_latent) put<float>(clip, f);
            spit(entry_path(d, e.id, ".clip"), clip);
        }
        spit(d + "/manifest.jsonl", man.str());
    } catch (const std::exception& ex) {
        return fail(SW_ERUNTIME, ex.what());
    }
    return SW_OK;
}

int swcm_load_snapshot(swcm_cache* h, const char* dir) {
    if (!h || !dir) return fail(SW_EINVAL, "swcm_load_snapshot: null argument");
    const std::string d(dir);
    std::vector<swh::Entry> loaded;
    std::vector<std::vector<std::vector<float>>> rows;
    try {  // parse everything before touching the arena
        std::ifstream man(d + "/manifest.jsonl");
        if (!man) throw std::runtime_error("cannot open cache manifest in " + d);
        std::string line;
        while (std::getline(man, line)) {
            if (line.empty()) continue;
            JParser jp{line.data(), line.data() + line.size()};
            const JVal j = jp.parse();
            swh::Entry e;
            e.id = j.at("id").as_u64();
            e.duration_s = j.at("duration_s").num;
            e.importance = j.at("importance").num;
            e.last_update_h = j.at("last_update_h").num;
            e.admitted_h = j.at("admitted_h").num;
            e.refinement_attempts = (int)j.at("attempts").num;
            e.quality = j.at("quality").num;
            e.reuse_count = (size_t)j.at("reuse_count").as_u64();
            for (const JVal& s : j.at("recent_skips").arr) e.recent_skips.push_back(s.num);
            e.prompt = floats_b64(j.at("prompt_embedding").str);
            const JVal& segs = j.at("segments");
            auto blobs = read_swem(entry_path(d, e.id, ".emb"));
            if (blobs.size() != segs.arr.size() + 2)
                throw std::runtime_error("embedding blob count mismatch for entry " +
                                         std::to_string(e.id));
            std::vector<std::vector<float>> er;
            for (size_t i = 0; i < segs.arr.size(); ++i) {
                e.segs.push_back(swh::Seg{(int)segs.arr[i].at("level").num,
                                          segs.arr[i].at("start_s").num,
                                          segs.arr[i].at("length_s").num});
                if ((int)blobs[1 + i].size() != h->dim)
                    throw std::runtime_error("segment row dimension differs from the cache's");
                er.push_back(std::move(blobs[1 + i]));
            }
            e.clip_embedding = blobs.back();
            const std::string cb = slurp(entry_path(d, e.id, ".clip"));
            if (cb.size() < 4 || std::memcmp(cb.data(), "SWSC", 4))
                throw std::runtime_error("not a clip payload (bad magic): " +
                                         entry_path(d, e.id, ".clip"));
            Rd r{reinterpret_cast<const uint8_t*>(cb.data()) + 4,
                 reinterpret_cast<const uint8_t*>(cb.data()) + cb.size()};
            r.get<double>();  // clip.duration_s (the manifest's duration_s is the entry's)
            e.latent_rate = (int)r.get<uint32_t>();
            e.clip_seed = r.get<uint64_t>();
            e.clip_skip = r.get<float>();
            const uint32_t n = r.get<uint32_t>();
            e.clip_latent.resize(n);
            for (auto& x : e.clip_latent) x = r.get<float>();
            loaded.push_back(std::move(e));
            rows.push_back(std::move(er));
        }
    } catch (const std::exception& ex) {
        return fail(SW_ERUNTIME, ex.what());
    }
    // entries_.clear(); index_ = IvfIndex::build({}, C, seed, nprobe)
    for (const auto& kv : h->entries) {
        const int rc = sw_arena_remove(h->ctx, kv.first);
        if (rc < 0) return rc;
    }
    h->entries.clear();
    int32_t ivf = 0, C = 1, nprobe = 8;
    uint64_t interval = 1024, seed = 0;
    int rc = sw_ivf_config(h->ctx, &ivf, &C, &nprobe, &interval, &seed);
    if (rc < 0) return rc;
    if (ivf) {
        rc = sw_ivf_configure(h->ctx, C, nprobe, 1024, seed);  // a fresh IvfIndex's interval
        if (rc < 0) return rc;
    }
    const bool lat1d = h->latent_1d();
    // std::map order: ascending id, as index_entry runs over entries_
    std::vector<size_t> order(loaded.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return loaded[a].id < loaded[b].id; });
    uint64_t max_id = 0;
    for (size_t oi : order) {
        swh::Entry& e = loaded[oi];
        std::vector<float> flat;
        std::vector<sw_segment> ss;
        for (size_t i = 0; i < e.segs.size(); ++i) {
            flat.insert(flat.end(), rows[oi][i].begin(), rows[oi][i].end());
            ss.push_back(sw_segment{e.segs[i].level, 0, e.segs[i].start, e.segs[i].length});
        }
        const bool with_lat = lat1d && !e.clip_latent.empty();
        rc = sw_arena_insert(h->ctx, e.id, (int32_t)e.segs.size(), flat.data(), ss.data(),
                             with_lat ? e.clip_latent.data() : nullptr,
                             with_lat ? (int32_t)e.clip_latent.size() : 0);
        if (rc < 0) return rc;
        max_id = std::max(max_id, e.id);
        const uint64_t id = e.id;
        h->entries[id] = std::move(e);
    }
    h->next_id = max_id + 1;
    h->last_evicted.clear();
    return SW_OK;
}

}  // extern "C"
