// Snapshot formats loaded straight into (and saved from) the device arena — SURVEY §8f row 3.
//
//   SWIX  IvfIndex::save / load (index.cpp:345-408): "SWIX", u32 C, u32 nprobe, u32 D,
//         C x D f32 centroids, then per list: u64 count, count x {u64 id, u8 level,
//         f32 start_s, f32 length_s, D x f32 embedding}. Little endian (binio, core.cpp:287-330).
//   SWEM  save_embeddings / load_embeddings (core.cpp:183-220): "SWEM", u32 count, u32 dim,
//         count x dim f32.
//   SWMB  BanditModel::save / load (gater.cpp:277-306): "SWMB", u32 feature_dim, u32 arms (14),
//         arms x fd f32 theta, arms x fd f32 psi — read into / written from the context's
//         device-resident Skip Gater parameters.
//
// A warm restart of a large cache is then one file read + one bulk arena insert, without the
// host-side re-insert (and re-clustering) the reference's load path implies.
#include <algorithm>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "../sw_internal.cuh"

namespace sw {

namespace {

struct Reader {  // binio::Reader (core.hpp:149-158): bounds-checked little-endian reads
    const uint8_t* p;
    const uint8_t* end;
    void need(size_t n) const {
        if ((size_t)(end - p) < n) throw Error(SW_ERUNTIME, "snapshot truncated");
    }
    template <typename T>
    T get() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
};

std::string read_file(const char* path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw Error(SW_ERUNTIME, std::string("cannot open ") + path);
    return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

template <typename T>
void put(std::string& out, T v) {
    out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

}  // namespace

// ---------------------------------------------------------------- SWIX
// Loads an index snapshot into an EMPTY context: its entries (rows grouped by entry id, in
// (level, start) order), the centroids and every row's stored list. The context switches to
// IVF mode with the snapshot's C and nprobe (IvfIndex::load leaves seed 0 and rebuild count 0).
void swix_load(Ctx& c, const char* path, void (*insert)(Ctx&, int64_t, const uint64_t*,
                                                        const int64_t*, const float*,
                                                        const sw_segment*)) {
    SW_REQUIRE(c.slot_of.empty(), "load a snapshot into an empty arena");
    const std::string bytes = read_file(path);
    Reader r{reinterpret_cast<const uint8_t*>(bytes.data()),
             reinterpret_cast<const uint8_t*>(bytes.data()) + bytes.size()};
    r.need(4);
    if (std::memcmp(r.p, "SWIX", 4) != 0)
        throw Error(SW_ERUNTIME, std::string("not an index snapshot (bad magic): ") + path);
    r.p += 4;
    const uint32_t C = r.get<uint32_t>();
    const uint32_t nprobe = r.get<uint32_t>();
    const uint32_t dim = r.get<uint32_t>();
    SW_REQUIRE(C <= (uint32_t)kMaxCentroids, "snapshot has more than 256 lists");
    SW_REQUIRE(C == 0 || (int)dim == c.D, "snapshot dimension differs from the context's");
    std::vector<float> cent((size_t)C * dim);
    for (auto& f : cent) f = r.get<float>();
    struct Row {
        int level;
        double start, length;
        int list;
        const uint8_t* emb;
    };
    std::map<uint64_t, std::vector<Row>> ents;
    int64_t total = 0;
    for (uint32_t j = 0; j < C; ++j) {
        const uint64_t cnt = r.get<uint64_t>();
        for (uint64_t i = 0; i < cnt; ++i) {
            const uint64_t id = r.get<uint64_t>();
            Row row;
            row.level = r.get<uint8_t>();
            row.start = r.get<float>();
            row.length = r.get<float>();
            row.list = (int)j;
            r.need((size_t)dim * 4);
            row.emb = r.p;
            r.p += (size_t)dim * 4;
            ents[id].push_back(row);
            ++total;
        }
    }
    std::vector<uint64_t> ids;
    std::vector<int64_t> off{0};
    std::vector<float> rows;
    std::vector<sw_segment> segs;
    std::vector<int16_t> lists;
    rows.reserve((size_t)total * dim);
    for (auto& [id, rs] : ents) {
        std::stable_sort(rs.begin(), rs.end(), [](const Row& a, const Row& b) {
            return a.level != b.level ? a.level < b.level : a.start < b.start;
        });
        SW_REQUIRE((int)rs.size() <= c.Rp, "snapshot entry has more rows than rows_per_entry");
        ids.push_back(id);
        for (const Row& x : rs) {
            const size_t o = rows.size();
            rows.resize(o + dim);
            std::memcpy(rows.data() + o, x.emb, (size_t)dim * 4);
            sw_segment s{};
            s.level = x.level;
            s.start_s = x.start;
            s.length_s = x.length;
            segs.push_back(s);
            lists.push_back((int16_t)x.list);
        }
        off.push_back((int64_t)segs.size());
    }
    // bulk insert (no mutation counting), then the index state of IvfIndex::load
    c.ivf = false;
    if (!ids.empty())
        insert(c, (int64_t)ids.size(), ids.data(), off.data(), rows.data(), segs.data());
    c.ivf = true;
    c.grp_dirty = true;
    c.ivf_target = std::max<int>(1, (int)C);
    c.ivf_nprobe = (int)nprobe;
    c.ivf_seed = 0;
    c.ivf_mutations = 0;
    c.ivf_rebuilds = 0;
    c.ivf_C = (int)C;
    c.h_cent = cent;
    if (C > 0) {
        std::vector<float> pad((size_t)C * c.Df, 0.0f);
        for (uint32_t j = 0; j < C; ++j)
            std::memcpy(pad.data() + (size_t)j * c.Df, cent.data() + (size_t)j * dim, 4 * dim);
        mcopy(c, c.cent, pad.data(), 4 * pad.size(), cudaMemcpyHostToDevice);
    }
    // stored list of every row (the snapshot's lists, not recomputed); pad rows in no list
    {
        std::vector<int64_t> sl;
        std::vector<int32_t> nrr;
        for (uint64_t id : ids) {
            sl.push_back(c.slot_of.at(id));
            nrr.push_back(c.h_nrows[(size_t)sl.back()]);
        }
        ivf_mark_tails(c, sl, nrr);
    }
    size_t k = 0;
    for (uint64_t id : ids) {
        const int64_t slot = c.slot_of.at(id);
        const int nr = c.h_nrows[(size_t)slot];
        c.ivf_rows[(size_t)slot] = nr;
        mcopy(c, c.row_list + slot * c.Rp, lists.data() + k, sizeof(int16_t) * nr,
                           cudaMemcpyHostToDevice);
        k += (size_t)nr;
    }
}

// Saves the index in SWIX form. Rows inside a list are written in rebuild order (id, level,
// start), which is the reference's own list order after a rebuild.
void swix_save(Ctx& c, const char* path) {
    const int D = c.D;
    const int64_t nrow = c.high_water * c.Rp;
    std::vector<float> rows((size_t)nrow * c.Df);
    std::vector<sw_segment> segs((size_t)nrow);
    std::vector<int16_t> lists((size_t)nrow);
    if (nrow > 0) {
        mcopy(c, rows.data(), c.rows, 4 * rows.size(), cudaMemcpyDeviceToHost);
        mcopy(c, segs.data(), c.segs, sizeof(sw_segment) * nrow, cudaMemcpyDeviceToHost);
        mcopy(c, lists.data(), c.row_list, 2 * nrow, cudaMemcpyDeviceToHost);
    }
    const int C = c.ivf ? c.ivf_C : 1;
    std::vector<std::vector<std::pair<uint64_t, int64_t>>> per(C);
    for (auto& [id, slot] : c.slot_of) {
        const int nr = c.ivf ? c.ivf_rows[(size_t)slot] : c.h_nrows[(size_t)slot];
        for (int rr = 0; rr < nr; ++rr) {
            const int64_t row = slot * c.Rp + rr;
            const int l = c.ivf ? lists[(size_t)row] : 0;
            if (l >= 0 && l < C) per[(size_t)l].emplace_back(id, row);
        }
    }
    std::string out;
    out.append("SWIX", 4);
    put<uint32_t>(out, (uint32_t)C);
    put<uint32_t>(out, (uint32_t)(c.ivf ? c.ivf_nprobe : 1));
    put<uint32_t>(out, (uint32_t)(C > 0 ? D : 0));
    if (c.ivf) {
        for (float f : c.h_cent) put<float>(out, f);
    } else {  // exhaustive mode: one list; its centroid is the first stored row (index.cpp:228)
        std::vector<float> first((size_t)D, 0.0f);
        if (!per[0].empty()) {
            auto m = *std::min_element(per[0].begin(), per[0].end());
            std::memcpy(first.data(), rows.data() + m.second * c.Df, 4 * (size_t)D);
        }
        for (float f : first) put<float>(out, f);
    }
    for (auto& lst : per) {
        std::sort(lst.begin(), lst.end(), [&](const auto& a, const auto& b) {
            if (a.first != b.first) return a.first < b.first;
            const sw_segment &sa = segs[(size_t)a.second], &sb = segs[(size_t)b.second];
            if (sa.level != sb.level) return sa.level < sb.level;
            return sa.start_s < sb.start_s;
        });
        put<uint64_t>(out, (uint64_t)lst.size());
        for (auto& [id, row] : lst) {
            const sw_segment& s = segs[(size_t)row];
            put<uint64_t>(out, id);
            put<uint8_t>(out, (uint8_t)s.level);
            put<float>(out, (float)s.start_s);
            put<float>(out, (float)s.length_s);
            out.append(reinterpret_cast<const char*>(rows.data() + row * c.Df), 4 * (size_t)D);
        }
    }
    std::ofstream f(path, std::ios::binary);
    if (!f) throw Error(SW_ERUNTIME, std::string("cannot write ") + path);
    f.write(out.data(), (std::streamsize)out.size());
}

// SWEM (core.cpp:183-220)
int64_t swem_read(const char* path, float* out, int64_t cap_floats, int32_t* count, int32_t* dim) {
    const std::string bytes = read_file(path);
    Reader r{reinterpret_cast<const uint8_t*>(bytes.data()),
             reinterpret_cast<const uint8_t*>(bytes.data()) + bytes.size()};
    r.need(4);
    if (std::memcmp(r.p, "SWEM", 4) != 0)
        throw Error(SW_ERUNTIME, std::string("not an embedding file (bad magic): ") + path);
    r.p += 4;
    const uint32_t n = r.get<uint32_t>(), d = r.get<uint32_t>();
    r.need((size_t)n * d * 4);
    if (count) *count = (int32_t)n;
    if (dim) *dim = (int32_t)d;
    const int64_t nf = (int64_t)n * d;
    if (out) std::memcpy(out, r.p, 4 * (size_t)std::min(nf, cap_floats));
    return nf;
}

// ---------------------------------------------------------------- SWMB
void swmb_read(const char* path, std::vector<float>& theta, std::vector<float>& psi, int& fd) {
    const std::string bytes = read_file(path);
    Reader r{reinterpret_cast<const uint8_t*>(bytes.data()),
             reinterpret_cast<const uint8_t*>(bytes.data()) + bytes.size()};
    r.need(4);
    if (std::memcmp(r.p, "SWMB", 4) != 0)
        throw Error(SW_ERUNTIME, std::string("not a bandit model snapshot (bad magic): ") + path);
    r.p += 4;
    fd = (int)r.get<uint32_t>();
    const uint32_t arms = r.get<uint32_t>();
    if (arms != (uint32_t)kNumArms)  // gater.cpp:295-298
        throw Error(SW_ERUNTIME, "model snapshot arm count " + std::to_string(arms) +
                                     " does not match build (14)");
    theta.resize((size_t)kNumArms * fd);
    psi.resize((size_t)kNumArms * fd);
    for (auto& v : theta) v = r.get<float>();
    for (auto& v : psi) v = r.get<float>();
}

void swmb_write(const char* path, const float* theta, const float* psi, int fd) {
    std::string out("SWMB");
    put<uint32_t>(out, (uint32_t)fd);
    put<uint32_t>(out, (uint32_t)kNumArms);
    for (int i = 0; i < kNumArms * fd; ++i) put<float>(out, theta[i]);
    for (int i = 0; i < kNumArms * fd; ++i) put<float>(out, psi[i]);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw Error(SW_ERUNTIME, std::string("cannot write ") + path);
    f.write(out.data(), (std::streamsize)out.size());
    if (!f) throw Error(SW_ERUNTIME, std::string("short write to ") + path);
}

}  // namespace sw
