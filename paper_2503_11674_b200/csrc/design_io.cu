// design_io.cu — the binary design file (SoA) behind tdpg_design_bin_*: host-side I/O only.  The reference
// stores designs as JSON (design_io.cpp:63-193), which does not scale to millions of cells; this format
// holds the same Netlist / DesignConstraints / positions fields as flat arrays, so a 1M-cell design loads
// with a handful of reads.  Layout: paper_2503_11674_b200/design.py (save_bin / load_bin), which writes and
// reads the same bytes.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace tdpg {
int api_fail(int kind, const std::string& msg);
}

using namespace tdpg;

namespace {

constexpr char kMagic[8] = {'T', 'D', 'P', 'G', 'D', 'S', 'N', '1'};
constexpr int kHeader = 128;

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : f(std::fopen(p, mode)), path(p)
    {
        if (!f) throw Error(TDPG_ERR_PARSE, std::string("parse error: cannot open ") + p);
    }
    ~File()
    {
        if (f) std::fclose(f);
    }
    void read(void* dst, size_t bytes, const char* what)
    {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes)
            throw Error(TDPG_ERR_PARSE, "parse error: " + path + ": truncated (" + what + ")");
        const size_t pad = (8 - bytes % 8) % 8;
        char z[8];
        if (pad && std::fread(z, 1, pad, f) != pad && !std::feof(f))
            throw Error(TDPG_ERR_PARSE, "parse error: " + path + ": truncated (" + what + ")");
    }
    void write(const void* src, size_t bytes)
    {
        static const char z[8] = {0};
        const size_t pad = (8 - bytes % 8) % 8;
        if ((bytes && std::fwrite(src, 1, bytes, f) != bytes) || (pad && std::fwrite(z, 1, pad, f) != pad))
            throw Error(TDPG_ERR_PARSE, "parse error: " + path + ": write failed");
    }
};

struct Header {
    uint32_t version, flags;
    int64_t c[6]; // cells, pins, nets, net pins, sources, endpoints
    double sc[8]; // clock, r_unit, c_unit, core[4], default cell delay
};

Header read_header(File& f)
{
    char raw[kHeader];
    if (std::fread(raw, 1, kHeader, f.f) != kHeader || std::memcmp(raw, kMagic, 8) != 0)
        throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": not a binary design file");
    Header h;
    std::memcpy(&h.version, raw + 8, 4), std::memcpy(&h.flags, raw + 12, 4);
    std::memcpy(h.c, raw + 16, 48), std::memcpy(h.sc, raw + 64, 64);
    if (h.version != 1)
        throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": unsupported binary design version " +
                                        std::to_string(h.version));
    for (int i = 0; i < 6; ++i)
        if (h.c[i] < 0 || h.c[i] > INT32_MAX) throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": bad sizes");
    return h;
}

} // namespace

#define API_BEGIN try {
#define API_END                                                                   \
    return TDPG_OK;                                                               \
    }                                                                             \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }

extern "C" {

int tdpg_design_bin_info(const char* path, int64_t counts[6], int32_t* has_pin_names)
{
    API_BEGIN
    File f(path, "rb");
    const Header h = read_header(f);
    for (int i = 0; i < 6; ++i) counts[i] = h.c[i];
    if (has_pin_names) *has_pin_names = static_cast<int32_t>(h.flags & 1u);
    API_END
}

int tdpg_design_bin_read(const char* path, tdpg_netlist* d, double* positions, uint8_t* pos_explicit,
                         char* pin_name_blob, int64_t blob_cap)
{
    API_BEGIN
    File f(path, "rb");
    const Header h = read_header(f);
    const int64_t C = h.c[0], P = h.c[1], N = h.c[2], E = h.c[3], S = h.c[4], EP = h.c[5];
    if (d->n_cells != C || d->n_pins != P || d->n_nets != N || d->n_sources != S || d->n_endpoints != EP)
        throw Error(TDPG_ERR_VALIDATION, "validation error: tdpg_design_bin_read: the netlist's sizes do not match "
                                         "the file (tdpg_design_bin_info)");
    auto w = [](const void* p) { return const_cast<void*>(p); };
    f.read(w(d->cell_w), 8 * C, "cell_w"), f.read(w(d->cell_h), 8 * C, "cell_h");
    f.read(w(d->cell_delay), 8 * C, "cell_delay"), f.read(positions, 16 * C, "positions");
    f.read(w(d->pin_term), 16 * P, "pin_term"), f.read(w(d->pin_off), 16 * P, "pin_off");
    f.read(w(d->pin_cap), 8 * P, "pin_cap"), f.read(w(d->pin_cell), 4 * P, "pin_cell");
    f.read(w(d->net_start), 4 * (N + 1), "net_start"), f.read(w(d->net_pins), 4 * E, "net_pins");
    f.read(w(d->sources), 4 * S, "sources"), f.read(w(d->endpoints), 4 * EP, "endpoints");
    f.read(w(d->cell_fixed), C, "cell_fixed"), f.read(pos_explicit, C, "pos_explicit");
    f.read(w(d->pin_dir), P, "pin_dir");
    if (d->net_start[N] != E) throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": net_start / net_pins mismatch");
    d->clock_period = h.sc[0], d->r_unit = h.sc[1], d->c_unit = h.sc[2];
    std::memcpy(d->core, h.sc + 3, 4 * sizeof(double));
    if ((h.flags & 1u) && pin_name_blob) {
        uint64_t nb = 0;
        if (std::fread(&nb, 8, 1, f.f) != 1) throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": truncated (names)");
        if (static_cast<int64_t>(nb) > blob_cap)
            throw Error(TDPG_ERR_VALIDATION, "validation error: pin name buffer too small");
        if (nb && std::fread(pin_name_blob, 1, nb, f.f) != nb)
            throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": truncated (names)");
    }
    API_END
}

int tdpg_design_bin_write(const char* path, const tdpg_netlist* d, const double* positions,
                          const uint8_t* pos_explicit, double default_cell_delay)
{
    API_BEGIN
    File f(path, "wb");
    const int64_t C = d->n_cells, P = d->n_pins, N = d->n_nets, E = d->net_start[d->n_nets], S = d->n_sources,
                  EP = d->n_endpoints;
    char raw[kHeader] = {0};
    std::memcpy(raw, kMagic, 8);
    const uint32_t version = 1, flags = d->pin_names ? 1u : 0u;
    std::memcpy(raw + 8, &version, 4), std::memcpy(raw + 12, &flags, 4);
    const int64_t c[6] = {C, P, N, E, S, EP};
    std::memcpy(raw + 16, c, 48);
    const double sc[8] = {d->clock_period, d->r_unit, d->c_unit, d->core[0], d->core[1], d->core[2], d->core[3],
                          default_cell_delay};
    std::memcpy(raw + 64, sc, 64);
    f.write(raw, kHeader);
    f.write(d->cell_w, 8 * C), f.write(d->cell_h, 8 * C), f.write(d->cell_delay, 8 * C), f.write(positions, 16 * C);
    f.write(d->pin_term, 16 * P), f.write(d->pin_off, 16 * P), f.write(d->pin_cap, 8 * P);
    f.write(d->pin_cell, 4 * P), f.write(d->net_start, 4 * (N + 1)), f.write(d->net_pins, 4 * E);
    f.write(d->sources, 4 * S), f.write(d->endpoints, 4 * EP);
    f.write(d->cell_fixed, C), f.write(pos_explicit, C), f.write(d->pin_dir, P);
    if (flags) {
        std::string blob;
        for (int64_t p = 0; p < P; ++p) {
            blob += d->pin_names[p] ? d->pin_names[p] : "";
            blob.push_back('\0');
        }
        const uint64_t nb = blob.size();
        if (std::fwrite(&nb, 8, 1, f.f) != 1 || std::fwrite(blob.data(), 1, nb, f.f) != nb)
            throw Error(TDPG_ERR_PARSE, "parse error: " + f.path + ": write failed");
    }
    API_END
}

} // extern "C"
