// Grid I/O and the bench-mode stage table of the drop-in (SURVEY.md section
// 8(f) item 4), behind the C ABI of include/fsx.h.
//
// Formats follow the reference (proj/include/fftstencil/grid_io.hpp,
// proj/src/grid_io.cpp):
//   raw  little-endian float64, row-major dims then field, plus a
//        "<path>.meta" sidecar "dims = d0 d1 ...\nfields = m\ndtype = float64\n
//        order = row-major\n" (grid_io.cpp:112-191); read back with the same
//        validation (unknown key / dtype / order, missing dims, byte count);
//   csv  one line per (cell, field) "i1,...,id,f,value" with shortest
//        round-trip decimals (grid_io.cpp:37-110).
// read_grid detects raw by the presence of the sidecar (grid_io.hpp:14).
// Problems raise the reference's IoError, here FSX_ERR_IO with the message.
//
// fsx_load_grid_device reads a raw grid STRAIGHT INTO DEVICE MEMORY: the
// file is read in 64 MiB chunks into two pinned staging buffers, and each
// chunk's H2D copy runs while the next chunk is read from disk (no full host
// copy of the grid).  fsx_format_stage_table prints run_bench's table
// (proj/src/runner.cpp:46-62).
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include <cuda_runtime.h>

#include "fsx.h"

extern "C" void fsx_internal_set_error(const char* msg);  // fsx_api.cpp (thread-local fsx_last_error)

namespace {

using i64 = long long;

struct IoErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ArgErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DevErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class F>
fsx_status guarded_io(F&& f) {
    try {
        f();
        fsx_internal_set_error("");
        return FSX_OK;
    } catch (const IoErr& e) {
        fsx_internal_set_error(e.what());
        return FSX_ERR_IO;
    } catch (const ArgErr& e) {
        fsx_internal_set_error(e.what());
        return FSX_ERR_SPEC;
    } catch (const DevErr& e) {
        fsx_internal_set_error(e.what());
        return FSX_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        fsx_internal_set_error("fsx: host allocation failed");
        return FSX_ERR_OOM;
    } catch (const std::exception& e) {
        fsx_internal_set_error(e.what());
        return FSX_ERR_IO;
    }
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw DevErr(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

std::string meta_path(const std::string& path) { return path + ".meta"; }

bool exists(const std::string& p) {
    struct stat sb;
    return ::stat(p.c_str(), &sb) == 0;
}

// GridShape invariants (proj/include/fftstencil/grid.hpp:21-45)
i64 shape_values(const fsx_shape* s) {
    if (!s) throw ArgErr("GridShape: null shape");
    if (s->rank < 1 || s->rank > FSX_MAX_RANK) throw ArgErr("GridShape: need at least one dimension");
    if (s->fields < 1) throw ArgErr("GridShape: fields must be >= 1");
    __int128 n = s->fields;
    for (int a = 0; a < s->rank; ++a) {
        if (s->dims[a] < 1) throw ArgErr("GridShape: every dimension must be >= 1");
        n *= s->dims[a];
        if (n > (__int128)INT64_MAX / 8) throw ArgErr("GridShape: total value count overflows");
    }
    return (i64)n;
}

std::string format_double(double v) {
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);  // shortest round-trip
    return std::string(buf, res.ptr);
}

double parse_double(std::string_view text, const std::string& where) {
    double v = 0;
    auto res = std::from_chars(text.data(), text.data() + text.size(), v);
    if (res.ec != std::errc() || res.ptr != text.data() + text.size())
        throw IoErr(where + ": bad number '" + std::string(text) + "'");
    return v;
}

i64 parse_index(std::string_view text, const std::string& where) {
    i64 v = 0;
    auto res = std::from_chars(text.data(), text.data() + text.size(), v);
    if (res.ec != std::errc() || res.ptr != text.data() + text.size())
        throw IoErr(where + ": bad integer '" + std::string(text) + "'");
    return v;
}

struct File {
    FILE* f = nullptr;
    File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// ------------------------------------------------------------------ raw
void write_raw(const fsx_shape* s, const double* data, const std::string& path) {
    const i64 n = shape_values(s);
    static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "raw format is little-endian");
    {
        File out(path, "wb");
        if (!out.f) throw IoErr("cannot open '" + path + "' for writing");
        if (n && std::fwrite(data, sizeof(double), (size_t)n, out.f) != (size_t)n)
            throw IoErr("write failed on '" + path + "'");
    }
    File meta(meta_path(path), "w");
    if (!meta.f) throw IoErr("cannot open '" + meta_path(path) + "' for writing");
    std::string m = "dims =";
    for (int a = 0; a < s->rank; ++a) m += " " + std::to_string(s->dims[a]);
    m += "\nfields = " + std::to_string(s->fields) + "\ndtype = float64\norder = row-major\n";
    if (std::fwrite(m.data(), 1, m.size(), meta.f) != m.size()) throw IoErr("write failed on '" + meta_path(path) + "'");
}

// Parses and validates "<path>.meta" and the data file's byte count
// (proj/src/grid_io.cpp:133-180).
fsx_shape read_raw_shape(const std::string& path) {
    File meta(meta_path(path), "r");
    if (!meta.f) throw IoErr("cannot open '" + meta_path(path) + "'");
    std::vector<i64> dims;
    int fields = -1;
    std::string line;
    size_t lineno = 0;
    char buf[4096];
    std::string text;
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, meta.f)) > 0) text.append(buf, got);
    std::stringstream all(text);
    while (std::getline(all, line)) {
        ++lineno;
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw IoErr(meta_path(path) + ":" + std::to_string(lineno) + ": expected 'key = value'");
        std::stringstream key_ss(line.substr(0, eq)), val_ss(line.substr(eq + 1));
        std::string key;
        key_ss >> key;
        if (key == "dims") {
            i64 d;
            while (val_ss >> d) dims.push_back(d);
        } else if (key == "fields") {
            val_ss >> fields;
        } else if (key == "dtype") {
            std::string v;
            val_ss >> v;
            if (v != "float64") throw IoErr(meta_path(path) + ": unsupported dtype '" + v + "'");
        } else if (key == "order") {
            std::string v;
            val_ss >> v;
            if (v != "row-major") throw IoErr(meta_path(path) + ": unsupported order '" + v + "'");
        } else {
            throw IoErr(meta_path(path) + ":" + std::to_string(lineno) + ": unknown key '" + key + "'");
        }
    }
    if (dims.empty() || fields < 1) throw IoErr(meta_path(path) + ": missing dims or fields");
    if ((int)dims.size() > FSX_MAX_RANK) throw IoErr(meta_path(path) + ": more than 8 dims");
    fsx_shape s{};
    s.rank = (int)dims.size();
    s.fields = fields;
    for (int a = 0; a < s.rank; ++a) s.dims[a] = dims[a];
    i64 n;
    try {
        n = shape_values(&s);
    } catch (const ArgErr& e) {
        throw IoErr(meta_path(path) + ": " + e.what());
    }
    const unsigned long long expected = (unsigned long long)n * sizeof(double);
    struct stat sb;
    if (::stat(path.c_str(), &sb) != 0) throw IoErr("cannot stat '" + path + "'");
    if ((unsigned long long)sb.st_size != expected)
        throw IoErr(path + ": expected " + std::to_string(expected) + " bytes, got " + std::to_string((long long)sb.st_size));
    return s;
}

void same_shape(const fsx_shape& file, const fsx_shape* want, const std::string& path) {
    if (!want) return;
    bool ok = file.rank == want->rank && file.fields == want->fields;
    for (int a = 0; ok && a < file.rank; ++a) ok = file.dims[a] == want->dims[a];
    if (!ok) throw IoErr(path + ": grid shape differs from the caller's shape");
}

void read_raw(const std::string& path, const fsx_shape* want, double* out) {
    const fsx_shape s = read_raw_shape(path);
    same_shape(s, want, path);
    const i64 n = shape_values(&s);
    File in(path, "rb");
    if (!in.f) throw IoErr("cannot open '" + path + "'");
    if (n && std::fread(out, sizeof(double), (size_t)n, in.f) != (size_t)n) throw IoErr(path + ": short read");
}

// ------------------------------------------------------------------ csv
bool next_index(std::vector<i64>& idx, const fsx_shape* s) {
    for (int a = s->rank - 1; a >= 0; --a) {
        if (++idx[a] < s->dims[a]) return true;
        idx[a] = 0;
    }
    return false;
}

void write_csv(const fsx_shape* s, const double* data, const std::string& path) {
    shape_values(s);
    File out(path, "w");
    if (!out.f) throw IoErr("cannot open '" + path + "' for writing");
    const int m = s->fields;
    std::vector<i64> idx(s->rank, 0);
    i64 cell = 0;
    std::string line;
    do {
        for (int f = 0; f < m; ++f) {
            line.clear();
            for (i64 i : idx) line += std::to_string(i) + ',';
            line += std::to_string(f) + ',' + format_double(data[cell * m + f]) + '\n';
            if (std::fwrite(line.data(), 1, line.size(), out.f) != line.size()) throw IoErr("write failed on '" + path + "'");
        }
        ++cell;
    } while (next_index(idx, s));
}

struct Csv {
    std::vector<std::vector<std::string>> rows;
    fsx_shape shape{};
};

Csv scan_csv(const std::string& path) {
    File in(path, "r");
    if (!in.f) throw IoErr("cannot open '" + path + "'");
    std::string text;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, in.f)) > 0) text.append(buf, got);
    Csv c;
    std::stringstream ss(text);
    std::string line;
    size_t lineno = 0, columns = 0;
    while (std::getline(ss, line)) {
        ++lineno;
        if (line.empty()) continue;
        std::vector<std::string> parts;
        std::stringstream ls(line);
        std::string part;
        while (std::getline(ls, part, ',')) parts.push_back(part);
        if (parts.size() < 3) throw IoErr(path + ":" + std::to_string(lineno) + ": expected 'i1,...,id,f,value'");
        if (columns == 0) columns = parts.size();
        if (parts.size() != columns) throw IoErr(path + ":" + std::to_string(lineno) + ": inconsistent column count");
        c.rows.push_back(std::move(parts));
    }
    if (c.rows.empty()) throw IoErr(path + ": empty grid file");
    const int rank = (int)columns - 2;
    if (rank > FSX_MAX_RANK) throw IoErr(path + ": more than 8 dims");
    std::vector<i64> dims(rank, 0);
    i64 max_field = 0;
    for (size_t r = 0; r < c.rows.size(); ++r) {
        const std::string where = path + ":" + std::to_string(r + 1);
        for (int a = 0; a < rank; ++a) dims[a] = std::max(dims[a], parse_index(c.rows[r][a], where) + 1);
        max_field = std::max(max_field, parse_index(c.rows[r][rank], where));
    }
    c.shape.rank = rank;
    c.shape.fields = (int)max_field + 1;
    for (int a = 0; a < rank; ++a) c.shape.dims[a] = dims[a];
    i64 n;
    try {
        n = shape_values(&c.shape);
    } catch (const ArgErr& e) {
        throw IoErr(path + ": " + e.what());
    }
    if (n != (i64)c.rows.size())
        throw IoErr(path + ": got " + std::to_string(c.rows.size()) + " lines for a grid of " + std::to_string(n) + " values");
    return c;
}

void read_csv(const Csv& c, const std::string& path, double* out) {
    const fsx_shape& s = c.shape;
    const i64 n = shape_values(&s);
    std::vector<bool> seen((size_t)n, false);
    for (size_t r = 0; r < c.rows.size(); ++r) {
        const std::string where = path + ":" + std::to_string(r + 1);
        i64 flat = 0;
        for (int a = 0; a < s.rank; ++a) {
            const i64 i = parse_index(c.rows[r][a], where);
            if (i < 0 || i >= s.dims[a]) throw IoErr(where + ": index out of range");
            flat = flat * s.dims[a] + i;
        }
        const i64 f = parse_index(c.rows[r][s.rank], where);
        if (f < 0 || f >= s.fields) throw IoErr(where + ": field out of range");
        const i64 pos = flat * s.fields + f;
        if (seen[(size_t)pos]) throw IoErr(where + ": duplicate cell");
        seen[(size_t)pos] = true;
        out[pos] = parse_double(c.rows[r][s.rank + 1], where);
        if (!std::isfinite(out[pos])) throw IoErr(where + ": non-finite value");
    }
}

// ------------------------------------------------------------------ raw straight to the device
void load_device(const std::string& path, const fsx_shape* want, double* d_out, const fsx_options* opt) {
    const fsx_shape s = read_raw_shape(path);
    same_shape(s, want, path);
    if (!d_out) throw ArgErr("fsx_load_grid_device: null device pointer");
    const i64 n = shape_values(&s);
    const size_t bytes = (size_t)n * sizeof(double);
    ck(cudaSetDevice(opt ? opt->device : 0), "cudaSetDevice");
    cudaStream_t st = (opt && opt->stream) ? reinterpret_cast<cudaStream_t>(opt->stream) : nullptr;
    bool own = false;
    if (!st) {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
        own = true;
    }
    constexpr size_t kChunk = size_t(64) << 20;
    const size_t chunk = bytes < kChunk ? (bytes ? bytes : 16) : kChunk;
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int fd = -1;
    auto cleanup = [&] {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) {
                cudaEventSynchronize(done[i]);
                cudaEventDestroy(done[i]);
            }
            if (stage[i]) cudaFreeHost(stage[i]);
        }
        if (own) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        if (fd >= 0) ::close(fd);
    };
    try {
        for (int i = 0; i < 2; ++i) {
            ck(cudaHostAlloc(&stage[i], chunk, cudaHostAllocDefault), "cudaHostAlloc (staging)");
            ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
        }
        fd = ::open(path.c_str(), O_RDONLY);
        if (fd < 0) throw IoErr("cannot open '" + path + "'");
        size_t off = 0;
        int k = 0;
        bool used[2] = {false, false};
        while (off < bytes) {
            const size_t len = std::min(chunk, bytes - off);
            if (used[k]) ck(cudaEventSynchronize(done[k]), "cudaEventSynchronize");  // staging buffer free again
            size_t got = 0;
            while (got < len) {
                const ssize_t r = ::pread(fd, static_cast<char*>(stage[k]) + got, len - got, (off_t)(off + got));
                if (r < 0 && errno == EINTR) continue;
                if (r <= 0) throw IoErr(path + ": short read");
                got += (size_t)r;
            }
            ck(cudaMemcpyAsync(reinterpret_cast<char*>(d_out) + off, stage[k], len, cudaMemcpyHostToDevice, st),
               "cudaMemcpyAsync (grid H2D)");
            ck(cudaEventRecord(done[k], st), "cudaEventRecord");
            used[k] = true;
            off += len;
            k ^= 1;
        }
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

}  // namespace

extern "C" {

fsx_status fsx_write_grid(const fsx_shape* shape, const double* data, const char* path, int32_t format) {
    return guarded_io([&] {
        if (!path || !data) throw ArgErr("fsx_write_grid: null argument");
        if (format == FSX_GRID_RAW) write_raw(shape, data, path);
        else if (format == FSX_GRID_CSV) write_csv(shape, data, path);
        else throw ArgErr("fsx_write_grid: unknown format");
    });
}

fsx_status fsx_read_grid_shape(const char* path, fsx_shape* shape) {
    return guarded_io([&] {
        if (!path || !shape) throw ArgErr("fsx_read_grid_shape: null argument");
        *shape = exists(meta_path(path)) ? read_raw_shape(path) : scan_csv(path).shape;
    });
}

fsx_status fsx_read_grid(const char* path, const fsx_shape* shape, double* out) {
    return guarded_io([&] {
        if (!path || !out) throw ArgErr("fsx_read_grid: null argument");
        if (exists(meta_path(path))) {
            read_raw(path, shape, out);
        } else {
            const Csv c = scan_csv(path);
            same_shape(c.shape, shape, path);
            read_csv(c, path, out);
        }
    });
}

fsx_status fsx_load_grid_device(const char* path, const fsx_shape* shape, double* d_out, const fsx_options* opt) {
    return guarded_io([&] {
        if (!path) throw ArgErr("fsx_load_grid_device: null path");
        load_device(path, shape, d_out, opt);
    });
}

fsx_status fsx_format_stage_table(const fsx_stage_timings* st, double total, double naive_seconds, char* buf,
                                  int64_t buflen) {
    return guarded_io([&] {
        if (!st || !buf || buflen <= 0) throw ArgErr("fsx_format_stage_table: null argument");
        // proj/src/runner.cpp:46-62: "  <name padded to 20><value, fixed, 6 decimals>"
        std::string out = "stage timings (seconds):\n";
        auto row = [&](const char* name, double v) {
            char line[96];
            std::snprintf(line, sizeof line, "  %-20s%.6f\n", name, v);
            out += line;
        };
        row("forward_fft", st->forward_fft);
        row("squaring", st->squaring);
        row("hadamard", st->hadamard);
        row("inverse_fft", st->inverse_fft);
        row("boundary_recursion", st->boundary_recursion);
        row("total", total);
        if (naive_seconds >= 0) row("naive_total", naive_seconds);
        if ((int64_t)out.size() + 1 > buflen) throw ArgErr("fsx_format_stage_table: buffer too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
    });
}

}  // extern "C"
