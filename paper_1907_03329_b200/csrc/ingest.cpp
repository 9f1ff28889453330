// M4 CSV ingestion straight into the engine's upload layout.
//
// The reference's data path is sequential and goes through a JSON bundle:
//   cmd_prepare (commands.hpp:141-201): parse_m4_train_csv (data.hpp:205-232) ->
//   parse_info_csv (:251-279) -> apply_info (:282-290) -> filter by frequency ->
//   equalize_lengths (:147-160) -> save_prepared (JSON) ; then load_prepared (:49-74) ->
//   Trainer(vector<SeriesRecord>) copying every row again.
// Here the train CSV is read once, its lines are parsed by all host threads in parallel
// (std::from_chars, the reference's own number parser, so values are bit-identical), and the
// kept series' last C + 2*O values land directly in one pinned host block (row-major
// n x (C + 2O) fp64, the layout esrnn_trainer_create uploads with a single async copy and
// lays out time-major on the device).  Errors are the reference's: same exception class
// (status), same message, and the same precedence (the first failing line in file order;
// within a line the id checks before the values; train-file errors before info-file errors
// before join errors).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cuda_runtime_api.h>

#include "esrnn_b200.h"

namespace {

thread_local std::string g_ingest_err;

struct IngestError {
    esrnn_status st;
    std::string msg;
};

[[noreturn]] void fail(esrnn_status st, std::string msg) { throw IngestError{st, std::move(msg)}; }

const char* const kCategoryNames[6] = {"Demographic", "Finance", "Industry", "Macro", "Micro", "Other"};

// data.hpp detail::trim: blanks and \r at both ends, then one pair of enclosing quotes
std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    if (s.size() >= 2 && s.front() == '"' && s.back() == '"') s = s.substr(1, s.size() - 2);
    return s;
}

// data.hpp detail::split_csv_line
template <typename Fn>
void for_each_cell(std::string_view line, Fn&& fn) {
    std::size_t start = 0, c = 0;
    for (std::size_t i = 0; i <= line.size(); ++i) {
        if (i == line.size() || line[i] == ',') {
            if (!fn(c++, trim(line.substr(start, i - start)))) return;
            start = i + 1;
        }
    }
}

int parse_category(std::string_view s) {  // data.hpp:38-42
    for (int i = 0; i < 6; ++i)
        if (s == kCategoryNames[i]) return i;
    fail(ESRNN_VALIDATION_ERROR, "unknown category \"" + std::string(s) + "\"");
}

int parse_frequency(std::string_view s) {  // data.hpp:44-49
    if (s == "Yearly") return 0;
    if (s == "Quarterly") return 1;
    if (s == "Monthly") return 2;
    fail(ESRNN_VALIDATION_ERROR, "unknown frequency \"" + std::string(s) + "\"");
}

// The file mapped read-only (pages faulted in by the parsing threads, in parallel) instead
// of copied into a buffer; falls back to a read for non-mappable files.
struct FileView {
    const char* data = nullptr;
    size_t size = 0;
    void* map = nullptr;
    std::string copy;
    ~FileView() {
        if (map) munmap(map, size);
    }
};

bool read_file(const char* path, FileView& fv) {
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat sb {};
    if (fstat(fd, &sb) == 0 && S_ISREG(sb.st_mode) && sb.st_size > 0) {
        void* m = mmap(nullptr, static_cast<size_t>(sb.st_size), PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
        if (m != MAP_FAILED) {
            madvise(m, static_cast<size_t>(sb.st_size), MADV_SEQUENTIAL | MADV_WILLNEED);
            fv.map = m;
            fv.data = static_cast<const char*>(m);
            fv.size = static_cast<size_t>(sb.st_size);
            close(fd);
            return true;
        }
    }
    char buf[1 << 16];
    ssize_t got;
    while ((got = read(fd, buf, sizeof buf)) > 0) fv.copy.append(buf, static_cast<size_t>(got));
    close(fd);
    fv.data = fv.copy.data();
    fv.size = fv.copy.size();
    return true;
}

// std::getline semantics: '\n'-terminated lines; a last line without '\n' counts, an empty
// tail after the final '\n' does not.  Newline positions found by all threads.
std::vector<std::string_view> split_lines(const FileView& buf, int threads) {
    const size_t n = buf.size;
    const int P = std::max(1, std::min<int>(threads, static_cast<int>(n / (1 << 20)) + 1));
    std::vector<std::vector<size_t>> nl(P);
    std::vector<std::thread> th;
    for (int p = 0; p < P; ++p)
        th.emplace_back([&, p] {
            const size_t lo = n * p / P, hi = n * (p + 1) / P;
            const char* b = buf.data;
            for (size_t i = lo; i < hi;) {
                const void* q = std::memchr(b + i, '\n', hi - i);
                if (!q) break;
                const size_t pos = static_cast<const char*>(q) - b;
                nl[p].push_back(pos);
                i = pos + 1;
            }
        });
    for (auto& t : th) t.join();
    std::vector<std::string_view> lines;
    size_t start = 0;
    for (auto& v : nl)
        for (size_t pos : v) {
            lines.emplace_back(buf.data + start, pos - start);
            start = pos + 1;
        }
    if (start < n) lines.emplace_back(buf.data + start, n - start);
    return lines;
}

struct Row {
    std::string_view id;
    int line = -1;
    int64_t off = 0;  // into the owning chunk's value store
    int32_t len = 0;
    int chunk = 0;
};

struct LineError {
    int line = INT32_MAX;
    bool id_stage = false;  // raised before the duplicate-id check of its line
    esrnn_status st = ESRNN_OK;
    std::string msg;
};

struct Parsed {
    std::vector<Row> rows;                  // data rows in file order
    std::vector<std::vector<double>> vals;  // per chunk
};

// parse_m4_train_csv (data.hpp:205-232), lines split over the threads
Parsed parse_train(const std::vector<std::string_view>& lines, int threads) {
    const int nl = static_cast<int>(lines.size());
    const int P = std::max(1, std::min(threads, nl / 256 + 1));
    std::vector<std::vector<Row>> rows(P);
    std::vector<std::vector<double>> vals(P);
    std::vector<LineError> errs(P);
    std::vector<std::thread> th;
    for (int p = 0; p < P; ++p)
        th.emplace_back([&, p] {
            const int lo = 1 + static_cast<int>(static_cast<int64_t>(nl - 1) * p / P);  // line 0 = header
            const int hi = 1 + static_cast<int>(static_cast<int64_t>(nl - 1) * (p + 1) / P);
            auto& R = rows[p];
            auto& V = vals[p];
            if (hi > lo) {  // ~7 bytes per cell in M4 files: one allocation per chunk
                const size_t bytes = static_cast<size_t>(lines[hi - 1].data() - lines[lo].data()) + lines[hi - 1].size();
                V.reserve(bytes / 6 + 16);
                R.reserve(static_cast<size_t>(hi - lo));
            }
            for (int li = lo; li < hi; ++li) {
                const std::string_view line = lines[li];
                if (trim(line).empty()) continue;
                Row r;
                r.line = li;
                r.chunk = p;
                r.off = static_cast<int64_t>(V.size());
                LineError& e = errs[p];
                for_each_cell(line, [&](size_t c, std::string_view cell) {
                    if (c == 0) {
                        r.id = cell;
                        if (cell.empty()) e = {li, true, ESRNN_PARSE_ERROR, "data row with empty id"};
                        return !cell.empty();
                    }
                    if (cell.empty()) return false;
                    double v = 0.0;
                    const char* last = cell.data() + cell.size();
                    auto [ptr, ec] = std::from_chars(cell.data(), last, v);
                    if (ec != std::errc() || ptr != last) {
                        e = {li, false, ESRNN_PARSE_ERROR,
                             "row " + std::string(r.id) + ", column " + std::to_string(c + 1) + ": \"" +
                                 std::string(cell) + "\" is not a number"};
                        return false;
                    }
                    if (!(v > 0.0)) {
                        e = {li, false, ESRNN_VALIDATION_ERROR,
                             "row " + std::string(r.id) + ", column " + std::to_string(c + 1) +
                                 ": values must be strictly positive, got " + std::string(cell)};
                        return false;
                    }
                    V.push_back(v);
                    return true;
                });
                if (e.line == li) {
                    R.push_back(r);  // the id still takes part in the duplicate check
                    break;
                }
                r.len = static_cast<int32_t>(V.size() - r.off);
                R.push_back(r);
            }
        });
    for (auto& t : th) t.join();
    // the first error in file order: per-chunk first parse errors and duplicate ids (checked
    // before a line's values, after its empty-id check)
    LineError first;
    for (auto& e : errs)
        if (e.line < first.line) first = e;
    Parsed out;
    size_t total = 0;
    for (auto& R : rows) total += R.size();
    out.rows.reserve(total);
    std::unordered_set<std::string_view> seen;
    seen.reserve(total * 2);
    for (auto& R : rows)
        for (const Row& r : R) {
            if (r.line > first.line || (r.line == first.line && first.id_stage)) break;
            if (!seen.insert(r.id).second) fail(ESRNN_VALIDATION_ERROR, "duplicate id \"" + std::string(r.id) + "\"");
            if (r.line == first.line) break;
            out.rows.push_back(r);
        }
    if (first.st != ESRNN_OK) fail(first.st, first.msg);
    out.vals = std::move(vals);
    return out;
}

struct Info {
    int category, frequency;
};

// parse_info_csv (data.hpp:251-279)
std::unordered_map<std::string_view, Info> parse_info(const std::vector<std::string_view>& lines) {
    std::unordered_map<std::string_view, Info> out;
    out.reserve(lines.size() * 2);
    size_t id_col = 0, cat_col = 1, freq_col = 2;
    bool header = true;
    std::vector<std::string_view> cells;
    for (const std::string_view line : lines) {
        cells.clear();
        for_each_cell(line, [&](size_t, std::string_view c) {
            cells.push_back(c);
            return true;
        });
        if (header) {
            header = false;
            for (size_t i = 0; i < cells.size(); ++i) {
                if (cells[i] == "M4id" || cells[i] == "id") id_col = i;
                else if (cells[i] == "category" || cells[i] == "Category") cat_col = i;
                else if (cells[i] == "SP") freq_col = i;
            }
            continue;
        }
        if (trim(line).empty()) continue;
        const size_t need = std::max({id_col, cat_col, freq_col});
        if (cells.size() <= need)
            fail(ESRNN_PARSE_ERROR, "info row \"" + std::string(line) + "\": expected at least " +
                                        std::to_string(need + 1) + " columns");
        const std::string_view id = cells[id_col];
        if (out.count(id)) fail(ESRNN_VALIDATION_ERROR, "duplicate id \"" + std::string(id) + "\" in info file");
        const int cat = parse_category(cells[cat_col]);
        const int fq = parse_frequency(cells[freq_col]);
        out.emplace(id, Info{cat, fq});
    }
    return out;
}

// commands.hpp:84-114 length_stats
void length_stats(std::vector<int64_t> L, esrnn_ingest_stats* st) {
    st->raw_count = static_cast<int64_t>(L.size());
    if (L.empty()) return;
    std::sort(L.begin(), L.end());
    double acc = 0.0;
    for (int64_t v : L) acc += static_cast<double>(v);
    st->len_mean = acc / static_cast<double>(L.size());
    double sq = 0.0;
    for (int64_t v : L) sq += (static_cast<double>(v) - st->len_mean) * (static_cast<double>(v) - st->len_mean);
    st->len_stddev = L.size() > 1 ? std::sqrt(sq / static_cast<double>(L.size() - 1)) : 0.0;
    auto quantile = [&](double p) {
        const double pos = p * static_cast<double>(L.size() - 1);
        const size_t lo = static_cast<size_t>(pos);
        const double frac = pos - static_cast<double>(lo);
        if (lo + 1 >= L.size()) return static_cast<double>(L.back());
        return static_cast<double>(L[lo]) * (1.0 - frac) + static_cast<double>(L[lo + 1]) * frac;
    };
    st->len_min = static_cast<double>(L.front());
    st->len_q25 = quantile(0.25);
    st->len_q50 = quantile(0.50);
    st->len_q75 = quantile(0.75);
    st->len_max = static_cast<double>(L.back());
}

}  // namespace

struct esrnn_dataset {
    int64_t n = 0;
    int32_t length = 0;
    double* values = nullptr;  // n x length, pinned when a CUDA device is present
    bool pinned = false;
    std::vector<int32_t> categories;
    std::vector<std::string> ids;
    ~esrnn_dataset() {
        if (!values) return;
        if (pinned) cudaFreeHost(values);
        else std::free(values);
    }
};

extern "C" {

const char* esrnn_ingest_last_error(void) { return g_ingest_err.c_str(); }

esrnn_status esrnn_ingest_m4_csv(const char* train_csv, const char* info_csv, int32_t frequency,
                                 const esrnn_profile* profile, int32_t threads, esrnn_dataset** out,
                                 esrnn_ingest_stats* stats) {
    *out = nullptr;
    g_ingest_err.clear();
    try {
        if (!train_csv || !*train_csv || !info_csv || !*info_csv)
            fail(ESRNN_CONFIG_ERROR, "prepare: paths.train_csv and paths.info_csv are required");
        const int P = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
        const bool timing = std::getenv("ESRNN_INGEST_TIMING") != nullptr;
        auto t_last = std::chrono::steady_clock::now();
        auto lap = [&](const char* what) {
            if (!timing) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[ingest] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
            t_last = now;
        };
        FileView tbuf, ibuf;
        if (!read_file(train_csv, tbuf)) fail(ESRNN_ERROR, "cannot open \"" + std::string(train_csv) + "\"");
        if (!read_file(info_csv, ibuf)) fail(ESRNN_ERROR, "cannot open \"" + std::string(info_csv) + "\"");
        lap("read");
        const auto tlines = split_lines(tbuf, P);
        lap("lines");
        Parsed parsed = parse_train(tlines, P);
        lap("parse");
        const auto info = parse_info(split_lines(ibuf, 1));
        lap("info");
        // apply_info (data.hpp:282-290) in series order, then the frequency filter
        std::vector<const Row*> sel;
        std::vector<int32_t> cats;
        std::vector<int64_t> raw_len;
        for (const Row& r : parsed.rows) {
            auto it = info.find(r.id);
            if (it == info.end()) fail(ESRNN_VALIDATION_ERROR, "series \"" + std::string(r.id) + "\" missing from info file");
            if (it->second.frequency != frequency) continue;
            sel.push_back(&r);
            cats.push_back(it->second.category);
            raw_len.push_back(r.len);
        }
        esrnn_ingest_stats st{};
        length_stats(raw_len, &st);
        lap("join+stats");
        // equalize_lengths (data.hpp:147-160): keep the last C + 2*O values of long-enough rows
        const int32_t target = profile->min_length + 2 * profile->horizon;
        std::vector<int64_t> keep;
        for (size_t i = 0; i < sel.size(); ++i)
            if (sel[i]->len >= target) keep.push_back(static_cast<int64_t>(i));
        if (keep.empty()) fail(ESRNN_VALIDATION_ERROR, "no series after filtering");
        auto ds = std::make_unique<esrnn_dataset>();
        ds->n = static_cast<int64_t>(keep.size());
        ds->length = target;
        const size_t bytes = sizeof(double) * static_cast<size_t>(ds->n) * target;
        void* p = nullptr;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
            ds->pinned = true;
        } else {
            cudaGetLastError();
            p = std::malloc(std::max<size_t>(bytes, 1));
            if (!p) fail(ESRNN_ERROR, "ingest: out of host memory");
        }
        ds->values = static_cast<double*>(p);
        lap("alloc");
        ds->categories.resize(keep.size());
        ds->ids.resize(keep.size());
        const int64_t n = ds->n;
        const int W = static_cast<int>(std::min<int64_t>(P, std::max<int64_t>(1, n / 512)));
        std::vector<std::thread> th;
        for (int w = 0; w < W; ++w)
            th.emplace_back([&, w] {
                for (int64_t i = n * w / W; i < n * (w + 1) / W; ++i) {
                    const Row& r = *sel[keep[i]];
                    const double* src = parsed.vals[r.chunk].data() + r.off + (r.len - target);
                    std::memcpy(ds->values + static_cast<size_t>(i) * target, src, sizeof(double) * target);
                    ds->categories[i] = cats[keep[i]];
                    ds->ids[i].assign(r.id);
                }
            });
        for (auto& t : th) t.join();
        lap("equalise");
        st.kept = n;
        st.dropped = st.raw_count - n;
        st.equalized_length = target;
        if (stats) *stats = st;
        *out = ds.release();
        return ESRNN_OK;
    } catch (const IngestError& e) {
        g_ingest_err = e.msg;
        return e.st;
    } catch (const std::exception& e) {
        g_ingest_err = e.what();
        return ESRNN_ERROR;
    }
}

esrnn_status esrnn_dataset_shape(const esrnn_dataset* d, int64_t* n, int32_t* length) {
    if (!d) return ESRNN_CONTRACT_ERROR;
    *n = d->n;
    *length = d->length;
    return ESRNN_OK;
}

const double* esrnn_dataset_values(const esrnn_dataset* d) { return d ? d->values : nullptr; }

const int32_t* esrnn_dataset_categories(const esrnn_dataset* d) { return d ? d->categories.data() : nullptr; }

const char* esrnn_dataset_id(const esrnn_dataset* d, int64_t i) {
    return (d && i >= 0 && i < d->n) ? d->ids[static_cast<size_t>(i)].c_str() : nullptr;
}

void esrnn_dataset_destroy(esrnn_dataset* d) { delete d; }

}  // extern "C"
