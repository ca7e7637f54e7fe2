// mmio.cpp -- MatrixMarket ingestion for the B200 backend.
//
// Host-side parse of a "matrix coordinate" file into an entry list with the
// reference's exact acceptance rules and messages (src/matrix/io.cpp:71-191:
// real / integer / pattern fields, general / symmetric symmetry, symmetric
// files expanded to both triangles with single diagonal entries, 1-based
// indices, comment and blank lines skipped, UnsupportedFormatError /
// FormatError with the offending line number).  The canonical COO
// (stable sort + duplicate sum) is then assembled on the device by
// lbk_coo_assemble_f64, replacing the reference's host coo_from_entries.
// The whole file is read in one go and tokenised with std::from_chars
// (no iostream per line), which is what makes SuiteSparse-size files cheap.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "lbk.h"

struct lbk_mm_s {
    int32_t nrows = 0, ncols = 0;
    std::vector<int32_t> rows, cols;
    std::vector<double> vals;
};

namespace {

thread_local std::string g_mm_err;

struct MmError {
    lbk_status status;
    std::string msg;
};

[[noreturn]] void fail(const std::string& m, size_t line)
{
    throw MmError{LBK_FORMAT_ERROR, m + " (line " + std::to_string(line) + ")"};
}
[[noreturn]] void fail_unsupported(const std::string& m, size_t line)
{
    throw MmError{LBK_UNSUPPORTED_FORMAT, m + " (line " + std::to_string(line) + ")"};
}

std::string lower(std::string_view s)
{
    std::string o(s);
    for (auto& c : o) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return o;
}

// whitespace tokens of one line (istringstream >> semantics)
int tokens(std::string_view line, std::string_view* out, int max)
{
    int n = 0;
    size_t i = 0;
    while (i < line.size() && n < max) {
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        if (i >= line.size()) break;
        size_t j = i;
        while (j < line.size() && !std::isspace(static_cast<unsigned char>(line[j]))) ++j;
        out[n++] = line.substr(i, j - i);
        i = j;
    }
    return n;
}

int64_t parse_index(std::string_view t, size_t line)
{
    int64_t v = 0;
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    if (ec != std::errc{} || p != t.data() + t.size())
        fail("invalid index '" + std::string(t) + "'", line);
    return v;
}

double parse_value(std::string_view t, size_t line)
{
    double v = 0;
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    if (ec != std::errc{} || p != t.data() + t.size())
        fail("invalid numeric value '" + std::string(t) + "'", line);
    return v;
}

struct LineReader {
    const char* p;
    const char* e;
    size_t no = 0;
    bool next(std::string_view& out)
    {
        if (p >= e) return false;
        const char* q = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
        const char* end = q ? q : e;
        out = std::string_view(p, static_cast<size_t>(end - p));
        // '\r' is kept, as std::getline keeps it (io.cpp:77-137): it is
        // whitespace to the tokenizer, so CRLF entry lines parse, and a CRLF
        // blank line is non-empty -- rejected exactly where the reference
        // rejects it (CRLF parity decided, tests/test_mmio.py)
        p = q ? q + 1 : e;
        ++no;
        return true;
    }
};

void parse(const std::string& text, lbk_mm_s& m)
{
    LineReader rd{text.data(), text.data() + text.size()};
    std::string_view line;
    if (!rd.next(line)) fail("empty stream, expected MatrixMarket banner", 1);
    std::string_view tk[6];
    const int nt = tokens(line, tk, 5);
    std::string tag = nt > 0 ? lower(tk[0]) : "", object = nt > 1 ? lower(tk[1]) : "",
                format = nt > 2 ? lower(tk[2]) : "", field = nt > 3 ? lower(tk[3]) : "",
                symmetry = nt > 4 ? lower(tk[4]) : "";
    if (tag != "%%matrixmarket") fail("missing %%MatrixMarket banner", rd.no);
    if (object != "matrix") fail_unsupported("unsupported object '" + object + "'", rd.no);
    if (format != "coordinate")
        fail_unsupported("unsupported format '" + format + "', only coordinate is accepted", rd.no);
    if (field != "real" && field != "integer" && field != "pattern")
        fail_unsupported("unsupported field '" + field + "'", rd.no);
    if (symmetry != "general" && symmetry != "symmetric")
        fail_unsupported("unsupported symmetry '" + symmetry + "'", rd.no);
    const bool pattern = field == "pattern", symmetric = symmetry == "symmetric";

    int64_t nrows = 0, ncols = 0, nnz = 0;
    for (;;) {
        if (!rd.next(line)) fail("unexpected end of stream before size line", rd.no + 1);
        if (line.empty() || line[0] == '%') continue;
        const int k = tokens(line, tk, 4);
        if (k != 3) fail("size line must be '<rows> <cols> <nnz>'", rd.no);
        nrows = parse_index(tk[0], rd.no);
        ncols = parse_index(tk[1], rd.no);
        nnz = parse_index(tk[2], rd.no);
        if (nrows < 0 || ncols < 0 || nnz < 0) fail("negative size", rd.no);
        break;
    }
    // nnz comes from the file: cap the reservation by what the text can
    // hold (an entry line has >= 4 bytes), so a hostile header can neither
    // overflow 2*nnz nor make reserve() throw
    const int64_t fit = static_cast<int64_t>(text.size() / 4) + 1;
    const int64_t want = nnz < fit ? nnz : fit;
    const size_t cap = static_cast<size_t>(symmetric ? 2 * want : want);
    m.rows.reserve(cap);
    m.cols.reserve(cap);
    m.vals.reserve(cap);
    int64_t seen = 0;
    while (seen < nnz) {
        if (!rd.next(line))
            fail("expected " + std::to_string(nnz) + " entries, got " + std::to_string(seen),
                 rd.no + 1);
        if (line.empty() || line[0] == '%') continue;
        const int k = tokens(line, tk, 3);
        if (k < 2) fail("entry line must start with '<row> <col>'", rd.no);
        double value = 1.0;
        if (!pattern) {
            if (k < 3) fail("missing value", rd.no);
            value = parse_value(tk[2], rd.no);
        }
        const int64_t row = parse_index(tk[0], rd.no) - 1, col = parse_index(tk[1], rd.no) - 1;
        if (row < 0 || row >= nrows || col < 0 || col >= ncols)
            fail("entry (" + std::string(tk[0]) + ", " + std::string(tk[1]) + ") outside declared " +
                     std::to_string(nrows) + "x" + std::to_string(ncols) + " shape",
                 rd.no);
        m.rows.push_back(static_cast<int32_t>(row));
        m.cols.push_back(static_cast<int32_t>(col));
        m.vals.push_back(value);
        if (symmetric && row != col) {
            m.rows.push_back(static_cast<int32_t>(col));
            m.cols.push_back(static_cast<int32_t>(row));
            m.vals.push_back(value);
        }
        ++seen;
    }
    m.nrows = static_cast<int32_t>(nrows);
    m.ncols = static_cast<int32_t>(ncols);
}

}  // namespace

extern "C" {

const char* lbk_mm_last_error(void) { return g_mm_err.c_str(); }

lbk_status lbk_mm_read(const char* path, lbk_mm* out)
{
    if (!path || !out) return LBK_USAGE_ERROR;
    try {
        std::FILE* f = std::fopen(path, "rb");
        if (!f) {
            g_mm_err = std::string("cannot open '") + path + "'";
            return LBK_FORMAT_ERROR;
        }
        std::string text;
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        text.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
        if (sz > 0 && std::fread(text.data(), 1, text.size(), f) != text.size()) {
            std::fclose(f);
            g_mm_err = std::string("cannot read '") + path + "'";
            return LBK_FORMAT_ERROR;
        }
        std::fclose(f);
        auto m = std::make_unique<lbk_mm_s>();
        parse(text, *m);
        *out = m.release();
        return LBK_OK;
    } catch (const MmError& e) {
        g_mm_err = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_mm_err = "host allocation failed";
        return LBK_OUT_OF_MEMORY;
    } catch (const std::length_error&) {
        g_mm_err = "host allocation failed (size)";
        return LBK_OUT_OF_MEMORY;
    } catch (const std::exception& e) {  // nothing may cross the C ABI
        g_mm_err = e.what();
        return LBK_FORMAT_ERROR;
    }
}

lbk_status lbk_mm_info(lbk_mm m, int32_t* nrows, int32_t* ncols, int64_t* n_entries)
{
    if (!m) return LBK_USAGE_ERROR;
    if (nrows) *nrows = m->nrows;
    if (ncols) *ncols = m->ncols;
    if (n_entries) *n_entries = static_cast<int64_t>(m->vals.size());
    return LBK_OK;
}

lbk_status lbk_mm_entries(lbk_mm m, const int32_t** rows, const int32_t** cols, const double** vals)
{
    if (!m) return LBK_USAGE_ERROR;
    if (rows) *rows = m->rows.data();
    if (cols) *cols = m->cols.data();
    if (vals) *vals = m->vals.data();
    return LBK_OK;
}

lbk_status lbk_mm_free(lbk_mm m)
{
    delete m;
    return LBK_OK;
}

}  // extern "C"
