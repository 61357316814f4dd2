// Matrix Market ingestion (coordinate, real, general | symmetric) -> CSR, restating
// read_matrix_market (src/core/matrix_market.cpp:26-91) and csr_from_triplets
// (src/core/sparse_csr.cpp:38-79): same header rules, 1-based bounds check, symmetric expansion,
// duplicates summed, the same IngestionError texts ("<path>:<line>: <what>").  The file is read
// in one block and parsed with from_chars (no iostreams); triplets are ordered by (row, col)
// with a stable counting sort, so duplicates are summed in file order.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "api.hpp"

namespace bosp {
inline namespace b200 {

namespace {

[[noreturn]] void fail(const std::string& path, size_t line, const std::string& what) {
    throw IngestionError(path + ":" + std::to_string(line) + ": " + what);
}

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

struct Cursor {
    const char* p;
    const char* end;
    bool next_line(const char*& b, const char*& e) {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        if (e > b && e[-1] == '\r') --e;
        return true;
    }
};

const char* skip_ws(const char* s, const char* e) {
    while (s < e && (*s == ' ' || *s == '\t')) ++s;
    return s;
}

template <class T>
bool parse_num(const char*& s, const char* e, T& v) {
    s = skip_ws(s, e);
    if (s >= e) return false;
    if (*s == '+') ++s;  // from_chars rejects a leading '+', iostreams accept it
    const auto r = std::from_chars(s, e, v);
    if (r.ec != std::errc()) return false;
    s = r.ptr;
    return true;
}

std::vector<std::string> words(const char* b, const char* e) {
    std::vector<std::string> w;
    while (true) {
        b = skip_ws(b, e);
        if (b >= e) break;
        const char* s = b;
        while (b < e && *b != ' ' && *b != '\t') ++b;
        w.emplace_back(s, b);
    }
    return w;
}

}  // namespace

SparseMatrixCSR read_matrix_market(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IngestionError(path + ": cannot open file");
    std::string buf;
    {
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
        const size_t got = buf.empty() ? 0 : std::fread(&buf[0], 1, buf.size(), f);
        buf.resize(got);
        std::fclose(f);
    }
    Cursor cur{buf.data(), buf.data() + buf.size()};
    const char *b, *e;
    size_t lineno = 0;
    if (!cur.next_line(b, e)) fail(path, 1, "empty file");
    ++lineno;
    const std::vector<std::string> hdr = words(b, e);
    auto hw = [&](size_t i) { return i < hdr.size() ? hdr[i] : std::string(); };
    if (hw(0) != "%%MatrixMarket") fail(path, lineno, "missing %%MatrixMarket banner");
    if (lower(hw(1)) != "matrix" || lower(hw(2)) != "coordinate")
        fail(path, lineno, "only coordinate matrices are supported");
    if (lower(hw(3)) != "real") fail(path, lineno, "only real-valued matrices are supported (field '" + hw(3) + "')");
    const std::string sym = lower(hw(4));
    if (sym != "general" && sym != "symmetric") fail(path, lineno, "only general or symmetric matrices are supported");
    const bool symmetric = sym == "symmetric";

    uint64_t rows = 0, cols = 0, nnz = 0;
    for (;;) {
        if (!cur.next_line(b, e)) fail(path, lineno + 1, "missing size line");
        ++lineno;
        if (e > b && b[0] == '%') continue;
        const char* s = b;
        if (!(parse_num(s, e, rows) && parse_num(s, e, cols) && parse_num(s, e, nnz))) fail(path, lineno, "malformed size line");
        break;
    }
    std::vector<int64_t> ti, tj;
    std::vector<double> tv;
    const size_t reserve = static_cast<size_t>(std::min<uint64_t>(nnz, uint64_t(1) << 28)) * (symmetric ? 2 : 1);
    ti.reserve(reserve);
    tj.reserve(reserve);
    tv.reserve(reserve);
    uint64_t seen = 0;
    while (seen < nnz) {
        if (!cur.next_line(b, e))
            fail(path, lineno + 1, "unexpected end of file, expected " + std::to_string(nnz) + " entries");
        ++lineno;
        if (e == b || b[0] == '%') continue;
        const char* s = b;
        long long i = 0, j = 0;
        double v = 0.0;
        if (!(parse_num(s, e, i) && parse_num(s, e, j) && parse_num(s, e, v)))
            fail(path, lineno, "malformed coordinate entry");
        if (i < 1 || j < 1 || static_cast<uint64_t>(i) > rows || static_cast<uint64_t>(j) > cols)
            fail(path, lineno, "coordinate out of declared bounds");
        ti.push_back(i - 1);
        tj.push_back(j - 1);
        tv.push_back(v);
        if (symmetric && i != j) {
            ti.push_back(j - 1);
            tj.push_back(i - 1);
            tv.push_back(v);
        }
        ++seen;
    }

    // (row, col) order by two stable counting passes (column, then row); duplicates then sit
    // together in file order and are summed (csr_from_triplets, sparse_csr.cpp:58-73)
    const size_t nt = tv.size();
    std::vector<size_t> by_col(nt), order(nt);
    {
        std::vector<size_t> cnt(static_cast<size_t>(cols) + 1, 0);
        for (size_t k = 0; k < nt; ++k) ++cnt[static_cast<size_t>(tj[k]) + 1];
        for (size_t c = 0; c < cols; ++c) cnt[c + 1] += cnt[c];
        for (size_t k = 0; k < nt; ++k) by_col[cnt[static_cast<size_t>(tj[k])]++] = k;
    }
    std::vector<size_t> rcnt(static_cast<size_t>(rows) + 1, 0);
    for (size_t k = 0; k < nt; ++k) ++rcnt[static_cast<size_t>(ti[k]) + 1];
    for (size_t r = 0; r < rows; ++r) rcnt[r + 1] += rcnt[r];
    {
        std::vector<size_t> pos(rcnt.begin(), rcnt.end() - 1);
        for (size_t q = 0; q < nt; ++q) {
            const size_t k = by_col[q];
            order[pos[static_cast<size_t>(ti[k])]++] = k;
        }
    }
    SparseMatrixCSR m;
    m.rows = static_cast<size_t>(rows);
    m.cols = static_cast<size_t>(cols);
    m.row_offsets.assign(static_cast<size_t>(rows) + 1, 0);
    m.col_indices.reserve(nt);
    m.values.reserve(nt);
    size_t k = 0;
    while (k < nt) {
        const int64_t r = ti[order[k]], c = tj[order[k]];
        double v = 0.0;
        while (k < nt && ti[order[k]] == r && tj[order[k]] == c) v += tv[order[k++]];
        m.col_indices.push_back(static_cast<size_t>(c));
        m.values.push_back(v);
        m.row_offsets[static_cast<size_t>(r) + 1] = m.values.size();
    }
    for (size_t r = 1; r <= rows; ++r) m.row_offsets[r] = std::max(m.row_offsets[r], m.row_offsets[r - 1]);
    m.check_invariants();
    return m;
}

}  // namespace b200
}  // namespace bosp
