// Matrix Market coordinate I/O (the load step before the
// path): load_matrix_market / write_matrix_market of matrix_market.hpp:27-116,
// same accepted formats, same symmetric expansion (an off-diagonal (i, j)
// entry also yields (j, i)), same error messages (IoError).
//
// Host code. The file is read in one piece and the entry lines are parsed in
// parallel chunks (split at line boundaries); entries keep file order, the
// first error in file order is the one reported, and lines after the declared
// entry count are ignored, as the reference's sequential reader does. Numbers
// follow the reference's istream extraction (long long, then double: sign,
// digits, point, exponent; no inf/nan/hex).
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "errors.hpp"
#include "mtx.hpp"

namespace fb {


namespace {

std::string lower(std::string s) {
    for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}

inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f'; }

// istream >> long long on [p, e): skip whitespace, [+-]digits
bool parse_ll(const char*& p, const char* e, long long& out) {
    while (p < e && (is_ws(*p) || *p == '\n')) ++p;
    const char* s = p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* d = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == d) return false;
    std::string tok(s, size_t(p - s));
    errno = 0;
    char* end = nullptr;
    out = std::strtoll(tok.c_str(), &end, 10);
    return errno == 0 && end == tok.c_str() + tok.size();
}

// istream >> double on [p, e): [+-] digits [. digits] [eE [+-] digits]
bool parse_double(const char*& p, const char* e, double& out) {
    while (p < e && (is_ws(*p) || *p == '\n')) ++p;
    const char* s = p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    int nd = 0;
    while (p < e && *p >= '0' && *p <= '9') { ++p; ++nd; }
    if (p < e && *p == '.') {
        ++p;
        while (p < e && *p >= '0' && *p <= '9') { ++p; ++nd; }
    }
    if (nd == 0) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        const char* q = p + 1;
        if (q < e && (*q == '+' || *q == '-')) ++q;
        const char* qd = q;
        while (q < e && *q >= '0' && *q <= '9') ++q;
        if (q == qd) return false;  // dangling exponent: extraction fails
        p = q;
    }
    std::string tok(s, size_t(p - s));
    errno = 0;
    out = std::strtod(tok.c_str(), nullptr);
    return !(errno == ERANGE && std::isinf(out));  // overflow: failbit
}

// the first whitespace-separated word of [p, e)
std::string word(const char*& p, const char* e) {
    while (p < e && is_ws(*p)) ++p;
    const char* s = p;
    while (p < e && !is_ws(*p)) ++p;
    return std::string(s, size_t(p - s));
}

struct Chunk {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    int64_t lines = 0;         // entry lines seen (non-blank, non-comment)
    int64_t err_line = -1;     // chunk-local ordinal of the first bad entry line
    std::string err;
};

}  // namespace

void mtx_read(const std::string& path, MtxData& out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open '" + path + "' for reading");
    std::string buf;
    {
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        buf.resize(sz > 0 ? size_t(sz) : 0);
        const size_t got = sz > 0 ? std::fread(&buf[0], 1, buf.size(), f) : 0;
        std::fclose(f);
        buf.resize(got);
    }
    const char* p = buf.data();
    const char* const e = p + buf.size();
    auto next_line = [&](const char*& q, const char*& ls, const char*& le) {  // getline
        if (q >= e) return false;
        ls = q;
        const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(e - q)));
        le = nl ? nl : e;
        q = nl ? nl + 1 : e;
        return true;
    };
    const char *ls, *le;
    if (!next_line(p, ls, le)) throw IoError(path + ": empty file");
    {
        const char* b = ls;
        const std::string tag = word(b, le), object = lower(word(b, le)), format = lower(word(b, le)),
                          field = lower(word(b, le)), symmetry = lower(word(b, le));
        if (tag != "%%MatrixMarket") throw IoError(path + ": missing %%MatrixMarket banner");
        if (object != "matrix" || format != "coordinate")
            throw IoError(path + ": only coordinate matrices are supported");
        if (field != "real" && field != "integer") throw IoError(path + ": only real-valued matrices are supported");
        if (symmetry != "general" && symmetry != "symmetric")
            throw IoError(path + ": only general or symmetric storage is supported");
        out.r.clear();
        out.c.clear();
        out.v.clear();
        // symmetric flag carried below
        const bool symmetric = symmetry == "symmetric";
        do {
            if (!next_line(p, ls, le)) throw IoError(path + ": missing size line");
        } while (ls == le || *ls == '%');
        long long rows = -1, cols = -1, nnz = -1;
        {
            const char* q = ls;
            if (!(parse_ll(q, le, rows) && parse_ll(q, le, cols) && parse_ll(q, le, nnz)) || rows < 0 || cols < 0 ||
                nnz < 0)
                throw IoError(path + ": malformed size line '" + std::string(ls, size_t(le - ls)) + "'");
        }
        if (symmetric && rows != cols) throw IoError(path + ": symmetric matrix must be square");
        out.rows = rows;
        out.cols = cols;

        // entry region [p, e): chunks at line boundaries, parsed in parallel
        const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        const size_t span = size_t(e - p);
        const int nch = span < (1u << 20) ? 1 : int(nt);
        std::vector<const char*> cut(size_t(nch) + 1);
        cut[0] = p;
        for (int k = 1; k < nch; ++k) {
            const char* q = p + span * size_t(k) / size_t(nch);
            if (q < cut[size_t(k) - 1]) q = cut[size_t(k) - 1];
            const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(e - q)));
            cut[size_t(k)] = nl ? nl + 1 : e;
        }
        cut[size_t(nch)] = e;
        std::vector<Chunk> ch(static_cast<size_t>(nch));
        auto work = [&](int k) {
            Chunk& C = ch[size_t(k)];
            const char* q = cut[size_t(k)];
            const char* qe = cut[size_t(k) + 1];
            const char *a, *b;
            while (q < qe) {
                a = q;
                const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(qe - q)));
                b = nl ? nl : qe;
                q = nl ? nl + 1 : qe;
                if (a == b || *a == '%') continue;
                const int64_t ord = C.lines++;
                if (C.err_line >= 0) continue;  // count lines only after the first error
                const char* t = a;
                long long i = 0, j = 0;
                double v = 0.0;
                if (!(parse_ll(t, b, i) && parse_ll(t, b, j) && parse_double(t, b, v))) {
                    C.err_line = ord;
                    C.err = path + ": malformed entry line '" + std::string(a, size_t(b - a)) + "'";
                    continue;
                }
                if (i < 1 || i > rows || j < 1 || j > cols) {
                    C.err_line = ord;
                    C.err = path + ": entry (" + std::to_string(i) + ", " + std::to_string(j) +
                            ") outside declared dimensions";
                    continue;
                }
                C.r.push_back(i - 1);
                C.c.push_back(j - 1);
                C.v.push_back(v);
                if (symmetric && i != j) {
                    C.r.push_back(j - 1);
                    C.c.push_back(i - 1);
                    C.v.push_back(v);
                }
            }
        };
        if (nch == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (int k = 0; k < nch; ++k) th.emplace_back(work, k);
            for (auto& t : th) t.join();
        }
        // entries in file order up to the declared count; first error before it
        int64_t seen = 0;
        for (int k = 0; k < nch; ++k) {
            const Chunk& C = ch[size_t(k)];
            if (C.err_line >= 0 && seen + C.err_line < nnz) throw IoError(C.err);
            seen += C.lines;
            if (seen >= nnz) break;
        }
        if (seen < nnz) throw IoError(path + ": unexpected end of file after " + std::to_string(seen) + " entries");
        // keep exactly nnz entry lines (a symmetric off-diagonal line gave two triplets)
        int64_t left = nnz;
        for (int k = 0; k < nch && left > 0; ++k) {
            Chunk& C = ch[size_t(k)];
            if (C.lines <= left) {
                out.r.insert(out.r.end(), C.r.begin(), C.r.end());
                out.c.insert(out.c.end(), C.c.begin(), C.c.end());
                out.v.insert(out.v.end(), C.v.begin(), C.v.end());
                left -= C.lines;
            } else {
                // re-walk this chunk's triplets to its first `left` lines
                int64_t taken = 0;
                size_t t = 0;
                while (taken < left && t < C.r.size()) {
                    const bool pair = symmetric && C.r[t] != C.c[t];
                    const size_t w = pair ? 2 : 1;
                    for (size_t u = 0; u < w; ++u) {
                        out.r.push_back(C.r[t + u]);
                        out.c.push_back(C.c[t + u]);
                        out.v.push_back(C.v[t + u]);
                    }
                    t += w;
                    ++taken;
                }
                left = 0;
            }
        }
    }
}

void mtx_write(const std::string& path, int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci,
               const double* v) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open '" + path + "' for writing");
    const int64_t nnz = rp[rows];
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)rows,
                           (long long)cols, (long long)nnz) > 0;
    for (int64_t i = 0; i < rows && ok; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            char b[64];
            std::snprintf(b, sizeof(b), "%.17g", v[p]);
            if (std::fprintf(f, "%lld %lld %s\n", (long long)(i + 1), (long long)(ci[p] + 1), b) < 0) {
                ok = false;
                break;
            }
        }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IoError("failed while writing '" + path + "'");
}

}  // namespace fb
