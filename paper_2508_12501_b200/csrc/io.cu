// Mesh and operator I/O either side of the path:
// read_obj / write_obj (proj/src/mesh_io.cpp:19-82) and
// SparseOperator::write_matrix_market (proj/src/sparse.cpp:247-259), with the
// reference's formats, error messages and (for the writers) byte-identical
// output. Host code: the writers export the level's arrays from the device.
#include "common.cuh"

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace {

thread_local std::string g_io_err;

struct ObjMesh {
    std::vector<double> pos;
    std::vector<int> tri;
};

// read_obj (mesh_io.cpp:19-69): "v x y z" and "f i j k" records (bare 1-based
// indices), '#' comments and blank lines skipped, anything else is an error.
decmg_gpu::Status read_obj(const std::string& path, ObjMesh* m) {
    using decmg_gpu::Status;
    std::ifstream in(path);
    if (!in) return Status::Err(DECMG_RUNTIME, "cannot open " + path);
    auto fail = [&](int line, const std::string& what) {
        return Status::Err(DECMG_RUNTIME, path + ":" + std::to_string(line) + ": " + what);
    };
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        std::istringstream is(line);
        std::string kind;
        if (!(is >> kind) || kind[0] == '#') continue;
        if (kind == "v") {
            double x, y, z;
            if (!(is >> x >> y >> z)) return fail(lineno, "malformed vertex record");
            m->pos.insert(m->pos.end(), {x, y, z});
        } else if (kind == "f") {
            std::vector<long> idx;
            std::string tok;
            while (is >> tok) {
                std::size_t used = 0;
                long v = 0;
                try {
                    v = std::stol(tok, &used);
                } catch (const std::exception&) {
                    return fail(lineno, "malformed face index '" + tok + "'");
                }
                if (used != tok.size()) return fail(lineno, "malformed face index '" + tok + "'");
                idx.push_back(v);
            }
            if (idx.size() != 3) return fail(lineno, "non-triangular face at line " + std::to_string(lineno));
            const long nv = static_cast<long>(m->pos.size() / 3);
            for (int i = 0; i < 3; ++i) {
                if (idx[i] < 1 || idx[i] > nv) return fail(lineno, "face index out of range");
                m->tri.push_back(static_cast<int>(idx[i] - 1));
            }
        } else {
            return fail(lineno, "unsupported record '" + kind + "'");
        }
    }
    if (m->tri.empty()) return Status::Err(DECMG_RUNTIME, path + ": no faces");
    return Status::Ok();
}

template <class T>
decmg_gpu::Status fetch(const T* dev, size_t n, std::vector<T>* h) {
    h->resize(n);
    if (n && cudaMemcpy(h->data(), dev, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
        return decmg_gpu::Status::Err(DECMG_CUDA, "export: device copy failed");
    return decmg_gpu::Status::Ok();
}

int io_fail(decmg_gpu_ctx* ctx, const decmg_gpu::Status& s) {
    if (ctx) ctx->err = s.msg;
    g_io_err = s.msg;
    return s.code;
}

}  // namespace

extern "C" {

DECMG_API const char* decmg_io_last_error(void) { return g_io_err.c_str(); }

DECMG_API int decmg_read_obj(const char* path, double* pos, int* nv, int* tri, int* nt) {
    if (!path || !nv || !nt) return DECMG_INVALID_ARGUMENT;
    ObjMesh m;
    const decmg_gpu::Status s = read_obj(path, &m);
    if (!s.ok()) return io_fail(nullptr, s);
    const int n = static_cast<int>(m.pos.size() / 3), t = static_cast<int>(m.tri.size() / 3);
    if (pos) std::copy(m.pos.begin(), m.pos.end(), pos);
    if (tri) std::copy(m.tri.begin(), m.tri.end(), tri);
    *nv = n;
    *nt = t;
    return DECMG_OK;
}

// write_obj (mesh_io.cpp:71-82) of level k's complex
DECMG_API int decmg_gpu_write_obj(decmg_gpu_ctx* ctx, int level, const char* path) {
    if (!ctx || !path) return DECMG_INVALID_ARGUMENT;
    if (level < 0 || level >= static_cast<int>(ctx->lv.size()) || !ctx->lv[level].pos)
        return io_fail(ctx, decmg_gpu::Status::Err(DECMG_INVALID_ARGUMENT, "write_obj: level has no mesh"));
    cudaSetDevice(ctx->device);
    const decmg_gpu::Level& m = ctx->lv[level];
    std::vector<double> pos;
    std::vector<int> cor;
    decmg_gpu::Status s = fetch(m.pos, 3 * static_cast<size_t>(m.nv), &pos);
    if (s.ok()) s = fetch(m.corners, 3 * static_cast<size_t>(m.nt), &cor);
    if (!s.ok()) return io_fail(ctx, s);
    std::FILE* f = std::fopen(path, "w");
    if (!f) return io_fail(ctx, decmg_gpu::Status::Err(DECMG_RUNTIME, std::string("cannot open ") + path + " for writing"));
    for (int v = 0; v < m.nv; ++v) std::fprintf(f, "v %.17g %.17g %.17g\n", pos[3 * v], pos[3 * v + 1], pos[3 * v + 2]);
    for (int t = 0; t < m.nt; ++t) std::fprintf(f, "f %d %d %d\n", cor[3 * t] + 1, cor[3 * t + 1] + 1, cor[3 * t + 2] + 1);
    std::fclose(f);
    return DECMG_OK;
}

// SparseOperator::write_matrix_market (sparse.cpp:247-259) of level k's L
// ("laplacian0", operators.cpp:120), P ("prolongation", multigrid.cpp:215) or
// R ("restriction", geometric_map.cpp:222): entries in column-major (CSC)
// order, rows ascending within a column, %.17g values.
DECMG_API int decmg_gpu_write_matrix_market(decmg_gpu_ctx* ctx, int level, char op, const char* path) {
    if (!ctx || !path) return DECMG_INVALID_ARGUMENT;
    const int L = static_cast<int>(ctx->lv.size());
    if (level < 0 || level >= L || (op != 'L' && level + 1 >= L) || (op != 'L' && op != 'P' && op != 'R'))
        return io_fail(ctx, decmg_gpu::Status::Err(DECMG_INVALID_ARGUMENT, "write_matrix_market: no such operator"));
    cudaSetDevice(ctx->device);
    const decmg_gpu::Level& m = ctx->lv[level];
    const int nc = level + 1 < L ? ctx->lv[level + 1].nv : 0;
    const int* rp = op == 'L' ? m.L_rp : (op == 'P' ? m.P_rp : m.R_rp);
    const int* ci = op == 'L' ? m.L_ci : (op == 'P' ? m.P_ci : m.R_ci);
    const double* v = op == 'L' ? m.L_v : (op == 'P' ? m.P_v : m.R_v);
    const int rows = op == 'R' ? nc : m.nv, cols = op == 'P' ? nc : m.nv;
    const int64_t nnz = op == 'L' ? m.nnzL : (op == 'P' ? m.nnzP : m.nnzR);
    const char* tag = op == 'L' ? "laplacian0" : (op == 'P' ? "prolongation" : "restriction");
    std::vector<int> hrp, hci;
    std::vector<double> hv;
    decmg_gpu::Status s = fetch(rp, static_cast<size_t>(rows) + 1, &hrp);
    if (s.ok()) s = fetch(ci, static_cast<size_t>(nnz), &hci);
    if (s.ok()) s = fetch(v, static_cast<size_t>(nnz), &hv);
    if (!s.ok()) return io_fail(ctx, s);
    // CSR -> CSC: counting sort by column, rows visited in ascending order
    std::vector<int64_t> cp(static_cast<size_t>(cols) + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) ++cp[hci[k] + 1];
    for (int j = 0; j < cols; ++j) cp[j + 1] += cp[j];
    std::vector<int> ri(nnz);
    std::vector<double> cv(nnz);
    std::vector<int64_t> next(cp.begin(), cp.end() - 1);
    for (int i = 0; i < rows; ++i)
        for (int k = hrp[i]; k < hrp[i + 1]; ++k) {
            const int64_t dst = next[hci[k]]++;
            ri[dst] = i;
            cv[dst] = hv[k];
        }
    std::FILE* f = std::fopen(path, "w");
    if (!f) return io_fail(ctx, decmg_gpu::Status::Err(DECMG_RUNTIME, std::string("cannot open ") + path + " for writing"));
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%% %s\n", tag);
    std::fprintf(f, "%d %d %lld\n", rows, cols, static_cast<long long>(nnz));
    for (int j = 0; j < cols; ++j)
        for (int64_t k = cp[j]; k < cp[j + 1]; ++k) std::fprintf(f, "%d %d %.17g\n", ri[k] + 1, j + 1, cv[k]);
    std::fclose(f);
    return DECMG_OK;
}

}  // extern "C"
