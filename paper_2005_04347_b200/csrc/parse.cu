// parse.cu -- loading a network on the device: parse_network / read_network
// (io.cpp:83-175) and validate (network.cpp:151-216), SURVEY.md 8f ranks 1-2.
//
// The text is copied to HBM once and every step is data-parallel:
//   1. line starts: newline counts per 256-byte chunk, exclusive scan,
//      scatter (u64 positions, so files beyond 4 GB work);
//   2. one thread per line: strip '\r', split on ' '/'\t', classify the first
//      token (comment, "asnn", "inputs", "outputs", "edge", other) and, for
//      edge lines, parse "<source> <target> <weight>" with the from_chars
//      contract of parse_id / parse_weight (parse_tok.cuh);
//   3. significant lines (not blank / comment) are numbered by a scan: the
//      first three must be the header, inputs and outputs lines, every later
//      one an edge line -- the reference's section state machine;
//   4. errors: each line reports its own code and the first failing line wins
//      (64-bit atomicMin of line << 8 | code) -- exactly the line at which
//      the sequential parser would have thrown; duplicate edges come from a
//      stable radix sort by (source, target): the later line of an equal pair;
//   5. the ids of the inputs / outputs lines are tokenised in parallel;
//   6. make_network (sorted unique ids) and validate on the device: duplicate
//      declarations, input/output overlap, inputs with incoming connections,
//      and a Kahn pass for cycles (the cycle's text, only needed for the error
//      message, is recovered by the reference's DFS order on the host).
// The host formats messages from the failing line's own text; every weight
// token is decided on the device (parse_tok.cuh, exact slow path included).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "corpus.hpp"
#include "engine.hpp"
#include "parse_tok.cuh"
#include "sort.cuh"

namespace asnn_b200 {
namespace {

using namespace parse;

constexpr uint32_t kT = 256;
inline uint32_t nb(uint64_t n) { return static_cast<uint32_t>((n + kT - 1) / kT); }

#define CKP(expr)                                                      \
    do {                                                               \
        cudaError_t e_ = (expr);                                       \
        if (e_ != cudaSuccess) return cuda_fail(dev, e_, #expr);       \
    } while (0)
#define RCP(expr)          \
    do {                   \
        int r_ = (expr);   \
        if (r_) return r_; \
    } while (0)

// line kinds
enum : uint8_t { K_SKIP = 0, K_ASNN = 1, K_INPUTS = 2, K_OUTPUTS = 3, K_EDGE = 4, K_OTHER = 5 };
// error codes, in the reference's wording (formatted on the host)
enum : uint8_t {
    ERR_NONE = 0,
    ERR_HEADER,        // expected header 'asnn 1'
    ERR_VERSION,       // unsupported version '<v>'
    ERR_INPUTS_KW,     // expected 'inputs' line
    ERR_OUTPUTS_KW,    // expected 'outputs' line
    ERR_UNKNOWN,       // unknown line '<kw>'
    ERR_EDGE_NTOK,     // edge needs '<source> <target> <weight>'
    ERR_BAD_SRC,       // bad node id '<tok 1>'
    ERR_BAD_TGT,       // bad node id '<tok 2>'
    ERR_BAD_W,         // bad weight '<tok 3>'
    ERR_SELF,          // self-loop at node <id>
    ERR_DUP,           // duplicate edge a->b
    ERR_BAD_ID,        // bad node id '<tok>' on the inputs / outputs line (token index in aux)
};
enum : uint8_t { ES_OK = 0, ES_NTOK, ES_SRC, ES_TGT, ES_W, ES_SELF };

__device__ __forceinline__ bool tok_eq(const char* p, uint32_t n, const char* lit, uint32_t ln) {
    if (n != ln) return false;
    for (uint32_t i = 0; i < n; ++i)
        if (p[i] != lit[i]) return false;
    return true;
}

__global__ void k_nl_count(const char* __restrict__ t, uint64_t len, uint32_t* __restrict__ cnt) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t b = c * 256, e = min(b + 256, len);
    if (b >= len) return;
    uint32_t n = 0;
    for (uint64_t i = b; i < e; ++i) n += t[i] == '\n';
    cnt[c] = n;
}

// starts[j + 1] = position after the j-th newline; starts[0] = 0 and
// starts[n_lines] = len + 1 are written by the host.
__global__ void k_nl_write(const char* __restrict__ t, uint64_t len, const uint32_t* __restrict__ off,
                           uint64_t* __restrict__ starts) {
    const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t b = c * 256, e = min(b + 256, len);
    if (b >= len) return;
    uint32_t j = off[c];
    for (uint64_t i = b; i < e; ++i)
        if (t[i] == '\n') starts[++j] = i + 1;
}

struct LineOut {
    uint8_t* kind;
    uint8_t* estat;
    uint8_t* hdr;  // bit0: exactly 2 tokens, bit1: version token == "1"
    uint32_t* src;
    uint32_t* tgt;
    float* w;
};

// One line per thread (io.cpp:92-146 for one line).
__global__ void k_parse_lines(const char* __restrict__ t, const uint64_t* __restrict__ starts, uint32_t n_lines,
                              LineOut o) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_lines) return;
    const uint64_t s = starts[i];
    uint64_t e = starts[i + 1] - 1;  // excludes the '\n' (or is len for the last line)
    if (e > s && t[e - 1] == '\r') --e;
    uint32_t ts[4], tl[4], nt = 0;
    uint64_t p = s;
    while (p < e) {
        while (p < e && is_ws(t[p])) ++p;
        const uint64_t b = p;
        while (p < e && !is_ws(t[p])) ++p;
        if (p > b) {
            if (nt < 4) {
                ts[nt] = static_cast<uint32_t>(b - s);
                tl[nt] = static_cast<uint32_t>(p - b);
            }
            ++nt;
        }
    }
    uint8_t kind = K_SKIP, es = ES_OK, hdr = 0;
    uint32_t a = 0, b = 0;
    float w = 0.0f;
    if (nt > 0 && t[s + ts[0]] != '#') {
        const char* k0 = t + s + ts[0];
        if (tok_eq(k0, tl[0], "asnn", 4)) {
            kind = K_ASNN;
            hdr = (nt == 2 ? 1 : 0) | (nt >= 2 && tok_eq(t + s + ts[1], tl[1], "1", 1) ? 2 : 0);
        } else if (tok_eq(k0, tl[0], "inputs", 6)) {
            kind = K_INPUTS;
        } else if (tok_eq(k0, tl[0], "outputs", 7)) {
            kind = K_OUTPUTS;
        } else if (tok_eq(k0, tl[0], "edge", 4)) {
            kind = K_EDGE;
            if (nt != 4) {
                es = ES_NTOK;
            } else if (parse_u32(t + s + ts[1], t + s + ts[1] + tl[1], a) != kTokOk) {
                es = ES_SRC;
            } else if (parse_u32(t + s + ts[2], t + s + ts[2] + tl[2], b) != kTokOk) {
                es = ES_TGT;
            } else {
                const uint8_t r = parse_f32(t + s + ts[3], t + s + ts[3] + tl[3], w);
                if (r != kTokOk) es = ES_W;
                else if (a == b) es = ES_SELF;  // checked after the weight, as the reference does
            }
        } else {
            kind = K_OTHER;
        }
    }
    o.kind[i] = kind;
    o.estat[i] = es;
    o.hdr[i] = hdr;
    o.src[i] = a;
    o.tgt[i] = b;
    o.w[i] = w;
}

__global__ void k_sig_flags(const uint8_t* __restrict__ kind, uint32_t n, uint32_t* __restrict__ f) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = kind[i] != K_SKIP;
}

// Per-line errors of the section state machine (io.cpp:104-145); also flags
// the edge lines to keep and the weights the host must resolve.
__global__ void k_line_errors(const uint8_t* __restrict__ kind, const uint8_t* __restrict__ estat,
                              const uint8_t* __restrict__ hdr, const uint32_t* __restrict__ sig, uint32_t n,
                              unsigned long long* __restrict__ first_err, uint32_t* __restrict__ special,
                              uint32_t* __restrict__ keep) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = 0;
    const uint8_t k = kind[i];
    if (k == K_SKIP) return;
    const uint32_t si = sig[i];
    uint8_t err = ERR_NONE;
    if (si < 3) special[si] = i;
    if (si == 0) {
        if (k != K_ASNN || !(hdr[i] & 1)) err = ERR_HEADER;
        else if (!(hdr[i] & 2)) err = ERR_VERSION;
    } else if (si == 1) {
        if (k != K_INPUTS) err = ERR_INPUTS_KW;
    } else if (si == 2) {
        if (k != K_OUTPUTS) err = ERR_OUTPUTS_KW;
    } else if (k != K_EDGE) {
        err = ERR_UNKNOWN;
    } else {
        switch (estat[i]) {
            case ES_NTOK: err = ERR_EDGE_NTOK; break;
            case ES_SRC: err = ERR_BAD_SRC; break;
            case ES_TGT: err = ERR_BAD_TGT; break;
            case ES_W: err = ERR_BAD_W; break;
            case ES_SELF: err = ERR_SELF; break;
            default: keep[i] = 1; break;  // ES_OK
        }
    }
    if (err != ERR_NONE) atomicMin(first_err, (static_cast<unsigned long long>(i) << 8) | err);
}

__global__ void k_compact_edges(const uint32_t* __restrict__ keep, const uint32_t* __restrict__ idx, uint32_t n,
                                const uint32_t* __restrict__ src, const uint32_t* __restrict__ tgt,
                                const float* __restrict__ w, const uint8_t* __restrict__ estat,
                                uint32_t* __restrict__ es, uint32_t* __restrict__ et, float* __restrict__ ew,
                                uint32_t* __restrict__ eline) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !keep[i]) return;
    const uint32_t j = idx[i];
    es[j] = src[i];
    et[j] = tgt[i];
    ew[j] = w[i];
    eline[j] = i;
}

// Sorted by (source, target) with stable order: the later of two equal
// neighbours is a duplicate at its line (io.cpp:137-140).
__global__ void k_dup_edges(const uint32_t* __restrict__ order, uint64_t E, const uint32_t* __restrict__ es,
                            const uint32_t* __restrict__ et, const uint32_t* __restrict__ eline,
                            unsigned long long* __restrict__ first_err) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k == 0 || k >= E) return;
    const uint32_t a = order[k - 1], b = order[k];
    if (es[a] == es[b] && et[a] == et[b])
        atomicMin(first_err, (static_cast<unsigned long long>(eline[b]) << 8) | ERR_DUP);
}

// Token starts of one line [s, e) (the keyword is token 0).
__global__ void k_tok_flags(const char* __restrict__ t, uint64_t s, uint64_t e, uint32_t* __restrict__ f) {
    const uint64_t p = s + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= e) return;
    f[p - s] = !is_ws(t[p]) && (p == s || is_ws(t[p - 1]));
}

// ids[k - 1] for every token k >= 1; bad tokens report their index.
__global__ void k_tok_ids(const char* __restrict__ t, uint64_t s, uint64_t e, const uint32_t* __restrict__ f,
                          const uint32_t* __restrict__ idx, uint32_t* __restrict__ ids,
                          unsigned int* __restrict__ first_bad) {
    const uint64_t p = s + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= e || !f[p - s]) return;
    const uint32_t k = idx[p - s];
    if (k == 0) return;
    uint64_t q = p;
    while (q < e && !is_ws(t[q])) ++q;
    uint32_t v = 0;
    if (parse_u32(t + p, t + q, v) != kTokOk) atomicMin(first_bad, k);
    ids[k - 1] = v;
}

// validate: flags[i] = 1 when x[i] occurs earlier in x (sorted copy + stable
// order: order[] sorts x by value, ties by position).
__global__ void k_dup_decl(const uint32_t* __restrict__ sorted_vals, const uint32_t* __restrict__ order, uint32_t n,
                           uint32_t* __restrict__ flag) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    flag[order[k]] = k > 0 && sorted_vals[k] == sorted_vals[k - 1];
}

__device__ __forceinline__ bool in_sorted(const uint32_t* __restrict__ a, uint32_t n, uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t m = (lo + hi) / 2;
        if (a[m] < v) lo = m + 1;
        else hi = m;
    }
    return lo < n && a[lo] == v;
}

__global__ void k_member_flags(const uint32_t* __restrict__ x, uint64_t n, const uint32_t* __restrict__ set,
                               uint32_t n_set, uint32_t* __restrict__ flag) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = in_sorted(set, n_set, x[i]);
}

__global__ void k_unique_flags(const uint32_t* __restrict__ s, uint64_t n, uint32_t* __restrict__ f) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) f[i] = i == 0 || s[i] != s[i - 1];
}

__global__ void k_scatter_flagged(const uint32_t* __restrict__ v, const uint32_t* __restrict__ f,
                                  const uint32_t* __restrict__ idx, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && f[i]) out[idx[i]] = v ? v[i] : static_cast<uint32_t>(i);
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = static_cast<uint32_t>(i);
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t n,
                             uint32_t* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

__global__ void k_parse_weights(const char* __restrict__ buf, const uint64_t* __restrict__ off, uint64_t n,
                                float* __restrict__ out, uint8_t* __restrict__ status) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float v = 0.0f;
    const uint8_t r = parse_f32(buf + off[i], buf + off[i + 1], v);
    out[i] = r == kTokOk ? v : 0.0f;
    status[i] = r;
}

// validate (network.cpp:180-201): per connection, in the reference's order of
// checks -- unknown endpoint, self-loop, duplicate (a later equal pair in the
// stable (source, target) order), input with an incoming connection.
enum : uint8_t { CS_OK = 0, CS_UNKNOWN, CS_SELF, CS_DUP, CS_INPUT_IN };
__global__ void k_conn_status(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t E,
                              const uint32_t* __restrict__ nodes, uint32_t N, const uint32_t* __restrict__ ins_sorted,
                              uint32_t n_in, const uint32_t* __restrict__ dup, uint32_t* __restrict__ status,
                              uint32_t* __restrict__ flag, uint32_t* __restrict__ valid) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= E) return;
    const uint32_t a = src[k], b = dst[k];
    uint32_t st = CS_OK;
    if (!in_sorted(nodes, N, a) || !in_sorted(nodes, N, b)) st = CS_UNKNOWN;
    else if (a == b) st = CS_SELF;
    else if (dup[k]) st = CS_DUP;
    else if (n_in && in_sorted(ins_sorted, n_in, b)) st = CS_INPUT_IN;
    status[k] = st;
    flag[k] = st != CS_OK;
    valid[k] = st == CS_OK || st == CS_INPUT_IN;
}

// dup[order[k]] = 1 when the k-th pair in stable (source, target) order equals
// the one before it.
__global__ void k_dup_pairs(const uint32_t* __restrict__ order, uint64_t E, const uint32_t* __restrict__ src,
                            const uint32_t* __restrict__ dst, uint32_t* __restrict__ dup) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= E) return;
    const uint32_t b = order[k];
    dup[b] = k > 0 && src[order[k - 1]] == src[b] && dst[order[k - 1]] == dst[b];
}

// declared ids: flags bit0 = an earlier occurrence in the list, bit1 = unknown
__global__ void k_decl_flags(const uint32_t* __restrict__ ids, uint32_t n, const uint32_t* __restrict__ dupf,
                             const uint32_t* __restrict__ nodes, uint32_t N, uint32_t* __restrict__ flags,
                             uint32_t* __restrict__ any) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t f = (dupf[i] ? 1u : 0u) | (in_sorted(nodes, N, ids[i]) ? 0u : 2u);
    flags[i] = f;
    any[i] = f != 0;
}

// normalize (network.cpp:69-85): ids -> positions in the sorted node list
__global__ void k_remap(const uint32_t* __restrict__ nodes, uint32_t N, const uint32_t* __restrict__ in,
                        uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t v = in[i];
    uint32_t lo = 0, hi = N;
    while (lo < hi) {
        const uint32_t m = (lo + hi) / 2;
        if (nodes[m] < v) lo = m + 1;
        else hi = m;
    }
    out[i] = lo;
}

// ---- host helpers ---------------------------------------------------------------
std::vector<std::string_view> split_ws(std::string_view line) {
    std::vector<std::string_view> out;
    size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
        const size_t b = i;
        while (i < line.size() && line[i] != ' ' && line[i] != '\t') ++i;
        if (i > b) out.push_back(line.substr(b, i - b));
    }
    return out;
}

std::string_view line_text(const char* text, uint64_t len, uint64_t s, uint64_t e_plus1) {
    uint64_t e = std::min<uint64_t>(e_plus1 - 1, len);
    std::string_view v(text + s, e - s);
    if (!v.empty() && v.back() == '\r') v.remove_suffix(1);
    return v;
}

// The reference's ParseError message for `code` on this line (io.cpp).
std::string parse_message(uint8_t code, std::string_view line, uint32_t aux) {
    const auto tok = split_ws(line);
    auto t = [&](size_t k) { return k < tok.size() ? std::string(tok[k]) : std::string(); };
    switch (code) {
        case ERR_HEADER: return "expected header 'asnn 1'";
        case ERR_VERSION: return "unsupported version '" + t(1) + "'";
        case ERR_INPUTS_KW: return "expected 'inputs' line";
        case ERR_OUTPUTS_KW: return "expected 'outputs' line";
        case ERR_UNKNOWN: return "unknown line '" + t(0) + "'";
        case ERR_EDGE_NTOK: return "edge needs '<source> <target> <weight>'";
        case ERR_BAD_SRC: return "bad node id '" + t(1) + "'";
        case ERR_BAD_TGT: return "bad node id '" + t(2) + "'";
        case ERR_BAD_W: return "bad weight '" + t(3) + "'";
        case ERR_SELF: {
            uint32_t a = 0;
            std::from_chars(tok[1].data(), tok[1].data() + tok[1].size(), a);
            return "self-loop at node " + std::to_string(a);
        }
        case ERR_DUP: {
            uint32_t a = 0, b = 0;
            std::from_chars(tok[1].data(), tok[1].data() + tok[1].size(), a);
            std::from_chars(tok[2].data(), tok[2].data() + tok[2].size(), b);
            return "duplicate edge " + std::to_string(a) + "->" + std::to_string(b);
        }
        case ERR_BAD_ID: return "bad node id '" + t(aux) + "'";
        default: return "parse error";
    }
}

// find_cycle (network.cpp:107-149) on the device, for the message of a
// network the device already found cyclic: the reference's iterative DFS,
// roots in index order, successors in connection order, run by one thread
// over a stable successor CSR (error path only).  path[0] = length, then the
// cycle's node ids (first == last).
__global__ void k_edge_index(const uint32_t* __restrict__ nodes, uint32_t N, const uint32_t* __restrict__ ids,
                             uint64_t n, uint32_t* __restrict__ idx) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t lo = 0, hi = N;  // lower_bound (network.cpp:57-61)
    const uint32_t v = ids[k];
    while (lo < hi) {
        const uint32_t m = (lo + hi) / 2;
        if (nodes[m] < v) lo = m + 1;
        else hi = m;
    }
    idx[k] = lo;
}
__global__ void k_count_src(const uint32_t* __restrict__ si, uint64_t n, uint32_t* __restrict__ cnt) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) atomicAdd(&cnt[si[k]], 1u);
}
__global__ void k_find_cycle(const uint32_t* __restrict__ nodes, uint32_t N, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ succ, uint8_t* __restrict__ color,
                             uint32_t* __restrict__ st_node, uint32_t* __restrict__ st_pos,
                             uint32_t* __restrict__ path) {
    if (threadIdx.x || blockIdx.x) return;
    path[0] = 0;
    for (uint32_t root = 0; root < N; ++root) {
        if (color[root]) continue;
        uint32_t top = 0;
        st_node[0] = root;
        st_pos[0] = off[root];
        color[root] = 1;
        while (true) {
            const uint32_t node = st_node[top];
            if (st_pos[top] < off[node + 1]) {
                const uint32_t next = succ[st_pos[top]++];
                if (color[next] == 1) {  // walk the stack back to `next`
                    uint32_t len = 0, t = top;
                    path[1 + len++] = nodes[next];
                    while (true) {
                        path[1 + len++] = nodes[st_node[t]];
                        if (st_node[t] == next || t == 0) break;
                        --t;
                    }
                    // reverse path[2 .. len] into the reference's order, then close it
                    for (uint32_t i = 1, j = len; i < j; ++i, --j) {
                        const uint32_t x = path[i];
                        path[i] = path[j];
                        path[j] = x;
                    }
                    path[1 + len++] = nodes[next];
                    path[0] = len;
                    return;
                }
                if (color[next] == 0) {
                    color[next] = 1;
                    ++top;
                    st_node[top] = next;
                    st_pos[top] = off[next];
                }
            } else {
                color[node] = 2;
                if (top == 0) break;
                --top;
            }
        }
    }
}

template <typename T>
int d2h(asnn_dev* dev, std::vector<T>& h, const T* d, uint64_t n) {
    h.resize(n);
    if (n) CKP(download_host(dev, h.data(), d, n * sizeof(T), dev->stream));
    return ASNN_OK;
}

// compaction of flagged positions: out = indices i with f[i] (in order)
int flagged_indices(asnn_dev* dev, const uint32_t* f, uint64_t n, std::vector<uint32_t>& out) {
    cudaStream_t st = dev->stream;
    out.clear();
    if (!n) return ASNN_OK;
    DevBuf<uint32_t> idx, tot, res;
    CKP(idx.alloc(n));
    CKP(tot.alloc(1));
    RCP(exclusive_scan(dev, f, idx.p, n, tot.p, st));
    uint32_t m = 0;
    CKP(cudaMemcpyAsync(&m, tot.p, 4, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    if (!m) return ASNN_OK;
    CKP(res.alloc(m));
    k_scatter_flagged<<<nb(n), kT, 0, st>>>(nullptr, f, idx.p, n, res.p);
    RCP(d2h(dev, out, res.p, m));
    CKP(cudaStreamSynchronize(st));
    return ASNN_OK;
}

// ASNN_PARSE_TIMING=1: phase wall times (synchronising) on stderr.
struct PhaseClock {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t;
    explicit PhaseClock(cudaStream_t s) : on(getenv("ASNN_PARSE_TIMING") != nullptr), st(s), t(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "parse %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// validate (network.cpp:151-216) on device arrays: nodes sorted unique,
// inputs / outputs in declared order, connections in order.  Appends the
// reference's violation messages, in its order, to viol.
int validate_device(asnn_dev* dev, const uint32_t* nodes, uint32_t N, const uint32_t* ins, uint32_t n_in,
                    const uint32_t* outs, uint32_t n_out, const uint32_t* src, const uint32_t* dst, uint64_t E,
                    std::vector<std::string>& viol) {
    cudaStream_t st = dev->stream;
    if (!n_in) viol.push_back("inputs list is empty");
    if (!n_out) viol.push_back("outputs list is empty");
    DevBuf<uint32_t> sorted_in;  // sorted inputs (with repeats) for membership
    const uint32_t* lists[2] = {ins, outs};
    const uint32_t counts[2] = {n_in, n_out};
    for (int k = 0; k < 2; ++k) {  // check_declared (network.cpp:158-168)
        const uint32_t n = counts[k];
        if (!n) continue;
        DevBuf<uint32_t> keys, vals, dupf, flags, any;
        CKP(keys.alloc(n));
        CKP(vals.alloc(n));
        CKP(dupf.alloc(n));
        CKP(flags.alloc(n));
        CKP(any.alloc(n));
        CKP(cudaMemcpyAsync(keys.p, lists[k], n * 4ull, cudaMemcpyDeviceToDevice, st));
        k_iota<<<nb(n), kT, 0, st>>>(vals.p, n);
        SortBuffers sb;
        uint32_t *ks = nullptr, *vs = nullptr;
        RCP(radix_sort_pairs(dev, keys.p, vals.p, n, 32, sb, &ks, &vs, st));
        k_dup_decl<<<nb(n), kT, 0, st>>>(ks, vs, n, dupf.p);
        k_decl_flags<<<nb(n), kT, 0, st>>>(lists[k], n, dupf.p, nodes, N, flags.p, any.p);
        std::vector<uint32_t> hit, h_ids, h_flags;
        RCP(flagged_indices(dev, any.p, n, hit));
        if (!hit.empty()) {
            RCP(d2h(dev, h_ids, lists[k], n));
            RCP(d2h(dev, h_flags, flags.p, n));
            CKP(cudaStreamSynchronize(st));
            const char* what = k ? "outputs" : "inputs";
            for (uint32_t i : hit) {
                if (h_flags[i] & 1u)
                    viol.push_back("duplicate node " + std::to_string(h_ids[i]) + " in " + what);
                if (h_flags[i] & 2u)
                    viol.push_back("unknown node " + std::to_string(h_ids[i]) + " in " + what);
            }
        }
        if (k == 0) {
            CKP(sorted_in.alloc(n));
            CKP(cudaMemcpyAsync(sorted_in.p, ks, n * 4ull, cudaMemcpyDeviceToDevice, st));
        }
    }
    if (n_in && n_out) {  // input/output overlap, in outputs order (network.cpp:172-178)
        DevBuf<uint32_t> flag;
        CKP(flag.alloc(n_out));
        k_member_flags<<<nb(n_out), kT, 0, st>>>(outs, n_out, sorted_in.p, n_in, flag.p);
        std::vector<uint32_t> ov, h_out;
        RCP(flagged_indices(dev, flag.p, n_out, ov));
        if (!ov.empty()) {
            RCP(d2h(dev, h_out, outs, n_out));
            CKP(cudaStreamSynchronize(st));
            std::string m = "input/output overlap:";
            for (size_t i = 0; i < ov.size(); ++i) m += " " + std::to_string(h_out[ov[i]]);
            viol.push_back(m);
        }
    }
    if (!E) return ASNN_OK;
    // per connection (network.cpp:180-201)
    DevBuf<uint32_t> keys, vals, dup, status, flag, valid;
    CKP(keys.alloc(E));
    CKP(vals.alloc(E));
    CKP(dup.alloc(E));
    CKP(status.alloc(E));
    CKP(flag.alloc(E));
    CKP(valid.alloc(E));
    CKP(cudaMemcpyAsync(keys.p, dst, E * 4, cudaMemcpyDeviceToDevice, st));
    k_iota<<<nb(E), kT, 0, st>>>(vals.p, E);
    SortBuffers sb;
    uint32_t *ks = nullptr, *vs = nullptr;
    RCP(radix_sort_pairs(dev, keys.p, vals.p, E, 32, sb, &ks, &vs, st));
    DevBuf<uint32_t> k2, v2;
    CKP(k2.alloc(E));
    CKP(v2.alloc(E));
    k_gather_u32<<<nb(E), kT, 0, st>>>(src, vs, E, k2.p);
    CKP(cudaMemcpyAsync(v2.p, vs, E * 4, cudaMemcpyDeviceToDevice, st));
    SortBuffers sb2;
    uint32_t *ks2 = nullptr, *vs2 = nullptr;
    RCP(radix_sort_pairs(dev, k2.p, v2.p, E, 32, sb2, &ks2, &vs2, st));
    k_dup_pairs<<<nb(E), kT, 0, st>>>(vs2, E, src, dst, dup.p);
    k_conn_status<<<nb(E), kT, 0, st>>>(src, dst, E, nodes, N, sorted_in.p, n_in, dup.p, status.p, flag.p, valid.p);
    CKP(cudaGetLastError());
    std::vector<uint32_t> bad;
    RCP(flagged_indices(dev, flag.p, E, bad));
    std::vector<uint32_t> hs, ht, hst;
    if (!bad.empty()) {
        RCP(d2h(dev, hs, src, E));
        RCP(d2h(dev, ht, dst, E));
        RCP(d2h(dev, hst, status.p, E));
        CKP(cudaStreamSynchronize(st));
        for (uint32_t j : bad) {
            const std::string a = std::to_string(hs[j]), b = std::to_string(ht[j]);
            switch (hst[j]) {
                case CS_UNKNOWN: viol.push_back("connection " + a + "->" + b + " references an unknown node"); break;
                case CS_SELF: viol.push_back("self-loop at node " + a); break;
                case CS_DUP: viol.push_back("duplicate connection " + a + "->" + b); break;
                default: viol.push_back("input " + b + " has incoming connection from " + a); break;
            }
        }
    }
    // cycle over the accepted connections (network.cpp:204, find_cycle)
    DevBuf<uint32_t> vidx, tot, cs, cd;
    CKP(vidx.alloc(E));
    CKP(tot.alloc(1));
    RCP(exclusive_scan(dev, valid.p, vidx.p, E, tot.p, st));
    uint32_t nv = 0;
    CKP(cudaMemcpyAsync(&nv, tot.p, 4, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    if (!nv) return ASNN_OK;
    CKP(cs.alloc(nv));
    CKP(cd.alloc(nv));
    k_scatter_flagged<<<nb(E), kT, 0, st>>>(src, valid.p, vidx.p, E, cs.p);
    k_scatter_flagged<<<nb(E), kT, 0, st>>>(dst, valid.p, vidx.p, E, cd.p);
    bool cyclic = false;
    RCP(device_cycle_check(dev, nodes, N, cs.p, cd.p, nv, &cyclic));
    if (cyclic) {  // the reference's DFS names the cycle (on the device, error path only)
        DevBuf<uint32_t> si, di, cnt, off, t1, order, color_buf, stn, stp, path;
        CKP(si.alloc(nv));
        CKP(di.alloc(nv));
        CKP(cnt.alloc(N + 1));
        CKP(off.alloc(N + 1));
        CKP(t1.alloc(1));
        k_edge_index<<<nb(nv), kT, 0, st>>>(nodes, N, cs.p, nv, si.p);
        k_edge_index<<<nb(nv), kT, 0, st>>>(nodes, N, cd.p, nv, di.p);
        CKP(cudaMemsetAsync(cnt.p, 0, (N + 1) * 4ull, st));
        k_count_src<<<nb(nv), kT, 0, st>>>(si.p, nv, cnt.p);
        RCP(exclusive_scan(dev, cnt.p, off.p, N + 1, t1.p, st));
        // successors grouped by source, connection order kept (stable sort)
        SortBuffers sb;
        uint32_t *keys_out = nullptr, *vals_out = nullptr;
        int kb = 1;
        while (kb < 32 && (1ull << kb) < N) ++kb;
        RCP(radix_sort_pairs(dev, si.p, di.p, nv, kb, sb, &keys_out, &vals_out, st));
        CKP(color_buf.alloc((N + 3) / 4));
        CKP(cudaMemsetAsync(color_buf.p, 0, ((N + 3) / 4) * 4ull, st));
        CKP(stn.alloc(N + 1));
        CKP(stp.alloc(N + 1));
        CKP(path.alloc(N + 3));
        k_find_cycle<<<1, 32, 0, st>>>(nodes, N, off.p, vals_out, reinterpret_cast<uint8_t*>(color_buf.p), stn.p,
                                       stp.p, path.p);
        CKP(cudaGetLastError());
        uint32_t len = 0;
        CKP(cudaMemcpyAsync(&len, path.p, 4, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        std::vector<uint32_t> hp(len);
        if (len) CKP(cudaMemcpyAsync(hp.data(), path.p + 1, len * 4ull, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        std::string msg = "cycle";
        if (len) {
            msg += ":";
            for (uint32_t i = 0; i < len; ++i) msg += (i ? "->" : " ") + std::to_string(hp[i]);
        }
        viol.push_back(msg);
    }
    return ASNN_OK;
}

// A parsed, validated network resident on the device.
struct Parsed {
    DevBuf<uint32_t> nodes, inputs, outputs, src, dst;
    DevBuf<float> w;
    uint32_t N = 0, n_in = 0, n_out = 0;
    uint64_t E = 0;
};

int do_parse(asnn_dev* dev, const char* text, uint64_t len, Parsed& res, uint32_t* err_line) {
    cudaStream_t st = dev->stream;
    PhaseClock clk(st);
    if (err_line) *err_line = 0;
    asnn_timings& tm = dev->timings;
    cudaEventRecord(dev->ev0, st);
    // ---- 1. text and line starts
    DevBuf<char> d_text;
    CKP(d_text.alloc(len + 1));
    if (len) CKP(upload_host(dev, d_text.p, text, len, st));
    const uint64_t n_chunks = (len + 255) / 256;
    DevBuf<uint32_t> cnt, coff, tot;
    CKP(cnt.alloc(n_chunks + 1));
    CKP(coff.alloc(n_chunks + 1));
    CKP(tot.alloc(1));
    if (n_chunks) k_nl_count<<<nb(n_chunks), kT, 0, st>>>(d_text.p, len, cnt.p);
    RCP(exclusive_scan(dev, cnt.p, coff.p, n_chunks, tot.p, st));
    uint32_t n_nl = 0;
    CKP(cudaMemcpyAsync(&n_nl, tot.p, 4, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    const uint32_t n_lines = n_nl + 1;  // the segment after the last '\n' is a line too
    DevBuf<uint64_t> starts;
    CKP(starts.alloc(static_cast<uint64_t>(n_lines) + 1));
    const uint64_t h_first = 0, h_last = len + 1;
    CKP(cudaMemcpyAsync(starts.p, &h_first, 8, cudaMemcpyHostToDevice, st));
    CKP(cudaMemcpyAsync(starts.p + n_lines, &h_last, 8, cudaMemcpyHostToDevice, st));
    if (n_chunks) k_nl_write<<<nb(n_chunks), kT, 0, st>>>(d_text.p, len, coff.p, starts.p);
    clk.mark("text+line starts");
    // ---- 2. lines
    DevBuf<uint8_t> kind, estat, hdr;
    DevBuf<uint32_t> lsrc, ltgt, sigf, sig, keep, kidx;
    DevBuf<float> lw;
    CKP(kind.alloc(n_lines));
    CKP(estat.alloc(n_lines));
    CKP(hdr.alloc(n_lines));
    CKP(lsrc.alloc(n_lines));
    CKP(ltgt.alloc(n_lines));
    CKP(lw.alloc(n_lines));
    k_parse_lines<<<nb(n_lines), kT, 0, st>>>(d_text.p, starts.p, n_lines,
                                               LineOut{kind.p, estat.p, hdr.p, lsrc.p, ltgt.p, lw.p});
    CKP(cudaGetLastError());
    clk.mark("line parse");
    // ---- 3-4. sections and per-line errors
    CKP(sigf.alloc(n_lines));
    CKP(sig.alloc(n_lines));
    CKP(keep.alloc(n_lines));
    CKP(kidx.alloc(n_lines));
    k_sig_flags<<<nb(n_lines), kT, 0, st>>>(kind.p, n_lines, sigf.p);
    DevBuf<uint32_t> tot2;
    CKP(tot2.alloc(2));
    RCP(exclusive_scan(dev, sigf.p, sig.p, n_lines, tot2.p, st));
    DevBuf<unsigned long long> ferr;
    DevBuf<uint32_t> special;
    CKP(ferr.alloc(1));
    CKP(special.alloc(3));
    CKP(cudaMemsetAsync(ferr.p, 0xFF, 8, st));
    CKP(cudaMemsetAsync(special.p, 0xFF, 12, st));
    k_line_errors<<<nb(n_lines), kT, 0, st>>>(kind.p, estat.p, hdr.p, sig.p, n_lines, ferr.p, special.p, keep.p);
    RCP(exclusive_scan(dev, keep.p, kidx.p, n_lines, tot2.p + 1, st));
    uint32_t h_tot2[2], h_special[3];
    CKP(cudaMemcpyAsync(h_tot2, tot2.p, 8, cudaMemcpyDeviceToHost, st));
    CKP(cudaMemcpyAsync(h_special, special.p, 12, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    const uint32_t n_sig = h_tot2[0];
    const uint64_t E = h_tot2[1];
    DevBuf<uint32_t> es, et, eline;
    DevBuf<float> ew;
    CKP(es.alloc(E));
    CKP(et.alloc(E));
    CKP(ew.alloc(E));
    CKP(eline.alloc(E));
    k_compact_edges<<<nb(n_lines), kT, 0, st>>>(keep.p, kidx.p, n_lines, lsrc.p, ltgt.p, lw.p, estat.p, es.p,
                                                 et.p, ew.p, eline.p);
    CKP(cudaGetLastError());
    // duplicates: stable sort of edge indices by target, then by source
    if (E > 1) {
        DevBuf<uint32_t> keys, vals;
        CKP(keys.alloc(E));
        CKP(vals.alloc(E));
        CKP(cudaMemcpyAsync(keys.p, et.p, E * 4, cudaMemcpyDeviceToDevice, st));
        k_iota<<<nb(E), kT, 0, st>>>(vals.p, E);
        SortBuffers sb;
        uint32_t *ks = nullptr, *vs = nullptr;
        RCP(radix_sort_pairs(dev, keys.p, vals.p, E, 32, sb, &ks, &vs, st));
        DevBuf<uint32_t> k2;
        CKP(k2.alloc(E));
        k_gather_u32<<<nb(E), kT, 0, st>>>(es.p, vs, E, k2.p);
        DevBuf<uint32_t> v2;
        CKP(v2.alloc(E));
        CKP(cudaMemcpyAsync(v2.p, vs, E * 4, cudaMemcpyDeviceToDevice, st));
        SortBuffers sb2;
        uint32_t *ks2 = nullptr, *vs2 = nullptr;
        RCP(radix_sort_pairs(dev, k2.p, v2.p, E, 32, sb2, &ks2, &vs2, st));
        k_dup_edges<<<nb(E), kT, 0, st>>>(vs2, E, es.p, et.p, eline.p, ferr.p);
        CKP(cudaGetLastError());
    }
    clk.mark("sections+dups");
    // ---- 5. inputs / outputs ids
    std::vector<uint64_t> h_starts_sp(6, 0);
    DevBuf<uint32_t> ids[2];
    uint32_t n_ids[2] = {0, 0};
    unsigned long long h_bad_tok[2] = {~0ull, ~0ull};
    for (int k = 0; k < 2; ++k) {
        const uint32_t line = h_special[1 + k];
        if (line == 0xFFFFFFFFu) continue;
        uint64_t se[2];
        CKP(cudaMemcpyAsync(se, starts.p + line, 16, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        uint64_t s = se[0], e = std::min<uint64_t>(se[1] - 1, len);
        if (e > s && text[e - 1] == '\r') --e;
        const uint64_t L = e - s;
        if (!L) continue;
        DevBuf<uint32_t> f, idx, t1;
        DevBuf<unsigned int> bad;
        CKP(f.alloc(L));
        CKP(idx.alloc(L));
        CKP(t1.alloc(1));
        CKP(bad.alloc(1));
        CKP(cudaMemsetAsync(bad.p, 0xFF, 4, st));
        k_tok_flags<<<nb(L), kT, 0, st>>>(d_text.p, s, e, f.p);
        RCP(exclusive_scan(dev, f.p, idx.p, L, t1.p, st));
        uint32_t ntok = 0;
        CKP(cudaMemcpyAsync(&ntok, t1.p, 4, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        n_ids[k] = ntok ? ntok - 1 : 0;
        CKP(ids[k].alloc(n_ids[k] + 1));
        k_tok_ids<<<nb(L), kT, 0, st>>>(d_text.p, s, e, f.p, idx.p, ids[k].p, bad.p);
        unsigned int hb = 0;
        CKP(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        if (hb != 0xFFFFFFFFu) h_bad_tok[k] = hb;
    }
    clk.mark("ids");
    // ---- host side of the error decision
    unsigned long long h_ferr = 0;
    CKP(cudaMemcpyAsync(&h_ferr, ferr.p, 8, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    uint64_t best = h_ferr;  // (line << 8 | code), UINT64_MAX = none
    uint32_t best_aux = 0;
    for (int k = 0; k < 2; ++k)
        if (h_bad_tok[k] != ~0ull) {
            const uint64_t v = (static_cast<uint64_t>(h_special[1 + k]) << 8) | ERR_BAD_ID;
            if (v < best) {
                best = v;
                best_aux = static_cast<uint32_t>(h_bad_tok[k]);
            }
        }
    if (best == ~0ull && n_sig < 3) {  // io.cpp:149: no edges section reached
        std::string msg = "line " + std::to_string(n_lines) + ": truncated file";
        dev->err = msg;
        if (err_line) *err_line = n_lines;
        return ASNN_E_PARSE;
    }
    if (best != ~0ull) {
        const uint32_t line = static_cast<uint32_t>(best >> 8);
        uint64_t se[2];
        CKP(cudaMemcpyAsync(se, starts.p + line, 16, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        const std::string msg = parse_message(static_cast<uint8_t>(best & 0xFF),
                                              line_text(text, len, se[0], se[1]), best_aux);
        dev->err = "line " + std::to_string(line + 1) + ": " + msg;
        if (err_line) *err_line = line + 1;
        return ASNN_E_PARSE;
    }
    clk.mark("errors");
    // ---- 6. make_network (network.cpp:39-55): nodes = sorted unique ids
    const uint64_t n_all = n_ids[0] + n_ids[1] + 2 * E;
    DevBuf<uint32_t> all, nodes;
    CKP(all.alloc(n_all + 1));
    uint64_t o = 0;
    for (int k = 0; k < 2; ++k) {
        if (n_ids[k]) CKP(cudaMemcpyAsync(all.p + o, ids[k].p, n_ids[k] * 4ull, cudaMemcpyDeviceToDevice, st));
        o += n_ids[k];
    }
    if (E) {
        CKP(cudaMemcpyAsync(all.p + o, es.p, E * 4, cudaMemcpyDeviceToDevice, st));
        CKP(cudaMemcpyAsync(all.p + o + E, et.p, E * 4, cudaMemcpyDeviceToDevice, st));
    }
    uint32_t N = 0;
    if (n_all) {
        SortBuffers sb;
        uint32_t *ks = nullptr, *vs = nullptr;
        RCP(radix_sort_pairs(dev, all.p, nullptr, n_all, 32, sb, &ks, &vs, st));
        DevBuf<uint32_t> f, idx, t1;
        CKP(f.alloc(n_all));
        CKP(idx.alloc(n_all));
        CKP(t1.alloc(1));
        k_unique_flags<<<nb(n_all), kT, 0, st>>>(ks, n_all, f.p);
        RCP(exclusive_scan(dev, f.p, idx.p, n_all, t1.p, st));
        CKP(cudaMemcpyAsync(&N, t1.p, 4, cudaMemcpyDeviceToHost, st));
        CKP(cudaStreamSynchronize(st));
        CKP(nodes.alloc(N));
        k_scatter_flagged<<<nb(n_all), kT, 0, st>>>(ks, f.p, idx.p, n_all, nodes.p);
        CKP(cudaGetLastError());
    }
    clk.mark("make_network");
    // ---- validate (network.cpp:151-216)
    std::vector<std::string> viol;
    RCP(validate_device(dev, nodes.p, N, ids[0].p, n_ids[0], ids[1].p, n_ids[1], es.p, et.p, E, viol));
    clk.mark("validate");
    cudaEventRecord(dev->ev1, st);
    CKP(cudaStreamSynchronize(st));
    cudaEventElapsedTime(&tm.upload_ms, dev->ev0, dev->ev1);
    if (!viol.empty()) {
        std::string m = "invalid network";
        for (const auto& v : viol) m += "\n  " + v;
        dev->err = m;
        return ASNN_E_VALIDATION;
    }
    res.nodes = std::move(nodes);
    res.inputs = std::move(ids[0]);
    res.outputs = std::move(ids[1]);
    res.src = std::move(es);
    res.dst = std::move(et);
    res.w = std::move(ew);
    res.N = N;
    res.n_in = n_ids[0];
    res.n_out = n_ids[1];
    res.E = E;
    return ASNN_OK;
}

int parse_to_corpus(asnn_dev* dev, const char* text, uint64_t len, asnn_corpus** result, uint32_t* err_line) {
    *result = nullptr;
    Parsed p;
    RCP(do_parse(dev, text, len, p, err_line));
    PhaseClock clk(dev->stream);
    auto* c = new asnn_corpus;
    int rc = d2h(dev, c->nodes, p.nodes.p, p.N);
    if (!rc) rc = d2h(dev, c->inputs, p.inputs.p, p.n_in);
    if (!rc) rc = d2h(dev, c->outputs, p.outputs.p, p.n_out);
    if (!rc) rc = d2h(dev, c->src, p.src.p, p.E);
    if (!rc) rc = d2h(dev, c->dst, p.dst.p, p.E);
    if (!rc) rc = d2h(dev, c->w, p.w.p, p.E);
    const cudaError_t ce = cudaStreamSynchronize(dev->stream);
    if (!rc && ce != cudaSuccess) rc = cuda_fail(dev, ce, "parse download");
    if (rc) {
        delete c;
        return rc;
    }
    clk.mark("download");
    *result = c;
    return ASNN_OK;
}

int read_file(asnn_dev* dev, const char* path, std::vector<char>& buf) {
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        dev->err = std::string("cannot open ") + path;
        return ASNN_E_IO;
    }
    // one read of the whole file when its size is known (regular files)
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long size = std::ftell(f);
        if (size > 0) buf.reserve(static_cast<size_t>(size));
        std::rewind(f);
    }
    std::vector<char> tmp(1 << 20);
    size_t n;
    while ((n = std::fread(tmp.data(), 1, tmp.size(), f)) > 0) buf.insert(buf.end(), tmp.data(), tmp.data() + n);
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) {
        dev->err = std::string("failed reading ") + path;
        return ASNN_E_IO;
    }
    return ASNN_OK;
}

}  // namespace
}  // namespace asnn_b200

extern "C" {

int asnn_dev_parse_network(asnn_dev* dev, const char* text, uint64_t len, asnn_corpus** out, uint32_t* err_line) {
    if (!dev || !out || (!text && len)) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    const cudaError_t e = cudaSetDevice(dev->device);
    if (e != cudaSuccess) return asnn_b200::cuda_fail(dev, e, "cudaSetDevice");
    return asnn_b200::parse_to_corpus(dev, text, len, out, err_line);
}

// load -> levels: the parsed arrays stay on the device and go straight into
// compute_required / segment / flatten (no host round trip).
int asnn_dev_load_layout(asnn_dev* dev, const char* text, uint64_t len, asnn_dev_layout** out, uint32_t* err_line) {
    if (!dev || !out || (!text && len)) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    *out = nullptr;
    const cudaError_t e = cudaSetDevice(dev->device);
    if (e != cudaSuccess) return asnn_b200::cuda_fail(dev, e, "cudaSetDevice");
    asnn_b200::Parsed p;
    int rc = asnn_b200::do_parse(dev, text, len, p, err_line);
    if (rc) return rc;
    std::vector<uint32_t> ins, outs;
    rc = asnn_b200::d2h(dev, ins, p.inputs.p, p.n_in);
    if (!rc) rc = asnn_b200::d2h(dev, outs, p.outputs.p, p.n_out);
    if (rc) return rc;
    const cudaError_t ce = cudaStreamSynchronize(dev->stream);
    if (ce != cudaSuccess) return asnn_b200::cuda_fail(dev, ce, "load");
    return asnn_b200::build_device_network(dev, std::move(p.nodes), p.N, std::move(p.src), std::move(p.dst),
                                           std::move(p.w), p.E, std::move(ins), std::move(outs), out);
}

namespace {
// Network arrays of a desc on the device (nodes must be sorted and unique,
// the Network invariant make_network establishes, network.cpp:39-55).
struct DescOnDevice {
    asnn_b200::DevBuf<uint32_t> nodes, ins, outs, src, dst;
};
int upload_desc(asnn_dev* dev, const asnn_network_desc* n, DescOnDevice& d) {
    using namespace asnn_b200;
    if ((n->n_nodes && !n->nodes) || (n->n_inputs && !n->inputs) || (n->n_outputs && !n->outputs) ||
        (n->n_connections && (!n->source || !n->target)))
        return fail(dev, ASNN_E_INVALID, "null network array");
    for (uint32_t i = 1; i < n->n_nodes; ++i)
        if (n->nodes[i] <= n->nodes[i - 1])
            return fail(dev, ASNN_E_INVALID, "Network.nodes must be sorted ascending and unique");
    cudaStream_t st = dev->stream;
    CKP(d.nodes.alloc(n->n_nodes));
    CKP(d.ins.alloc(n->n_inputs));
    CKP(d.outs.alloc(n->n_outputs));
    CKP(d.src.alloc(n->n_connections));
    CKP(d.dst.alloc(n->n_connections));
    if (n->n_nodes) CKP(cudaMemcpyAsync(d.nodes.p, n->nodes, n->n_nodes * 4ull, cudaMemcpyHostToDevice, st));
    if (n->n_inputs) CKP(cudaMemcpyAsync(d.ins.p, n->inputs, n->n_inputs * 4ull, cudaMemcpyHostToDevice, st));
    if (n->n_outputs) CKP(cudaMemcpyAsync(d.outs.p, n->outputs, n->n_outputs * 4ull, cudaMemcpyHostToDevice, st));
    if (n->n_connections) {
        CKP(upload_host(dev, d.src.p, n->source, n->n_connections * 4, st));
        CKP(upload_host(dev, d.dst.p, n->target, n->n_connections * 4, st));
    }
    return ASNN_OK;
}
}  // namespace

// validate (network.cpp:151-216) of an in-memory network, on the device.
int asnn_dev_validate(asnn_dev* dev, const asnn_network_desc* net, char* report, uint64_t cap,
                      uint32_t* n_violations) {
    using namespace asnn_b200;
    if (!dev || !net || !n_violations || (cap && !report)) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    AllocStream alloc_on(dev->stream);
    CKP(cudaSetDevice(dev->device));
    DescOnDevice d;
    RCP(upload_desc(dev, net, d));
    std::vector<std::string> viol;
    RCP(validate_device(dev, d.nodes.p, net->n_nodes, d.ins.p, net->n_inputs, d.outs.p, net->n_outputs, d.src.p,
                        d.dst.p, net->n_connections, viol));
    CKP(cudaStreamSynchronize(dev->stream));
    *n_violations = static_cast<uint32_t>(viol.size());
    if (cap) {
        std::string all;
        for (size_t i = 0; i < viol.size(); ++i) all += (i ? "\n" : "") + viol[i];
        const size_t m = std::min<size_t>(all.size(), cap - 1);
        std::memcpy(report, all.data(), m);
        report[m] = 0;
    }
    return ASNN_OK;
}

// normalize (network.cpp:69-85): ids remapped to positions in nodes, on the device.
int asnn_dev_normalize(asnn_dev* dev, const asnn_network_desc* net, asnn_corpus** out) {
    using namespace asnn_b200;
    if (!dev || !net || !out) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    AllocStream alloc_on(dev->stream);
    *out = nullptr;
    CKP(cudaSetDevice(dev->device));
    DescOnDevice d;
    RCP(upload_desc(dev, net, d));
    cudaStream_t st = dev->stream;
    const uint32_t N = net->n_nodes;
    // every id must name a node (the reference dereferences node_index)
    std::vector<std::string> unused;
    DevBuf<uint32_t> flag;
    const uint64_t n_all = static_cast<uint64_t>(net->n_inputs) + net->n_outputs + 2 * net->n_connections;
    DevBuf<uint32_t> all, mapped;
    CKP(all.alloc(n_all + 1));
    CKP(mapped.alloc(n_all + 1));
    uint64_t o = 0;
    for (auto pr : {std::make_pair(d.ins.p, static_cast<uint64_t>(net->n_inputs)),
                    std::make_pair(d.outs.p, static_cast<uint64_t>(net->n_outputs)),
                    std::make_pair(d.src.p, net->n_connections), std::make_pair(d.dst.p, net->n_connections)}) {
        if (pr.second) CKP(cudaMemcpyAsync(all.p + o, pr.first, pr.second * 4, cudaMemcpyDeviceToDevice, st));
        o += pr.second;
    }
    CKP(flag.alloc(n_all + 1));
    if (n_all) {
        k_member_flags<<<nb(n_all), kT, 0, st>>>(all.p, n_all, d.nodes.p, N, flag.p);
        k_remap<<<nb(n_all), kT, 0, st>>>(d.nodes.p, N, all.p, n_all, mapped.p);
    }
    std::vector<uint32_t> known, m;
    RCP(d2h(dev, known, flag.p, n_all));
    RCP(d2h(dev, m, mapped.p, n_all));
    CKP(cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < n_all; ++i)
        if (!known[i]) return fail(dev, ASNN_E_INVALID, "normalize: an id names no node");
    auto* c = new asnn_corpus;
    c->nodes.resize(N);
    for (uint32_t i = 0; i < N; ++i) c->nodes[i] = i;
    uint64_t q = 0;
    c->inputs.assign(m.begin() + q, m.begin() + q + net->n_inputs);
    q += net->n_inputs;
    c->outputs.assign(m.begin() + q, m.begin() + q + net->n_outputs);
    q += net->n_outputs;
    c->src.assign(m.begin() + q, m.begin() + q + net->n_connections);
    q += net->n_connections;
    c->dst.assign(m.begin() + q, m.begin() + q + net->n_connections);
    c->w.assign(net->weight, net->weight + net->n_connections);
    *out = c;
    return ASNN_OK;
}

int asnn_dev_parse_weights(asnn_dev* dev, const char* buf, const uint64_t* off, uint64_t n, float* out,
                           uint8_t* status) {
    using namespace asnn_b200;
    if (!dev || (n && (!buf || !off || !out || !status))) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    if (!n) return ASNN_OK;
    CKP(cudaSetDevice(dev->device));
    cudaStream_t st = dev->stream;
    const uint64_t bytes = off[n];
    DevBuf<char> d_buf;
    DevBuf<uint64_t> d_off;
    DevBuf<float> d_out;
    DevBuf<uint8_t> d_st;
    CKP(d_buf.alloc(bytes + 1));
    CKP(d_off.alloc(n + 1));
    CKP(d_out.alloc(n));
    CKP(d_st.alloc(n));
    if (bytes) CKP(cudaMemcpyAsync(d_buf.p, buf, bytes, cudaMemcpyHostToDevice, st));
    CKP(cudaMemcpyAsync(d_off.p, off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
    k_parse_weights<<<nb(n), kT, 0, st>>>(d_buf.p, d_off.p, n, d_out.p, d_st.p);
    CKP(cudaGetLastError());
    CKP(cudaMemcpyAsync(out, d_out.p, n * 4, cudaMemcpyDeviceToHost, st));
    CKP(cudaMemcpyAsync(status, d_st.p, n, cudaMemcpyDeviceToHost, st));
    CKP(cudaStreamSynchronize(st));
    return ASNN_OK;
}

int asnn_dev_read_network(asnn_dev* dev, const char* path, asnn_corpus** out, uint32_t* err_line) {
    if (!dev || !path || !out) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    asnn_b200::AllocStream alloc_on(dev->stream);
    std::vector<char> buf;
    const int rc = asnn_b200::read_file(dev, path, buf);
    if (rc) return rc;
    const cudaError_t e = cudaSetDevice(dev->device);
    if (e != cudaSuccess) return asnn_b200::cuda_fail(dev, e, "cudaSetDevice");
    return asnn_b200::parse_to_corpus(dev, buf.data(), buf.size(), out, err_line);
}

}  // extern "C"
