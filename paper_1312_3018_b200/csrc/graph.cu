// graph.cu -- host graphs (edge lists owned by the library), the text edge-list
// loader and the device RMAT slice generator of include/tgraph.h.  None of this
// is on the timed path: it is the load step before partitioning.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "tg_inputs.h"
#include "tgraph.h"

namespace tg {

int guard(const std::function<void()>& f);  // api.cu

struct HostGraph {
  uint64_t V = 0;
  bool weighted = false;
  std::vector<uint32_t> src, dst, w;
};

namespace {

// Parse one unsigned decimal integer; advances p.  Rejects signs ('-' gives
// "negative"), empty fields and values above `max`.
enum class Num { ok, none, negative, bad, big };
Num parse_u64(const char*& p, uint64_t max, uint64_t* out) {
  while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
  if (*p == '\0' || *p == '\n') return Num::none;
  if (*p == '-') return Num::negative;
  if (*p == '+') ++p;
  if (*p < '0' || *p > '9') return Num::bad;
  uint64_t v = 0;
  while (*p >= '0' && *p <= '9') {
    const uint64_t d = (uint64_t)(*p - '0');
    if (v > (max - d) / 10) return Num::big;
    v = v * 10 + d;
    ++p;
  }
  if (*p != '\0' && *p != '\n' && *p != ' ' && *p != '\t' && *p != '\r') return Num::bad;
  *out = v;
  return Num::ok;
}

[[noreturn]] void line_error(uint64_t line, const std::string& what) {
  fail(TG_EINVAL, "edge list line " + std::to_string(line) + ": " + what);
}

__global__ void k_rmat_slice(tgin_rmat g, uint64_t first, uint64_t n, uint64_t wseed, uint32_t* src,
                             uint32_t* dst, uint32_t* w) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t s, d;
    tgin_rmat_edge_g(&g, first + i, &s, &d);
    src[i] = s;
    dst[i] = d;
    if (w) w[i] = tgin_weight(wseed, first + i);
  }
}

}  // namespace

}  // namespace tg

using namespace tg;

extern "C" {

int tg_graph_from_edges(uint64_t V, uint64_t E, const uint32_t* src, const uint32_t* dst,
                        const uint32_t* w, tg_graph** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr, TG_EINVAL, "NULL out");
    *out = nullptr;
    TG_REQUIRE(V >= 1 && V < (1ull << 31), TG_EINVAL, "V must be in [1, 2^31)");
    TG_REQUIRE(E == 0 || (src && dst), TG_EINVAL, "NULL edge arrays");
    for (uint64_t k = 0; k < E; ++k)
      TG_REQUIRE(src[k] < V && dst[k] < V, TG_EINVAL,
                 "edge " + std::to_string(k) + ": vertex id >= V");
    auto g = std::make_unique<HostGraph>();
    g->V = V;
    g->weighted = w != nullptr;
    g->src.assign(src, src + E);
    g->dst.assign(dst, dst + E);
    if (w) g->w.assign(w, w + E);
    *out = reinterpret_cast<tg_graph*>(g.release());
  });
}

int tg_graph_load_edge_list(const char* path, int directed, int weighted, tg_graph** out) {
  return guard([&] {
    TG_REQUIRE(out != nullptr && path != nullptr, TG_EINVAL, "NULL argument");
    *out = nullptr;
    std::FILE* f = std::fopen(path, "rb");
    TG_REQUIRE(f != nullptr, TG_EIO, std::string("cannot open ") + path + ": " + std::strerror(errno));
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> hold(f, std::fclose);
    auto g = std::make_unique<HostGraph>();
    g->weighted = weighted != 0;
    uint64_t declared = 0, max_id = 0, line = 0;
    bool have_decl = false, any = false;
    std::string buf;
    char chunk[1 << 16];
    auto handle = [&](const char* s) {
      ++line;
      const char* p = s;
      while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
      if (*p == '\0' || *p == '\n') return;
      if (*p == '#') {
        const char* key = std::strstr(p, "nodes:");
        if (key) {
          const char* q = key + 6;
          uint64_t n = 0;
          if (parse_u64(q, 1ull << 31, &n) != Num::ok) line_error(line, "bad '# nodes:' header");
          TG_REQUIRE(n >= 1 && n < (1ull << 31), TG_EINVAL,
                     "edge list line " + std::to_string(line) + ": nodes must be in [1, 2^31)");
          declared = n;
          have_decl = true;
        }
        return;
      }
      uint64_t v[3] = {0, 0, 0};
      const int nf = weighted ? 3 : 2;
      for (int i = 0; i < nf; ++i) {
        const Num r = parse_u64(p, i < 2 ? (1ull << 31) - 1 : 0xFFFFFFFFull, &v[i]);
        if (r == Num::negative) line_error(line, i < 2 ? "negative vertex id" : "negative weight");
        if (r == Num::none) line_error(line, i < 2 ? "expected 'src dst'" : "missing weight");
        if (r == Num::big) line_error(line, "value out of range");
        if (r != Num::ok) line_error(line, "malformed number");
      }
      while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
      if (*p != '\0' && *p != '\n') line_error(line, "trailing characters");
      if (have_decl && (v[0] >= declared || v[1] >= declared))
        line_error(line, "vertex id >= declared node count " + std::to_string(declared));
      max_id = std::max(max_id, std::max(v[0], v[1]));
      any = true;
      g->src.push_back((uint32_t)v[0]);
      g->dst.push_back((uint32_t)v[1]);
      if (weighted) g->w.push_back((uint32_t)v[2]);
      if (!directed) {
        g->src.push_back((uint32_t)v[1]);
        g->dst.push_back((uint32_t)v[0]);
        if (weighted) g->w.push_back((uint32_t)v[2]);
      }
    };
    while (std::fgets(chunk, sizeof(chunk), f)) {
      buf += chunk;
      if (!buf.empty() && buf.back() != '\n' && !std::feof(f)) continue;  // long line
      handle(buf.c_str());
      buf.clear();
    }
    TG_REQUIRE(!std::ferror(f), TG_EIO, std::string("read error on ") + path);
    if (!buf.empty()) handle(buf.c_str());
    // a '# nodes:' header after some edges still bounds every id
    if (have_decl)
      for (size_t k = 0; k < g->src.size(); ++k)
        TG_REQUIRE(g->src[k] < declared && g->dst[k] < declared, TG_EINVAL,
                   "vertex id >= declared node count " + std::to_string(declared));
    g->V = have_decl ? declared : (any ? max_id + 1 : 0);
    TG_REQUIRE(g->V >= 1, TG_EINVAL, "empty edge list without a '# nodes: N' header");
    TG_REQUIRE(g->V < (1ull << 31), TG_ECAPACITY, "more than 2^31 - 1 vertices");
    *out = reinterpret_cast<tg_graph*>(g.release());
  });
}

int tg_graph_info(const tg_graph* gh, uint64_t* V, uint64_t* E, int* weighted) {
  return guard([&] {
    TG_REQUIRE(gh != nullptr, TG_EINVAL, "NULL graph");
    const HostGraph& g = *reinterpret_cast<const HostGraph*>(gh);
    if (V) *V = g.V;
    if (E) *E = g.src.size();
    if (weighted) *weighted = g.weighted ? 1 : 0;
  });
}

int tg_graph_edges(const tg_graph* gh, uint32_t* src, uint32_t* dst, uint32_t* w) {
  return guard([&] {
    TG_REQUIRE(gh != nullptr, TG_EINVAL, "NULL graph");
    const HostGraph& g = *reinterpret_cast<const HostGraph*>(gh);
    const size_t E = g.src.size();
    TG_REQUIRE(E == 0 || (src && dst), TG_EINVAL, "NULL output arrays");
    if (E) {
      std::memcpy(src, g.src.data(), E * 4);
      std::memcpy(dst, g.dst.data(), E * 4);
      if (w && g.weighted) std::memcpy(w, g.w.data(), E * 4);
    }
  });
}

void tg_graph_free(tg_graph* g) { delete reinterpret_cast<HostGraph*>(g); }

int tg_engine_create(const tg_graph* gh, const tg_attr* attr, tg_engine** out) {
  if (!gh || !attr) {
    return guard([&] { fail(TG_EINVAL, "NULL graph or attr"); });
  }
  const HostGraph& g = *reinterpret_cast<const HostGraph*>(gh);
  if (attr->weighted && !g.weighted)
    return guard([&] { fail(TG_EINVAL, "attr.weighted set but the graph has no weights"); });
  return tg_engine_create_edges(g.V, g.src.size(), g.src.data(), g.dst.data(),
                                g.weighted ? g.w.data() : nullptr, TG_MEM_HOST, attr, out);
}

int tg_rmat_edges(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                  int scramble, uint64_t wseed, uint64_t first, uint64_t count, uint32_t* src,
                  uint32_t* dst, uint32_t* w, int mem) {
  return guard([&] {
    TG_REQUIRE(scale >= 1 && scale <= 31, TG_EINVAL, "scale must be in [1, 31]");
    TG_REQUIRE(edge_factor >= 1, TG_EINVAL, "edge_factor must be >= 1");
    TG_REQUIRE(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0 + 1e-12, TG_EINVAL,
               "RMAT probabilities: need a, b, c >= 0 and a + b + c <= 1");
    TG_REQUIRE(mem == TG_MEM_HOST || mem == TG_MEM_DEVICE, TG_EINVAL, "bad mem kind");
    const uint64_t E = (uint64_t)edge_factor << scale;
    TG_REQUIRE(first <= E && count <= E - first, TG_EINVAL, "slice beyond the edge stream");
    if (!count) return;
    TG_REQUIRE(src && dst, TG_EINVAL, "NULL output arrays");
    const tgin_rmat g = tgin_make_rmat(scale, a, b, c, seed, scramble);
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 26);
    DevBuf<uint32_t> ds, dd, dw;
    if (mem == TG_MEM_HOST) {
      ds.alloc(chunk);
      dd.alloc(chunk);
      if (w) dw.alloc(chunk);
    }
    for (uint64_t off = 0; off < count; off += chunk) {
      const uint64_t n = std::min(chunk, count - off);
      uint32_t* s = mem == TG_MEM_HOST ? ds.get() : src + off;
      uint32_t* d = mem == TG_MEM_HOST ? dd.get() : dst + off;
      uint32_t* ww = !w ? nullptr : (mem == TG_MEM_HOST ? dw.get() : w + off);
      k_rmat_slice<<<grid_for(n, 256, 148u * 32u), 256>>>(g, first + off, n, wseed, s, d, ww);
      TG_CK(cudaGetLastError());
      if (mem == TG_MEM_HOST) {
        TG_CK(cudaMemcpy(src + off, s, n * 4, cudaMemcpyDeviceToHost));
        TG_CK(cudaMemcpy(dst + off, d, n * 4, cudaMemcpyDeviceToHost));
        if (w) TG_CK(cudaMemcpy(w + off, ww, n * 4, cudaMemcpyDeviceToHost));
      }
    }
    TG_CK(cudaDeviceSynchronize());
  });
}

}  // extern "C"
