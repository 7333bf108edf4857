// output.cu -- the reference's output formats on the product side:
//   dump_solution  (proj/src/downpass.cpp:108-143): raw little-endian FP64 (interleaved re/im for complex),
//                  leaf-major / point-minor, written to <bin>.tmp and renamed, then a JSON sidecar
//                  {"dtype", "leaf_len", "n_leaves", "tree_ref"} the same way;
//   mesh_to_json   (proj/src/mesh.cpp:435-463): {"dim", "nodes": [{"children", "depth", "hi", "id", "lo"}], "p", "q"}.
// Both JSON texts are byte-identical to the reference's nlohmann::json::dump(1) output (keys sorted,
// one-space indentation, shortest round-trip doubles with ".0" on integral values; the image's nlohmann
// prints integer arrays on one line), checked against the reference build in tests/test_refine.py.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx_internal.cuh"

namespace {

std::string json_double(double v) {
  // nlohmann's number_float output: the shortest representation that round-trips (%.{1..17}g), integral
  // values printed with ".0"; exponent form as printf gives it ("1e-05" -> nlohmann "1e-05").
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string indent(int n) { return std::string(size_t(n), ' '); }

void json_array(std::string& out, const std::vector<std::string>& items, int ind) {
  if (items.empty()) {
    out += "[]";
    return;
  }
  out += "[\n";
  for (size_t i = 0; i < items.size(); ++i) {
    out += indent(ind + 1) + items[i];
    out += i + 1 < items.size() ? ",\n" : "\n";
  }
  out += indent(ind) + "]";
}

void write_file_atomic(const std::string& path, const std::string& tmp, const void* data, size_t bytes) {
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw hpsctx::HpsError{HPSG_ERR_INVALID, "dump_solution: cannot write " + tmp};
  const size_t w = bytes ? std::fwrite(data, 1, bytes, f) : 0;
  std::fclose(f);
  if (w != bytes) throw hpsctx::HpsError{HPSG_ERR_INVALID, "dump_solution: short write " + tmp};
  std::rename(tmp.c_str(), path.c_str());
}

}  // namespace

extern "C" int hpsg_mesh_json(const hpsg_tree_desc* t, char* out, size_t cap, size_t* len) {
  if (!t || !len || t->n_nodes < 1) return HPSG_ERR_INVALID;
  const int nchild = t->dim == 2 ? 4 : 8;
  std::string s = "{\n \"dim\": " + std::to_string(t->dim) + ",\n \"nodes\": ";
  std::vector<std::string> nodes;
  for (int i = 0; i < t->n_nodes; ++i) {
    std::string n = "{\n";
    std::vector<std::string> ch;
    if (t->n_children[i])
      for (int c = 0; c < nchild; ++c) ch.push_back(std::to_string(t->children[8 * i + c]));
    n += indent(3) + "\"children\": [";  // this nlohmann build prints integer arrays on one line
    for (size_t k = 0; k < ch.size(); ++k) n += (k ? "," : "") + ch[k];
    n += "]";
    n += ",\n" + indent(3) + "\"depth\": " + std::to_string(t->depth[i]) + ",\n";
    std::vector<std::string> hi{json_double(t->hi[3 * i]), json_double(t->hi[3 * i + 1]), json_double(t->hi[3 * i + 2])};
    std::vector<std::string> lo{json_double(t->lo[3 * i]), json_double(t->lo[3 * i + 1]), json_double(t->lo[3 * i + 2])};
    n += indent(3) + "\"hi\": ";
    json_array(n, hi, 3);
    n += ",\n" + indent(3) + "\"id\": " + std::to_string(i) + ",\n";
    n += indent(3) + "\"lo\": ";
    json_array(n, lo, 3);
    n += "\n" + indent(2) + "}";
    nodes.push_back(std::move(n));
  }
  json_array(s, nodes, 1);
  s += ",\n \"p\": " + std::to_string(t->p) + ",\n \"q\": " + std::to_string(t->p - 2) + "\n}";
  *len = s.size();
  if (!out) return HPSG_OK;
  if (cap < s.size() + 1) return HPSG_ERR_INVALID;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return HPSG_OK;
}

extern "C" int hpsg_dump_solution(hpsg_ctx* c, const double* d_u, int is_complex, const char* json_path,
                                  const char* bin_path, const char* tree_ref) {
  if (!c || !d_u || !json_path || !bin_path) return HPSG_ERR_INVALID;
  try {
    hpsg_stats st{};
    hpsg_get_stats(c, &st);
    const long long nl = st.n_leaves;
    const int leaf_len = nl > 0 ? int(st.n_points / nl) : 0;
    const size_t bytes = size_t(st.n_points) * (is_complex ? 16 : 8);
    std::vector<char> host(bytes);
    hpsctx::ck(cudaSetDevice(c->opts.device), "device");
    hpsctx::ck(cudaMemcpyAsync(host.data(), d_u, bytes, cudaMemcpyDeviceToHost, c->st), "u D2H");
    hpsctx::ck(cudaStreamSynchronize(c->st), "dump sync");
    write_file_atomic(bin_path, std::string(bin_path) + ".tmp", host.data(), bytes);
    std::string j = "{\n \"dtype\": \"";
    j += is_complex ? "complex128" : "float64";
    j += "\",\n \"leaf_len\": " + std::to_string(leaf_len) + ",\n \"n_leaves\": " + std::to_string(nl) +
         ",\n \"tree_ref\": \"";
    for (const char* p = tree_ref ? tree_ref : ""; *p; ++p) {  // JSON string escaping (nlohmann)
      const unsigned char ch = static_cast<unsigned char>(*p);
      if (ch == '"' || ch == '\\') {
        j += '\\';
        j += char(ch);
      } else if (ch < 0x20) {
        char e[8];
        std::snprintf(e, sizeof e, "\\u%04x", ch);
        j += e;
      } else {
        j += char(ch);
      }
    }
    j += "\"\n}\n";
    write_file_atomic(json_path, std::string(json_path) + ".tmp", j.data(), j.size());
    return HPSG_OK;
  } catch (const hpsctx::HpsError& e) {
    c->err = e.msg;
    return e.code;
  } catch (const hpsctx::CudaError& e) {
    c->err = std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.e);
    return HPSG_ERR_CUDA;
  }
}
