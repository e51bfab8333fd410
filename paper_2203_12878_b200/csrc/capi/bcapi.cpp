// bcapi.cpp -- C ABI of the BabyCUDA front end (include/mapcheck.h, NEXT-1):
// map_infer = parse + Fig. 6 typing + MAP printing (babycuda/bcfront.cpp).
#include <cstring>
#include <string>

#include "../../../include/mapcheck.h"
#include "../babycuda/bcfront.h"

namespace {
void put(const std::string& d, char* buf, size_t cap) {
  if (!buf || !cap) return;
  const size_t n = std::min(cap - 1, d.size());
  std::memcpy(buf, d.data(), n);
  buf[n] = 0;
}
}  // namespace

extern "C" map_status map_infer(const char* src, size_t len, uint64_t data_domain, char* map_out, size_t map_cap,
                                size_t* map_len, map_typing* ty, char* diag, size_t diag_cap) {
  if (!src || !ty) return MAP_E_ARG;
  try {
    const bcf::Kernel k = bcf::parse(std::string(src, len));
    const bcf::Typing t = bcf::type_check(k);
    std::memset(ty, 0, sizeof(*ty));
    ty->typable = t.typable ? 1 : 0;
    ty->kind = (int32_t)t.kind;
    ty->line = (uint32_t)t.line;
    ty->col = (uint32_t)t.col;
    put(t.var, ty->var, sizeof(ty->var));
    put("", diag, diag_cap);
    if (!t.typable && data_domain == 0) {
      put(std::to_string(t.line) + ":" + std::to_string(t.col) + ": not typable: '" + t.var + "' (read from an array) " +
              (t.kind == bcf::TY_DATA_INDEX ? "indexes an array" : "decides control flow"),
          diag, diag_cap);
      if (map_len) *map_len = 0;
      return MAP_E_TYPE;
    }
    const std::string text = bcf::map_text(k, t.typable ? 0 : data_domain);
    if (map_len) *map_len = text.size();
    put(text, map_out, map_cap);
    return MAP_OK;
  } catch (const bcf::Error& e) {
    put(e.msg, diag, diag_cap);
    return (map_status)e.status;
  } catch (...) {
    put("internal error", diag, diag_cap);
    return MAP_E_ARG;
  }
}
