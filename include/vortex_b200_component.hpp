// vortex_b200_component.hpp — header-only C++ adapter: the B200 retrieval stage as the
// reference's operator type.
//
// Reference contract (proj/include/vortex/runtime.hpp):
//   using ComponentFn = std::function<std::vector<Payload>(const std::vector<Payload>&)>;  // :179
//   Runtime::register_component(model_id, fn)                                               // :202-211
//   Runtime::complete_batch calls fn with the FIFO batch; outputs[i] <-> inputs[i],
//   and there must be at least as many outputs as inputs (:656-672, :665)
//   Payload = std::shared_ptr<const std::vector<uint8_t>>                                    // common.hpp:84-85
//   errors: vortex::error(errc, msg) (common.hpp:70-80)
//
// make_search_component(h, k) returns exactly that callable.  It decodes each payload
// (wire format below; identical to paper_2511_02062_b200/component.py), makes ONE fused
// GPU call for the whole batch (vx_search_rescore, or vx_search when the queries carry no
// tokens), and encodes one result payload per input, in input order.  Malformed input
// throws vortex::error(errc::bad_config, ...) when the reference headers are in the
// translation unit (else vortex_b200::error); a GPU failure throws with vx_last_error().
//
// Wire format (little endian):
//   query  : "VXQ1" u16 version=1 u16 dtype=0(f32) u32 dim u32 nq u32 tok_dim u32 0
//            f32[dim] f32[nq*tok_dim]
//   result : "VXR1" u16 version=1 u16 flags(bit0: maxsim valid) u32 k u32 0
//            k x { i64 id, f32 ip_score, f32 maxsim_score }
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vortex_b200.h"

#if __has_include("vortex/common.hpp")
#include "vortex/common.hpp"
#define VORTEX_B200_HAVE_REFERENCE_ERRORS 1
#endif

namespace vortex_b200 {

using Bytes = std::vector<std::uint8_t>;
using Payload = std::shared_ptr<const Bytes>;
using ComponentFn = std::function<std::vector<Payload>(const std::vector<Payload>&)>;

struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void bad_config(const std::string& what) {
#ifdef VORTEX_B200_HAVE_REFERENCE_ERRORS
  vortex::fail(vortex::errc::bad_config, what);
#else
  throw error("BadConfig: " + what);
#endif
}

[[noreturn]] inline void gpu_failure(const char* call, vx_status s) {
  std::string what = std::string(call) + " -> status " + std::to_string((int)s) + ": " +
                     vx_last_error();
#ifdef VORTEX_B200_HAVE_REFERENCE_ERRORS
  // The reference has no device errc; a failed stage execution is an unschedulable stage.
  vortex::fail(vortex::errc::unschedulable, what);
#else
  throw error(what);
#endif
}

struct QueryView {
  const float* q = nullptr;
  const float* tok = nullptr;
  std::uint32_t dim = 0, nq = 0, tok_dim = 0;
};

constexpr std::size_t kQueryHeader = 24, kResultHeader = 16;

inline Payload encode_query(const float* q, std::uint32_t dim, const float* tok = nullptr,
                            std::uint32_t nq = 0, std::uint32_t tok_dim = 0) {
  Bytes b(kQueryHeader + 4ull * (dim + (std::size_t)nq * tok_dim));
  std::uint16_t ver = 1, dt = 0;
  std::uint32_t z = 0;
  std::memcpy(b.data(), "VXQ1", 4);
  std::memcpy(b.data() + 4, &ver, 2);
  std::memcpy(b.data() + 6, &dt, 2);
  std::memcpy(b.data() + 8, &dim, 4);
  std::memcpy(b.data() + 12, &nq, 4);
  std::memcpy(b.data() + 16, &tok_dim, 4);
  std::memcpy(b.data() + 20, &z, 4);
  std::memcpy(b.data() + kQueryHeader, q, 4ull * dim);
  if (nq) std::memcpy(b.data() + kQueryHeader + 4ull * dim, tok, 4ull * nq * tok_dim);
  return std::make_shared<const Bytes>(std::move(b));
}

inline QueryView decode_query(const Payload& p) {
  if (!p || p->size() < kQueryHeader) bad_config("query payload too short");
  const std::uint8_t* d = p->data();
  std::uint16_t ver, dt;
  QueryView v;
  std::memcpy(&ver, d + 4, 2);
  std::memcpy(&dt, d + 6, 2);
  std::memcpy(&v.dim, d + 8, 4);
  std::memcpy(&v.nq, d + 12, 4);
  std::memcpy(&v.tok_dim, d + 16, 4);
  if (std::memcmp(d, "VXQ1", 4) != 0 || ver != 1 || dt != 0) bad_config("query payload header");
  const std::size_t need = kQueryHeader + 4ull * (v.dim + (std::size_t)v.nq * v.tok_dim);
  if (p->size() != need) bad_config("query payload size " + std::to_string(p->size()));
  v.q = reinterpret_cast<const float*>(d + kQueryHeader);
  v.tok = v.nq ? reinterpret_cast<const float*>(d + kQueryHeader + 4ull * v.dim) : nullptr;
  return v;
}

inline Payload encode_result(const std::int64_t* ids, const float* ip, const float* ms,
                             std::uint32_t k) {
  Bytes b(kResultHeader + 16ull * k);
  std::uint16_t ver = 1, flags = ms ? 1 : 0;
  std::uint32_t z = 0;
  std::memcpy(b.data(), "VXR1", 4);
  std::memcpy(b.data() + 4, &ver, 2);
  std::memcpy(b.data() + 6, &flags, 2);
  std::memcpy(b.data() + 8, &k, 4);
  std::memcpy(b.data() + 12, &z, 4);
  const float nan = std::numeric_limits<float>::quiet_NaN();
  for (std::uint32_t i = 0; i < k; ++i) {
    std::uint8_t* r = b.data() + kResultHeader + 16ull * i;
    std::memcpy(r, ids + i, 8);
    std::memcpy(r + 8, ip + i, 4);
    std::memcpy(r + 12, ms ? ms + i : &nan, 4);
  }
  return std::make_shared<const Bytes>(std::move(b));
}

struct ResultRec {
  std::int64_t id;
  float ip, ms;
};

inline std::vector<ResultRec> decode_result(const Payload& p) {
  if (!p || p->size() < kResultHeader || std::memcmp(p->data(), "VXR1", 4) != 0)
    bad_config("result payload");
  std::uint32_t k;
  std::memcpy(&k, p->data() + 8, 4);
  if (p->size() != kResultHeader + 16ull * k) bad_config("result payload size");
  std::vector<ResultRec> out(k);
  for (std::uint32_t i = 0; i < k; ++i) std::memcpy(&out[i], p->data() + kResultHeader + 16ull * i, 16);
  return out;
}

// The search stage as a ComponentFn.  `h` must outlive the returned function; calls must
// come from one thread at a time (the reference runtime is single-threaded,
// proj/SPEC.md:282).  dim: the index dimension; max_batch/max_k as created.
inline ComponentFn make_search_component(vx_index* h, std::uint32_t dim, std::uint32_t k) {
  return [h, dim, k](const std::vector<Payload>& inputs) -> std::vector<Payload> {
    const std::size_t B = inputs.size();
    std::vector<Payload> out;
    if (B == 0) return out;
    std::vector<QueryView> qs;
    qs.reserve(B);
    for (const auto& p : inputs) qs.push_back(decode_query(p));
    const std::uint32_t nq = qs[0].nq, td = qs[0].tok_dim;
    // row pointers straight into the payloads: the library gathers them into its pinned
    // staging buffer, so every query is copied exactly once on its way to HBM
    std::vector<const float*> qrows(B), trows(B);
    for (std::size_t i = 0; i < B; ++i) {
      if (qs[i].dim != dim) bad_config("query dim " + std::to_string(qs[i].dim));
      if (qs[i].nq != nq || qs[i].tok_dim != td) bad_config("ragged query tokens in one batch");
      qrows[i] = qs[i].q;
      trows[i] = qs[i].tok;
    }
    std::vector<std::int64_t> ids(B * k);
    std::vector<float> ip(B * k), ms(B * k);
    vx_status s;
    if (nq) {
      s = vx_search_rescore_rows(h, qrows.data(), trows.data(), (std::int32_t)B, (std::int32_t)nq,
                                 (std::int32_t)k, ids.data(), ip.data(), ms.data());
      if (s != VX_OK) gpu_failure("vx_search_rescore_rows", s);
    } else {
      s = vx_search_rows(h, qrows.data(), (std::int32_t)B, (std::int32_t)k, ids.data(), ip.data());
      if (s != VX_OK) gpu_failure("vx_search_rows", s);
    }
    out.reserve(B);
    for (std::size_t i = 0; i < B; ++i)
      out.push_back(encode_result(ids.data() + i * k, ip.data() + i * k,
                                  nq ? ms.data() + i * k : nullptr, k));
    return out;  // out.size() == inputs.size(): runtime.hpp:665 indexes outputs[i]
  };
}

}  // namespace vortex_b200
