// Share, seed and plaintext files of the reference (include/irismpc/io.hpp:28-60,
// src/io.cpp): the byte formats are identical, so files written by the
// reference's `irismpc share` dealer load here and vice versa.  Host code only;
// the streaming DB load that feeds these payloads into HBM is
// irismpc_gpu_load_db_files (api.cu).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/irismpc_gpu.h"

namespace {

uint64_t get_uint(const uint8_t* p, unsigned bytes) {
  uint64_t v = 0;
  for (unsigned i = 0; i < bytes; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}
void put_uint(std::vector<uint8_t>& b, uint64_t v, unsigned bytes) {
  for (unsigned i = 0; i < bytes; ++i) b.push_back((uint8_t)(v >> (8 * i)));
}

// code_bits / mask_bits (shares.hpp:37-46)
unsigned code_bits(uint32_t v) { return v == IRISMPC_GPU_VARIANT_NO_LIFT ? 32 : 16; }
unsigned mask_bits(uint32_t v) {
  return v == IRISMPC_GPU_VARIANT_PLAIN_MASK ? 0 : (v == IRISMPC_GPU_VARIANT_MPC_LIFT ? 16 : 32);
}

long long file_size(FILE* f) {
  if (std::fseek(f, 0, SEEK_END) != 0) return -1;
  const long long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  return n;
}

int write_all(const char* path, const std::vector<uint8_t>& head, const uint8_t* body, size_t len) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return IRISMPC_GPU_ERR_CONFIG;  // "cannot open for writing"
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  if (ok && len) ok = std::fwrite(body, 1, len, f) == len;
  ok = (std::fclose(f) == 0) && ok;
  return ok ? 0 : IRISMPC_GPU_ERR_CONFIG;  // "short write"
}

}  // namespace

extern "C" {

// read_share_file (io.cpp:125-146), header and size checks only
int irismpc_gpu_read_share_header(const char* path, irismpc_gpu_share_header* out) {
  if (!path || !out) return IRISMPC_GPU_ERR_CONFIG;
  FILE* f = std::fopen(path, "rb");
  if (!f) return IRISMPC_GPU_ERR_CONFIG;  // "cannot open"
  uint8_t b[24];
  const long long n = file_size(f);
  const bool got = n >= 24 && std::fread(b, 1, 24, f) == 24;
  std::fclose(f);
  if (!got || std::memcmp(b, "IRS1", 4) != 0) return IRISMPC_GPU_ERR_CONFIG;  // "not an IRS1 file"
  if (b[4] != 1) return IRISMPC_GPU_ERR_CONFIG;                                // "unsupported IRS1 version"
  irismpc_gpu_share_header h;
  h.backend = b[5];
  h.variant = b[6];
  h.party = b[7];
  h.l = (uint32_t)get_uint(b + 12, 4);
  h.s = get_uint(b + 16, 8);
  if (h.variant > IRISMPC_GPU_VARIANT_NO_LIFT || h.backend > 1) return IRISMPC_GPU_ERR_CONFIG;
  if (b[8] != code_bits(h.variant) || b[9] != mask_bits(h.variant))
    return IRISMPC_GPU_ERR_CONFIG;  // "IRS1 width fields inconsistent with variant"
  const size_t rec = irismpc_gpu_record_bytes(h.backend, h.variant, h.l);
  if ((unsigned long long)n != 24ull + h.s * rec) return IRISMPC_GPU_ERR_CONFIG;  // "IRS1 payload size mismatch"
  *out = h;
  return 0;
}

// write_share_file (io.cpp:109-123)
int irismpc_gpu_write_share_file(const char* path, const irismpc_gpu_share_header* h, const uint8_t* payload,
                                 size_t len) {
  if (!path || !h || h->variant > IRISMPC_GPU_VARIANT_NO_LIFT || h->backend > 1) return IRISMPC_GPU_ERR_CONFIG;
  std::vector<uint8_t> head = {'I', 'R', 'S', '1', 1, (uint8_t)h->backend, (uint8_t)h->variant,
                               (uint8_t)h->party, (uint8_t)code_bits(h->variant), (uint8_t)mask_bits(h->variant)};
  put_uint(head, 0, 2);
  put_uint(head, h->l, 4);
  put_uint(head, h->s, 8);
  return write_all(path, head, payload, len);
}

// read_seed_file (io.cpp:157-170) for parties 1..3, cross-checked
int irismpc_gpu_read_seed_files(const char* const paths[3], uint8_t seeds_out[48]) {
  if (!paths || !seeds_out) return IRISMPC_GPU_ERR_CONFIG;
  uint8_t own[3][16], prev[3][16];
  for (int p = 0; p < 3; ++p) {
    FILE* f = paths[p] ? std::fopen(paths[p], "rb") : nullptr;
    if (!f) return IRISMPC_GPU_ERR_CONFIG;
    uint8_t b[39];
    const size_t got = std::fread(b, 1, sizeof(b), f);
    std::fclose(f);
    if (got != 38 || std::memcmp(b, "IRSD", 4) != 0 || b[4] != 1) return IRISMPC_GPU_ERR_CONFIG;  // "not an IRSD file"
    if (b[5] != p + 1) return IRISMPC_GPU_ERR_CONFIG;  // "seed file belongs to another party"
    std::memcpy(own[p], b + 6, 16);
    std::memcpy(prev[p], b + 22, 16);
  }
  // party p holds (seed_p, seed_{p-1}) (rep3.hpp:124-127)
  for (int p = 0; p < 3; ++p)
    if (std::memcmp(prev[p], own[(p + 2) % 3], 16) != 0) return IRISMPC_GPU_ERR_CONFIG;
  for (int p = 0; p < 3; ++p) std::memcpy(seeds_out + 16 * p, own[p], 16);
  return 0;
}

// write_seed_file (io.cpp:148-155)
int irismpc_gpu_write_seed_file(const char* path, uint32_t party, const uint8_t own[16], const uint8_t prev[16]) {
  if (!path || !own || !prev) return IRISMPC_GPU_ERR_CONFIG;
  std::vector<uint8_t> head = {'I', 'R', 'S', 'D', 1, (uint8_t)party};
  head.insert(head.end(), own, own + 16);
  head.insert(head.end(), prev, prev + 16);
  return write_all(path, head, nullptr, 0);
}

// read_iris_db (io.cpp:90-107): header
int irismpc_gpu_read_iris_db_header(const char* path, uint32_t* l_out, uint64_t* s_out) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) return IRISMPC_GPU_ERR_CONFIG;
  uint8_t b[18];
  const long long n = file_size(f);
  const bool got = n >= 18 && std::fread(b, 1, 18, f) == 18;
  std::fclose(f);
  if (!got || std::memcmp(b, "IRMP", 4) != 0) return IRISMPC_GPU_ERR_CONFIG;  // "not an IRMP file"
  if (get_uint(b + 4, 2) != 1) return IRISMPC_GPU_ERR_CONFIG;                 // "unsupported IRMP version"
  const uint32_t l = (uint32_t)get_uint(b + 6, 4);
  const uint64_t s = get_uint(b + 10, 8);
  if ((unsigned long long)n != 18ull + 2ull * s * (l / 8)) return IRISMPC_GPU_ERR_CONFIG;  // "IRMP size mismatch"
  if (l_out) *l_out = l;
  if (s_out) *s_out = s;
  return 0;
}

// read_iris_db (io.cpp:90-107): rows -> LSB-first words
int irismpc_gpu_read_iris_db(const char* path, uint64_t* codes_out, uint64_t* masks_out, uint64_t rows_cap) {
  uint32_t l = 0;
  uint64_t s = 0;
  int rc = irismpc_gpu_read_iris_db_header(path, &l, &s);
  if (rc) return rc;
  if (s > rows_cap || !codes_out || !masks_out) return IRISMPC_GPU_ERR_CONFIG;
  FILE* f = std::fopen(path, "rb");
  if (!f) return IRISMPC_GPU_ERR_CONFIG;
  const uint64_t row = l / 8, wl = (l + 63) / 64;
  std::vector<uint8_t> buf(row);
  std::fseek(f, 18, SEEK_SET);
  for (int kind = 0; kind < 2 && rc == 0; ++kind) {
    uint64_t* dst = kind == 0 ? codes_out : masks_out;
    for (uint64_t r = 0; r < s; ++r) {
      if (row && std::fread(buf.data(), 1, row, f) != row) {
        rc = IRISMPC_GPU_ERR_CONFIG;
        break;
      }
      uint64_t* w = dst + r * wl;
      std::memset(w, 0, wl * 8);
      for (uint64_t i = 0; i < row; ++i) w[i / 8] |= (uint64_t)buf[i] << (8 * (i % 8));
    }
  }
  std::fclose(f);
  return rc;
}

// write_iris_db (io.cpp:74-88)
int irismpc_gpu_write_iris_db(const char* path, uint32_t l, uint64_t s, const uint64_t* codes,
                              const uint64_t* masks) {
  if (!path || l % 8 != 0) return IRISMPC_GPU_ERR_CONFIG;  // "db length must be a multiple of 8"
  std::vector<uint8_t> buf = {'I', 'R', 'M', 'P'};
  put_uint(buf, 1, 2);
  put_uint(buf, l, 4);
  put_uint(buf, s, 8);
  const uint64_t row = l / 8, wl = (l + 63) / 64;
  buf.reserve(18 + 2 * s * row);
  for (int kind = 0; kind < 2; ++kind) {
    const uint64_t* src = kind == 0 ? codes : masks;
    for (uint64_t r = 0; r < s; ++r)
      for (uint64_t i = 0; i < row; ++i) buf.push_back((uint8_t)(src[r * wl + i / 8] >> (8 * (i % 8))));
  }
  return write_all(path, buf, nullptr, 0);
}

}  // extern "C"
