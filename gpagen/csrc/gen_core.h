/*
 * gen_core.h -- seeded synthetic PC-sample stream generator (input generation only).
 *
 * Holds none of GPA's arithmetic: it only draws records.  Compiled twice from this one
 * header -- into the host entry (used to feed the CPU oracle) and into a CUDA kernel
 * (used to fill HBM for the GPU path) -- so both sides see byte-identical records.
 * Record k is a pure function of (seed, k, tables): any shard [k0, k1) can be produced
 * independently and sharding never changes the stream.
 *
 * Record layout (8 bytes, little endian): u32 pc | u16 count | u8 reason | u8 flags.
 */
#ifndef GPAGEN_GEN_CORE_H
#define GPAGEN_GEN_CORE_H
#include <stdint.h>

#if defined(__CUDACC__)
#define GG_HD __host__ __device__ __forceinline__
#else
#define GG_HD static inline
#endif

typedef struct {
  uint64_t seed;
  uint32_t n_instr;       /* alias table size over PCs */
  uint32_t n_slots;       /* 2 * R: slot s -> class s / R, reason s % R */
  uint32_t n_reasons;     /* R */
  uint32_t count_max;     /* 1: every record has count 1; else count in [1, count_max] */
  uint32_t invalid_ppm;   /* injected malformed records per million */
  uint32_t pc_offset;     /* added to every drawn pc (for multi-kernel streams) */
  const uint32_t *pc_thresh;   /* [n_instr] */
  const uint32_t *pc_alias;    /* [n_instr] */
  const uint8_t  *pc_profile;  /* [n_instr] profile index */
  const uint32_t *slot_thresh; /* [n_profiles * n_slots] */
  const uint32_t *slot_alias;  /* [n_profiles * n_slots] */
} gg_stream_params;

GG_HD uint64_t gg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

GG_HD uint32_t gg_alias_draw(uint64_t z, uint32_t n, const uint32_t *thresh,
                             const uint32_t *alias) {
  uint32_t col = (uint32_t)(((z & 0xffffffffull) * (uint64_t)n) >> 32);
  uint32_t u = (uint32_t)(z >> 32);
  return u < thresh[col] ? col : alias[col];
}

/* returns the 8-byte record as a u64 (pc in the low 32 bits) */
GG_HD uint64_t gg_record(const gg_stream_params *p, uint64_t k) {
  uint64_t x = p->seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
  uint64_t z1 = gg_mix64(x);
  uint64_t z2 = gg_mix64(x ^ 0xD1B54A32D192ED03ull);
  uint32_t pc = gg_alias_draw(z1, p->n_instr, p->pc_thresh, p->pc_alias);
  uint32_t prof = p->pc_profile[pc];
  uint32_t slot = gg_alias_draw(z2, p->n_slots, p->slot_thresh + (uint64_t)prof * p->n_slots,
                                p->slot_alias + (uint64_t)prof * p->n_slots);
  uint32_t cls = slot / p->n_reasons, reason = slot % p->n_reasons;
  uint32_t count = 1u, flags = cls;
  if (p->count_max > 1u || p->invalid_ppm) {
    uint64_t z3 = gg_mix64(x ^ 0x8CB92BA72F3D8DD7ull);
    if (p->count_max > 1u) count = 1u + (uint32_t)((z3 & 0xffffffffull) % p->count_max);
    if (p->invalid_ppm && (uint32_t)((z3 >> 32) % 1000000ull) < p->invalid_ppm) {
      switch ((uint32_t)(z3 >> 56) & 3u) {
        case 0: pc = p->n_instr + (uint32_t)(z3 >> 40 & 0xffu); break;   /* pc out of range */
        case 1: reason = p->n_reasons + (uint32_t)(z3 >> 48 & 3u); break; /* bad reason */
        case 2: flags |= 2u; break;                                       /* unknown flag */
        default: flags = 1u; reason = 0u; break;                          /* LAT without reason */
      }
    }
  }
  pc += p->pc_offset;
  return (uint64_t)pc | ((uint64_t)(count & 0xffffu) << 32) | ((uint64_t)(reason & 0xffu) << 48) |
         ((uint64_t)(flags & 0xffu) << 56);
}

#endif
