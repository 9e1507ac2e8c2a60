/* dmcg_synth.h — seeded synthetic mesh sequences for the BASELINE.json
 * configs (stand-ins for the paper's third-party datasets).  Host-only C ABI
 * of libdmcg_synth.so; not part of the reference interface.  Output axes use
 * the reference MeshSequence layout (vertex-major, x[i*F + f]); `f32`
 * selects float instead of double output.  Returns 0 or 5 (bad parameter). */
#ifndef DMCG_SYNTH_H
#define DMCG_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int dmcg_synth_icosphere_size(int level, uint32_t* n, uint32_t* n_faces);
/* configs 0, 2, 4: icosphere, rotation 0.05 t about a seeded axis, radial
 * sum_{l<=lmax} a_lm Y_lm sin(2 pi f_lm t / F + phi_lm), `bones` >0 adds the
 * piecewise-linear skeletal bend of config 2. */
int dmcg_synth_sphere(int level, uint32_t F, int lmax, int bones, uint64_t seed, int f32,
                      uint32_t* faces, void* const axes[3]);
/* config 1: torus nu x nv with travelling waves + Gaussian jitter. */
int dmcg_synth_torus(uint32_t nu, uint32_t nv, double R, double r, uint32_t F, int waves,
                     double jitter, uint64_t seed, int f32, uint32_t* faces,
                     void* const axes[3]);
/* config 3: jittered nx x ny grid, height field of moving Gaussian bumps. */
int dmcg_synth_grid(uint32_t nx, uint32_t ny, uint32_t F, int bumps, uint64_t seed, int f32,
                    uint32_t* faces, void* const axes[3]);
#ifdef __cplusplus
}
#endif
#endif
