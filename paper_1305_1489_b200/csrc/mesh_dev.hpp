// GPU mesh expansion and skeleton pattern (mesh_dev.cu). Stream-ordered;
// both synchronise the stream once at the end to report mesh errors.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hdgb {

// nfc of a valid expansion: (4 nelt + ndir + nneu) / 2 (mesh.cpp:136-137).
int expanded_face_count(int nelt, int ndir, int nneu);

// Device twin of expand_mesh (host_mesh.cpp). Layouts as HostMesh: coords
// nver x 3, elements nelt x 4, dir/neu rows x 3, faces nfc x 3, facebyele
// nelt x 4, all column-major. Throws MeshError / CudaError.
void expand_device(cudaStream_t s, int nver, const double* coords, int nelt, const int* elements, int ndir,
                   const int* dir, int nneu, const int* neu, int* faces, uint8_t* facetype, int* facebyele);

// Device twin of build_pattern_raw: facebase (nfc + 1), nbr (nfc x 8, row-major,
// -1 padded), slot (nelt x 16). Returns maxnbr.
int pattern_device(cudaStream_t s, int nelt, int nfc, const int* facebyele, int64_t* facebase, int* nbr,
                   uint8_t* slot);

}  // namespace hdgb
