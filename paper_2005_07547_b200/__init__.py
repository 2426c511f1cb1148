"""B200-native PSTF field cache (arXiv 2005.07547, data-parallel core).

Python mirror of the reference's ``pstf::FieldStore`` / ``FieldUpdateQueue`` API
(/root/reference/proj/core/include/pstf/field.h) over the C ABI in ``include/pstf_field.h``
(``lib/libpstf_b200.so``, hand-written sm_100a kernels).  There is no CPU implementation:
importing works anywhere, but every computing call needs the CUDA library and a B200 and
raises ``PstfError`` otherwise.
"""
from .field import (  # noqa: F401
    BLEND_LINEAR, BLEND_SQRT, KIND_FLI, KIND_LI, KIND_LO, KIND_LO_MINUS_E, MODE_ATOMIC,
    MODE_ORDERED, MODE_SEQUENTIAL, TECH_ALL, TECH_CAMERA, TECH_CONTINUATION, TECH_NEE,
    FieldStore, FieldStoreConfig, FieldUpdateQueue, PstfError, SpatioDirectionalKey,
    SNAPSHOT_DTYPE, SLOT_DTYPE, KEY_DTYPE, lib, library_path, read_snapshot, synth_generate,
    vertex_pass, vertex_pass_host, vertex_pass_cv, cv_lookup, vertex_soa, vertex_soa_from_fields,
    kernel_launch_count, red_peak,
    VERTEX_BYTES, VERTEX_F64_FIELDS, profile_enable, profile_collect, end_frame_all,
)
from .model import MODEL_ENTRY_DTYPE, MODEL_GMM, MODEL_GRID, MODEL_KDTREE, ModelStore  # noqa: F401,E402
