"""B200-native w-stacking imager (hot path of arxiv/paper_2504_00959).

uvw / visibility / weight arrays in, dirty image out, with the reference
``wstack`` package's grid, w-plane, kernel and FFT/phase conventions. All
numerics run in libwsb.so (hand-written sm_100a CUDA, include/wsb.h); this
package is the host-side mirror of the reference API.
"""

from .imager import (  # noqa: F401
    OPS_COLUMNS,
    FinalImage,
    FormatError,
    GridSpec,
    KernelSpec,
    PipelineResult,
    ComplexGrid,
    MeterError,
    RunRecord,
    SectorBatch,
    SlabRange,
    grid_all,
    grid_sector,
    slab_of,
    bucket_items_device,
    grid_slab_device,
    image,
    image_device,
    image_stream,
    image_time_chunks,
    write_dataset,
    ChunkSpec,
    last_timings,
    partition_1d,
    prepare_device,
    read_dataset,
    run_pipeline,
    unpack_grid_device,
    write_image,
)

__version__ = "0.1.0"
