"""B200-native StencilFFT-P (arXiv 2105.06676) periodic stencil solver.

Drop-in for the reference fftstencil library's periodic hot path
(solve_periodic / solve_periodic_vector / _cached / _implicit and the FFT /
spectrum building blocks).  The numerical path is hand-written sm_100a CUDA
in ``csrc/`` behind the C ABI ``include/fsx.h`` (``libfsx.so``); this package
is the Python host mirror of the reference interface.
"""
from .fftstencil import (  # noqa: F401
    ComplexGrid,
    CudaError,
    DiagonalSpectrum,
    Error,
    FieldGrid,
    GridShape,
    NumericError,
    SpecError,
    SpectrumCache,
    StageTimings,
    StencilKernel,
    device_check,
    device_count,
    evolve_periodic_naive,
    evolve_periodic_naive_device,
    fft,
    fold_kernels,
    get_devices,
    hadamard,
    last_stage_ms,
    multi_fft,
    multi_ifft,
    multiply_spectra,
    plan_describe,
    pow_spectrum,
    pseudo_inverse_spectrum,
    set_devices,
    solve_periodic,
    solve_periodic_batch,
    solve_periodic_cached,
    solve_periodic_batch_f32,
    solve_periodic_device,
    solve_periodic_device_f32,
    solve_periodic_f32,
    solve_periodic_implicit,
    solve_periodic_slabs,
    solve_periodic_vector,
    spectral_cut_columns,
    spectrum_from_kernel,
    step_periodic,
)
from .grid_io import (  # noqa: F401
    IoError,
    format_stage_table,
    load_grid_device,
    read_grid,
    read_grid_shape,
    run_bench,
    write_grid,
)
from . import _lib  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
