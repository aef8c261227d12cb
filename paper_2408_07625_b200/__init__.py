"""qvmc-b200: B200-native surrogate local-energy evaluation (arXiv 2408.07625).

Drop-in for the reference's hot path (proj/include/qvmc/{coupling,energy}.hpp):
``find_coupled_pairs`` / ``loop_over_*``, ``local_energies``,
``variational_energy`` and the fused ``surrogate_energy`` throughput path, all
computed by hand-written sm_100a kernels in ``lib/libqvmc_cuda.so`` through
the C ABI declared in ``include/qvmc_cuda.h``. The C++ drop-in for the
reference's own headers is ``lib/libqvmc_dropin.so``.
"""
from . import basis
from ._lib import QvmcLogicError, launch_count
from .coupling import (CoupledPairs, CouplingBackend, CouplingOptions, backend_name, find_coupled_pairs,
                       loop_over_batch, loop_over_terms, loop_over_trie, parse_backend)
from .energy import (EnergyReport, SampleBatch, last_stats, local_energies, normalise, surrogate_energy,
                     variational_energy)
from .hamiltonian import HamiltonianIndex, encode_strings
from .model import (AnqsModel, CounterRng, QuditLayout, SectorConstraint, fill_amplitudes, load_checkpoint,
                    sample_without_replacement)

__all__ = [
    "basis", "CounterRng", "sample_without_replacement", "QvmcLogicError", "launch_count", "CoupledPairs", "CouplingBackend", "CouplingOptions",
    "backend_name", "find_coupled_pairs", "loop_over_batch", "loop_over_terms", "loop_over_trie", "parse_backend",
    "EnergyReport", "SampleBatch", "last_stats", "local_energies", "normalise", "surrogate_energy",
    "variational_energy", "HamiltonianIndex", "encode_strings", "AnqsModel", "QuditLayout", "SectorConstraint",
    "fill_amplitudes", "load_checkpoint",
]
