"""B200-native PTSBE engine behind the reference's (``trajsim``) Python API.

Host side (Python, bit-exact with the reference): circuit and noise-model
registration (``circuit``, ``noise``), pre-trajectory sampling strategies
(``presample``), seeding, datasets (``execute``).  Device side: the batched
execution hot path -- fused gate/Kraus passes, Kraus renormalisation and bulk
shot sampling -- in hand-written sm_100a kernels (``csrc/``, built into
``libptsbe.so``) driven through a C ABI (``include/ptsbe.h``).

Same export list as ``pkg/src/trajsim/__init__.py:15-86`` minus the CPU
density-matrix oracle and the conventional Algorithm-1 simulator, which are
out of scope.  The conventional Algorithm-1
simulator (``trajectory``) runs on the device engine too.
"""

from .circuit import (
    GateOp,
    NoiseModel,
    NoiseRule,
    NoiseSite,
    NoisyCircuit,
    attach_noise,
    builtin_gate_matrix,
    circuit_hash,
    gate_op,
    make_circuit,
    matrix_op,
    noise_model_hash,
    parse_circuit,
    parse_noise_model,
    serialize_circuit,
    serialize_noise_model,
)
from .errors import AnnihilatedStateError, CircuitSyntaxError, ExecutionError, TrajsimError, ValidationError
from .noise import KrausChannel, UnitaryMixture, builtin_channel, detect_unitary_mixture, validate_cptp
from .presample import (
    PresampleConfig,
    SiteFilter,
    TrajectorySpec,
    canonical_selections,
    compatible,
    enumerate_cutoff,
    joint_probability,
    presample_band,
    presample_probabilistic,
    presample_probabilistic_iter,
    reallocate_proportional,
    site_outcome_probs,
    unique_kraus,
)
from .trajectory import DENSE_ENSEMBLE_LIMIT, RealizedTrajectory, select_index
from .version import __version__


def __getattr__(name):
    # device-backed modules load libptsbe.so lazily, so host-only use (parsing,
    # PTS) works on machines without the CUDA build
    import importlib
    lazy = {
        "Dataset": "execute", "ShotRecord": "execute", "format_records": "execute", "execute_all": "execute", "execute_naive": "execute",
        "execute_trajectory": "execute", "manifest_core": "execute", "mix_seed": "execute",
        "prepare_state": "execute", "stream_rng": "execute", "throughput_report": "execute",
        "unique_fraction": "execute", "run_specs": "execute", "presample_and_execute": "execute", "dataset_from_output": "execute",
        "execute_all_distributed": "distributed",
        "ComplexState": "statevector", "ShotBatch": "statevector", "apply_gate": "statevector",
        "apply_kraus_normalized": "statevector", "apply_matrix": "statevector", "init_zero": "statevector",
        "kraus_outcome_probability": "statevector", "sample_shots": "statevector",
        "Engine": "engine", "compile_circuit": "program", "write_throughput_csv": "execute",
        "run_trajectory": "trajectory", "sample_conventional": "trajectory",
    }
    if name in lazy:
        mod = importlib.import_module(f".{lazy[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
