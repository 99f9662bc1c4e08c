"""drivegrid on B200: the batched multi-world, multi-agent vehicle step of
SceneFactory (arXiv 2605.08528) as one fused sm_100a kernel per env step,
behind the reference package's own ``Engine`` / ``EnvHandle`` API.

Host-init modules (``params``, ``scenes``, ``friction``, ``config``,
``tables``) are plain numpy; ``engine`` and ``bindings`` drive the CUDA library
``libdrivegrid_b200.so`` through its C ABI (``include/drivegrid_b200.h``).
"""

from .params import (BicycleParams, ObsConfig, RewardConfig, SimConfig,  # noqa: F401
                     VehicleParams)

__version__ = "0.1.0"


def __getattr__(name):
    # the device engine pulls in torch + the native library; import lazily so
    # the host-init layer stays importable on machines without CUDA
    if name in ("Engine", "StepOutput"):
        from . import engine
        return getattr(engine, name)
    if name in ("EnvHandle", "make_env"):
        from . import bindings
        return getattr(bindings, name)
    if name in ("RootConfig", "build_engine", "parse_config"):
        from . import config
        return getattr(config, name)
    raise AttributeError(name)
