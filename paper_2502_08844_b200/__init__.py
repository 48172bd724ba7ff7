"""B200-native batched env step (drop-in for deskrl's BatchEnv hot path).

See DESIGN.md.  The public surface mirrors deskrl.envkit
(/root/reference/pkg/src/deskrl/envkit.py): EnvConfig, DynamicsParams,
BatchEnv, registered_tasks and the reference's error classes, plus the
device-resident DeviceBatchEnv.
"""

__version__ = "0.1.0"

from .envkit import (  # noqa: E402,F401
    BackendError,
    BatchEnv,
    ConfigError,
    DeviceBatchEnv,
    DynamicsParams,
    EnvConfig,
    Environment,
    InvalidInputError,
    StepResult,
    TaskSpec,
    UsageError,
    make_batch_env,
    make_env,
    registered_tasks,
    resolve_task,
)
