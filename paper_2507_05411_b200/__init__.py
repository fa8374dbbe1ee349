"""B200-native drop-in for the composer decoder training step (arxiv 2507.05411).

Public surface mirrors the reference package's names for the hot path (reference
pkg/src/composer/__init__.py): config composition, module runtime, PRNG, errors,
layers and the experiment registry — plus ``TrainEngine`` (the GPU training step).
"""

from . import errors
from .config import (
    REQUIRED,
    ComponentSchema,
    ConfigNode,
    FieldSpec,
    FunctionSpec,
    ValueKind,
    config_from_factory,
    default_config,
    parse_golden,
    parse_path,
    register_component,
    register_factory,
    serialize_golden,
    visit,
)
from .errors import *  # noqa: F401,F403
from .module import (
    PARAM_ALLOCATIONS,
    Behavior,
    InvocationContext,
    Module,
    ModuleTree,
    OutputCollection,
    RematTag,
    add_state_update,
    add_summary,
    backward_child,
    current_context,
    get_shared_state,
    init_state,
    instantiate,
    invoke,
    invoke_child,
    module_registry_digest,
    param,
    param_key,
    register_behavior,
    register_spec_function,
    value_and_grad,
)
from .prng import RngKey, child_key, generator, root_key, uniform
from . import layers  # noqa: E402  (registers every kind)
from .layers import ACTIVATION_NAMES, GateDecision, OptimizerSpec, load_balance_loss, scaled_hidden_dim
from .experiments import (
    BENCH_CONFIGS,
    EXPERIMENTS,
    build_experiment,
    experiment_names,
    register_experiment,
    synthetic_batch,
)
from .engine import TrainEngine, model_precision, set_dtype_policy
from .step import forward_loss, train_step
