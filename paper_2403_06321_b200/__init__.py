"""B200-native Vertex Block Descent (arXiv 2403.06321) hot path.

Drop-in for the reference ``vbdsim`` solver API on the per-colour Gauss-Seidel
vertex sweep for Stable Neo-Hookean tets: hand-written sm_100a CUDA kernels in
``libvbd_b200.so`` behind the C ABI of ``include/vbd_b200.h``.
"""

from .backend import NAME as BACKEND_NAME
from .context import Beam, DeviceContext
from .errors import DegenerateTet, EmptyDescentRange, IndexOutOfRange, NonFiniteState, SchemaError, VbdError
from .harness import (CONVERGENCE_HEADER, METRICS_HEADER, ObjectConfig, OutputConfig, SceneConfig, export_frame,
                      load_frame, parse_scene, run_convergence, run_simulation, scene_build, serialize_scene)
from .materials import MaterialParams
from .mesh import (ColorPartition, SpringNet, TetMesh, VertexAdjacency, build_spring_net,
                   build_tet_mesh, generate_beam, generate_chain, generate_cube, greedy_color,
                   incidence, incidence_from_elements, load_node_ele)
from .solver import (ContactParams, SimState, SolverParams, accelerate, chebyshev_omega,
                     color_pass, device_context, energy, inertia_target, initialize, local_solve,
                     make_state, max_penetration, metrics, step)
from .system import (Body, ConstraintArrays, FixedConstraint, SubspaceConstraint, System,
                     WorldBoxConstraint, build_system, compile_constraints)

from . import baselines  # noqa: E402

__version__ = "0.1.0"


def backend_name() -> str:
    return BACKEND_NAME


__all__ = [n for n in dir() if not n.startswith("_")]
