"""mixgraph: the Python package the reference declares (`proj/CMakeLists.txt:47-74`,
module `mixgraph._core`), served by the B200 renderer's pybind11 binding over its C++ API.

Everything in `_core` mirrors the C++ names (Graph, to_flat, compute_render_data, ProcessorSet,
render, ...). `render_grafx` is the paper's one-call form: parameters in
ORIGINAL node order, keyed by type (NodeType, name or code), sources [K][B][2][L].
"""
from ._core import *  # noqa: F401,F403
from ._core import (NodeType, ProcessorConfig, ProcessorSet, ScheduleOptions, Strategy,  # noqa: F401
                    compute_render_data, render, to_flat)


def render_grafx(sources, processors, parameters, render_data, keep_intermediates=False):
    """render(render_data, processors, render_data.reorder_params(parameters), sources)."""
    return render(render_data, processors, render_data.reorder_params(dict(parameters)), sources, keep_intermediates)
