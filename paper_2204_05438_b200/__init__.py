"""paper_2204_05438_b200 -- B200-native mesh -> polygons path of the terminal-edge
region mesher (arXiv 2204.05438), a drop-in for the reference `termesh`
package's label / traversal / reparation phases.

Every phase runs as hand-written sm_100a CUDA behind the C ABI in
include/termesh_b200.h (libtermesh_b200.so, built in-tree by
`python -m paper_2204_05438_b200.build`).  There is no CPU fallback.
"""

from .backend import GPU, SEQUENTIAL, Backend, parallel
from .errors import CapacityError, ParseError, StructuralError, TermeshError, ValidationError
from .io_formats import (TriangleFileSet, array_hash, canonicalize, generate_anisotropic_delaunay,
                         generate_clustered_delaunay, generate_random_delaunay, read_polymesh, read_triangulation,
                         triangulate_points, write_polymesh, write_triangulation)
from .labeling import EdgeLabels, label_all, label_frontiers, label_max, label_seeds
from .mesh_core import (BORDER, Triangulation, ValidationReport, compute_trivertex, edge_endpoints,
                        next_halfedge, prev_halfedge, signed_areas, squared_length, twin, validate)
from .pipeline import PhaseStats, PipelineConfig, RandomInput, bench, execute, load_input, run_pipeline
from .reparation import repair_all
from .traversal import (PolygonMesh, boundary_edge_count, build_polygon_mesh, enclosed_signed_areas,
                        extra_vertex_visits, repeated_vertex_flags, tip_flags, unique_vertices)

__version__ = "0.1.0"
