"""B200-native encoding hot path of Shallow Tree Matching Pursuit (arXiv 1412.0680).

Public names mirror the reference package ``stmp`` (pkg/src/stmp/__init__.py:51-63)
for the pursuit layer; tree learning stays with the reference's CPU code.
"""

__version__ = "0.1.0"

from .errors import FormatError, StaleTreeError
from .pursuit import (
    Dictionary,
    EncodeResult,
    ExactSelector,
    GpuDictionary,
    GpuTree,
    ScoreCounter,
    SearchParams,
    SparseCode,
    TreeSelector,
    encode,
    encode_host,
    exact_select,
    fingerprint_atoms,
    matching_pursuit,
    orthogonal_matching_pursuit,
    predicted_ip_count,
    retained_count,
    stmp_select,
)
from .patches import PatchLayout, aggregate_patches, apply_batch, extract_patches
from .pipelines import code_patches
from .tree import FlatTree, from_reference_tree, load_structure, read_tree_file, write_tree_file

__all__ = [
    "FormatError", "StaleTreeError", "Dictionary", "EncodeResult", "ExactSelector",
    "GpuDictionary", "GpuTree", "ScoreCounter", "SearchParams", "SparseCode", "TreeSelector",
    "encode", "encode_host", "exact_select", "fingerprint_atoms", "matching_pursuit",
    "orthogonal_matching_pursuit", "predicted_ip_count", "retained_count", "stmp_select",
    "code_patches", "PatchLayout", "aggregate_patches", "apply_batch", "extract_patches", "FlatTree", "from_reference_tree", "load_structure", "read_tree_file", "write_tree_file",
]
