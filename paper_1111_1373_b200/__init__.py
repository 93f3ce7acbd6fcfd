"""spectree_b200: B200-native classification-tree evaluation.

A drop-in GPU path for the reference ``spectree`` evaluate API
(/root/reference/proj/core): data decomposition (Algorithm 1) and speculative
decomposition with warp-shuffle pointer jumping (Algorithm 2), a random-forest
vote and a sample-sharded multi-GPU driver, as hand-written sm_100a CUDA behind
the C ABI in include/spectree_b200.h.  This package is the Python host mirror
of that boundary; the C++ mirror is include/spectree_b200.hpp.
"""
from .dataset import ClassAssignment, Dataset, tile_dataset
from .errors import (ArgumentError, CudaError, Error, IoError, NoDeviceError, ParseError,
                     SchemaError, StructureError)
from .evaluate import (VARIANTS, DataParallelConfig, Forest, GpuGeom, ReductionMode,
                       SpeculativeConfig, SpeculativeStats, check_attribute_range,
                       default_data_parallel, default_speculative, eval_data_parallel,
                       eval_depths_device, eval_device, eval_forest, eval_forest_device, eval_gpu,
                       eval_sharded, eval_speculative, eval_speculative_basic, last_launch_count,
                       mean_traversal_depth, traversal_depths, tree_info, validate_data_parallel,
                       validate_speculative)
from .frames import FrameStream
from .files import (dataset_info, eval_file, load_dataset_bin, load_labels_bin,
                    save_dataset_bin, save_labels_bin)
from .synthetic import (dataset_checksum, fnv1a64, generate_synthetic_dataset,
                        generate_synthetic_tree)
from .tree import (NO_CLASS, NODE_DTYPE, Diagnostic, EncodedTree, LinkedNode, decode,
                   encode_breadth_first, load_tree_json, load_tree_json_text, make_leaf,
                   make_split, processor_node_map, tree_to_json, validate)

__all__ = [n for n in dir() if not n.startswith("_")]
