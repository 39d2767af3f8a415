"""Host compiler: circuit graph -> block-sparse layered IR (bit-exact contract)."""
from .blocks import PAD, BlockLayout, detect_blocks, detect_blocks_csr, pow2_floor
from .build import CompileConfig, compile_circuit, graph_hash, layerize, node_depths
from .cache import dumps_compiled, load_compiled, loads_compiled, save_compiled
from .ir import (BackwardGroupIR, CompiledCircuit, FlowPushIR, ForwardGroupIR,
                 InputLayerIR, LayerReport, ProductEvalIR, SumLayerIR)
from .partition import PartitionPlan, partition_layer, round_child_counts

__all__ = [
    "PAD", "BlockLayout", "detect_blocks", "detect_blocks_csr", "pow2_floor",
    "CompileConfig", "compile_circuit", "graph_hash", "layerize", "node_depths",
    "BackwardGroupIR", "CompiledCircuit", "FlowPushIR", "ForwardGroupIR",
    "InputLayerIR", "LayerReport", "ProductEvalIR", "SumLayerIR",
    "PartitionPlan", "partition_layer", "round_child_counts",
    "dumps_compiled", "loads_compiled", "save_compiled", "load_compiled",
]
