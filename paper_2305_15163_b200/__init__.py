"""B200-native batched online solve of the DD NM-ROM with hyper-reduction
(arXiv 2305.15163) for 2-D steady Burgers.

Drop-in for the reference package's online path (``ddrom.driver.solve_rom``
-> ``build_problem`` -> ``init_guess`` -> ``sqp.iterate``), batched over many
parameters mu and executed by hand-written sm_100a CUDA kernels behind the C
ABI in ``include/ddnm.h`` (``libddnm.so``).  There is no CPU fallback.
"""

from .burgers import (A_RANGE, LAM_RANGE, FomOperators, Grid2D, ParameterPoint, assemble,
                      seeded_parameters)
from .driver import (BatchResult, BenchmarkRecord, DecodeBatch, EvalBatch, RomInstance,
                     RomSolution, build_problem, decode_batch, eval_gradients_batch, init_guess,
                     solve_rom, solve_rom_batch)
from .errors import ConvergenceError, FormatError, SingularityError
from .subdomain import (ShardedSolve, block_bounds,
                        solve_rom_batch_subdomain_sharded)
from .sqp import SqpBlock, SqpConfig, SqpProblem, SqpResult, iterate

__version__ = "0.1.0"

__all__ = [
    "A_RANGE", "LAM_RANGE", "FomOperators", "Grid2D", "ParameterPoint", "assemble",
    "seeded_parameters",
    "BatchResult", "BenchmarkRecord", "DecodeBatch", "EvalBatch", "RomInstance", "RomSolution",
    "build_problem", "decode_batch",
    "eval_gradients_batch", "init_guess", "solve_rom", "solve_rom_batch",
    "ConvergenceError", "FormatError", "SingularityError",
    "SqpBlock", "SqpConfig", "SqpProblem", "SqpResult", "iterate",
    "ShardedSolve", "block_bounds", "solve_rom_batch_subdomain_sharded",
]
