"""structfft on B200: the Hi-DFT hot path of arXiv 2211.15299 as sm_100a CUDA.

Drop-in names for the reference package's hot path (reference
__init__.py:10-92): SupportSet, pivots, classify, is_part_homogeneous,
pivoted_pattern, hidft, hidft_to_dft, sas_transform (mu* = 1), plus the
batched fused entry `hidft_to_dft_batched`.  All compute runs through the
C-ABI library libsfft_b200.so (include/structfft_b200.h); there is no CPU
fallback.
"""

from .congruence import (Classification, CongruenceTree, SupportSet, TreeNode, as_support,
                         assert_part_homogeneous, build_tree, classify, height_of, is_part_homogeneous,
                         level_weights, pivots, v2, validate_pivot_vector)
from .counting import OpCounter
from .errors import (BudgetExceededError, ContractViolationError, DeviceError, InvalidInputError,
                     StructFFTError)
from .hidft import (ButterflyPlan, HiDftResult, get_plan, hidft, hidft_to_dft, hidft_to_dft_batched,
                    hidft_to_dft_interleaved, stream_chain)
from .sampling import SamplingPattern, pivoted_pattern, pivoted_pattern_tensor
from .signals import BandlimitedSignal
from .sas import (CostReport, NodeSystem, SasPlan, SasResult, predicted_cost, sas_transform,
                  select_pivots)

__version__ = "0.1.0"
