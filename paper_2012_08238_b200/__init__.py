"""B200-native (sm_100a) sparse-FFT bucketization hot path.

Drop-in, device-resident counterparts of the reference package's hot-path
entry points (``sparsefft``: bucketize_flat / bucketize_spike, robust_noise_floor,
vote_tally / select_by_votes, run_voting / run_iterative / run_peeling,
run_algorithm), backed by hand-written CUDA kernels in libsfft_b200.so and
called through its C ABI (include/sfft_b200.h).  No CPU fallback.
"""

from .errors import (AmbiguousSplit, ConfigMismatch, FilterKindMismatch, InvalidParameter,
                     InvalidSpec, LengthMismatch, NearZeroResponse, NonDivisorParameter,
                     NonInvertibleScaling, RankDeficient, SchemaError, SingularMomentMatrix,
                     SparseFFTError, ZeroTonBucket)
from .signal import PermutationParams, SparseSpectrum, TimeSignal, phase_factor
from .filters import (WindowFilter, default_flat_support, default_gauss_sigma,
                      filter_freq_shift, make_dirichlet_bank, make_flat_filter)
from .bucketize import (BucketSet, HashMapView, bucketize_dirichlet, bucketize_flat,
                        bucketize_flat_batch, bucketize_spike, bucketize_spike_batch, hash_view,
                        hash_view_for)

__version__ = "0.1.0"
from .reconstruct import (VoteTable, estimate_freqshift, robust_noise_floor, select_by_votes,
                          vote_tally)
from .frameworks import (FRAMEWORKS, AlgorithmConfig, BatchResult, RecoveryResult,
                         run_algorithm, run_iterative, run_iterative_batch, run_oneshot,
                         run_oneshot_batch,
                         run_iterative_stream, run_peeling,
                         run_peeling_batch, run_voting, run_voting_batch)
