"""B200-native FastGM (arXiv 2302.05176): Gumbel-Max sketches on sm_100a.

Drop-in for the reference package ``gmsketch`` (its public names,
gmsketch/__init__.py:12-109), with every sketch computation in the CUDA
library libgmsketch_b200.so (C ABI: include/gmsketch_b200.h) and batched
entry points (sketch_csr, sketch_elements, sketch_pairs, merge_arrays,
estimate_jaccard_p_batch) for device-resident data.  There is no CPU
fallback: without the library or an sm_100 GPU, sketch calls raise.
"""

from .errors import (
    DatasetParseError,
    DeviceError,
    EmptyVectorError,
    GmSketchError,
    IncompleteSketchError,
    InconsistentWeightError,
    InvalidParameterError,
    InvalidWeightError,
    MismatchedSketchError,
    MissingElementError,
    QueueExhaustedError,
    UnknownDistributionError,
)
from .estimate import (
    CardinalityEstimate,
    SetAlgebraEstimate,
    SimilarityEstimate,
    estimate_cardinality,
    estimate_difference,
    estimate_jaccard_p,
    estimate_jaccard_p_batch,
    estimate_cardinality_batch,
    estimate_set_algebra,
    exact_jaccard_p,
    exact_jaccard_w,
    merge,
    merge_arrays,
)
from .randgen import (
    DEFAULT_STREAM_SALT,
    ElementQueueState,
    LazyPermutation,
    advance_queues,
    SeedScheme,
    derive_seed,
    mix64,
    next_order_statistic,
    perm_draw_batch,
    rand_int_between,
    uniform_open,
    uniform_open_batch,
)
from .sketch import (
    GenerationParams,
    GumbelMaxSketch,
    SketchBatch,
    WeightedVector,
    check_compatible,
    compute_ri,
    sketch_csr,
    sketch_csr_seeded,
    sketch_vector_seeds,
    sketch_csr_host,
    sketch_csr_host_many,
    exact_y_host,
    sketch_elements,
    sketch_elements_many,
    sketch_fast,
    sketch_fast_counted,
    sketch_from_json,
    sketch_many,
    sketch_naive,
    sketch_naive_counted,
    sketch_to_json,
)
from .stream import (
    StreamSketchState,
    parse_stream_items,
    sketch_pairs,
    sketch_stream,
    stream_finalize,
    stream_update,
)

__version__ = "0.1.0"
