/* mmfacts.h — facts ingest straight to the engine's CSR (libmmgpu.so).
 *
 * Replaces, at the C ABI:
 *   modmetrics::parse_facts(std::string_view)  facts.hpp:91-256
 *   modmetrics::load_facts(const std::string&) facts.hpp:258-265
 *   modmetrics::facts_to_json(model, deps)     facts.hpp:270-320
 * The reference goes text -> nlohmann DOM -> SystemModel/DependencyTable
 * (vector of vectors) -> (for the GPU) CSR. Here one streaming pass reads the
 * text into flat arrays and mm_facts_system() hands out an mm_system CSR view
 * that mm_upload() takes directly.
 *
 * Errors mirror the reference's exceptions: MM_E_PARSE <-> ParseError,
 * MM_E_VALIDATION <-> ValidationError (violations listed, same kinds/messages/
 * order), MM_E_IO <-> IoError, MM_E_RANGE <-> the nlohmann::json::out_of_range
 * (406, a float token overflowing a double) that escapes parse_facts
 * unwrapped; mm_facts_error() holds what() verbatim (for MM_E_RANGE: the
 * message after nlohmann's "[json.exception.out_of_range.406] " prefix). The
 * handle is returned even on failure so the caller can read the error; free
 * it with mm_facts_free. Host-only: no device is needed. */
#ifndef MMFACTS_H
#define MMFACTS_H

#include <stddef.h>
#include <stdint.h>

#include "mmgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* modmetrics::ViolationKind (model.hpp:72-85), same enumerator order. */
enum {
    MM_VK_NON_DENSE_CLASS_IDS = 0,
    MM_VK_DUPLICATE_METHOD_MEMBERSHIP = 1,
    MM_VK_DUPLICATE_ATTRIBUTE_MEMBERSHIP = 2,
    MM_VK_UNOWNED_METHOD = 3,
    MM_VK_UNOWNED_ATTRIBUTE = 4,
    MM_VK_OWNER_MISMATCH = 5,
    MM_VK_DEPENDENCY_TABLE_SIZE = 6,
    MM_VK_DANGLING_CALL_TARGET = 7,
    MM_VK_DANGLING_ACCESS_TARGET = 8,
    MM_VK_SELF_CALL = 9,
    MM_VK_UNSORTED_DEPENDENCY_SET = 10,
    MM_VK_UNSUPPORTED_SCHEMA_VERSION = 11
};

typedef struct mm_facts mm_facts;

/* parse_facts (facts.hpp:91). *out is always set (unless MM_E_ARG). */
mm_status mm_facts_parse(const char* text, size_t len, mm_facts** out);
/* load_facts (facts.hpp:258): MM_E_IO "cannot open <path>" / "read error on <path>". */
mm_status mm_facts_load(const char* path, mm_facts** out);
void mm_facts_free(mm_facts* f);

mm_status mm_facts_status(const mm_facts* f);
/* what() of the exception the reference would throw ("" on success). */
const char* mm_facts_error(const mm_facts* f);

/* CSR view of the loaded system (pointers live as long as f): the
 * ClassRecord lists in class order, sorted; owner tables; calls/accesses rows
 * sorted unique, self-calls dropped. MM_E_STATE if the parse failed. */
mm_status mm_facts_system(const mm_facts* f, mm_system* sys);

/* ValidationError::violations() (facts.hpp:33). */
uint32_t mm_facts_violation_count(const mm_facts* f);
mm_status mm_facts_violation(const mm_facts* f, uint32_t i, int* kind, const char** message);
/* LoadResult::warnings (facts.hpp:46). */
uint32_t mm_facts_warning_count(const mm_facts* f);
const char* mm_facts_warning(const mm_facts* f, uint32_t i);

/* ClassRecord::name, SystemModel::method_names / attribute_names (model.hpp:21,33-34):
 * UTF-8 bytes, not NUL-terminated (names may hold NUL); *len receives the size. */
const char* mm_facts_class_name(const mm_facts* f, uint32_t c, size_t* len);
const char* mm_facts_method_name(const mm_facts* f, uint32_t p, size_t* len);
const char* mm_facts_attribute_name(const mm_facts* f, uint32_t a, size_t* len);

/* facts_to_json (facts.hpp:270-320): canonical bytes, trailing newline.
 * Two-call size query: *n_out always receives the size; MM_E_CAPACITY when
 * out is NULL or cap is smaller. */
mm_status mm_facts_to_json(const mm_facts* f, char* out, size_t cap, size_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* MMFACTS_H */
